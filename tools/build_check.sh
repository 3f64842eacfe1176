#!/bin/bash
# Rebuild everything and fail loudly (used before every gpurun).
set -e
cd "$(dirname "$0")/.."
make -j3 -s -C paper_2504_03667_b200/csrc
make -s -C oracle
python -c "import __graft_entry__ as g; g.build()"
