"""The C-ABI boundary without a GPU: libsssp_cuda.so loads, exports every
function include/*.h declares, and fails loudly (no CPU fallback)."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for hdr in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(hdr).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(sssp_[a-z_0-9]+)\s*\(", src, re.M):
            names.add(m.group(1))
    return names


def test_headers_declare_the_boundary():
    names = declared_functions()
    for must in ("sssp_graph_create", "sssp_solve", "sssp_solve_batch", "sssp_graph_destroy",
                 "sssp_shard_create", "sssp_shard_export", "sssp_shard_connect", "sssp_status_string",
                 "sssp_gen_dense", "sssp_probe_sync"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2504_03667_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_native.EXPORTED) == declared_functions()


def test_abi_constants_and_strings():
    from paper_2504_03667_b200 import _native
    assert _native.lib.sssp_abi_version() == 3
    for code in range(9):
        assert _native.lib.sssp_status_string(code)
    assert ctypes.sizeof(_native.Options) == 56
    assert ctypes.sizeof(_native.Stats) == 168


def test_struct_layout_matches_header():
    """Compile a probe against include/sssp_cuda.h and compare struct sizes."""
    import subprocess
    import tempfile
    from paper_2504_03667_b200 import _native
    src = ('#include "sssp_cuda.h"\n#include <stdio.h>\n#include <stddef.h>\n'
           'int main(){printf("%zu %zu %zu\\n", sizeof(sssp_options), sizeof(sssp_solve_stats),'
           ' offsetof(sssp_solve_stats, weight_bytes));return 0;}\n')
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", os.path.join(d, "p"), c],
                       check=True)
        out = subprocess.run([os.path.join(d, "p")], capture_output=True, text=True, check=True)
    a, b, off = map(int, out.stdout.split())
    assert a == ctypes.sizeof(_native.Options) and b == ctypes.sizeof(_native.Stats)
    assert off == _native.Stats.weight_bytes.offset


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2504_03667_b200 as P
    g = P.generate_dense(16, 1)
    with pytest.raises(P.SsspError) as ei:
        P.dijkstra(g, 0)
    assert ei.value.status == 5  # SSSP_ERR_CUDA
