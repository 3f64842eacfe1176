"""Harness integration: kCsvHeader-compatible rows (bench.hpp:369-403),
efficiency arithmetic (bench.hpp:97-102, acceptance criterion 4), and the
device-side validated timed_run (bench.hpp:114-180)."""
import csv
import io

import numpy as np
import pytest

from paper_2504_03667_b200 import harness as H


def test_header_matches_reference_columns():
    ref_cols = ("engine,graph_id,n,m,workers,reps,phase_scatter_s,phase_rounds_s,phase_gather_s,"
                "phase_transfer_in_s,phase_transfer_out_s,phase_algorithm_s,total_s,"
                "allreduce_count,relax_checks,seed")
    assert H.KCSV_HEADER == ref_cols


def test_csv_row_shape(tmp_path):
    r = H.TimingRecord(engine="cuda-bucket", graph_id="dense:100:5", n=100, m=4950, workers=1,
                       reps=3, phase_transfer_in_s=0.01, phase_rounds_s=0.001,
                       phase_transfer_out_s=0.0001, total_s=0.0111, allreduce_count=4,
                       relax_checks=1000, seed=5, rows_read=10, classes=4, algorithmic_bytes=1000)
    p = tmp_path / "r.csv"
    H.write_csv([r], str(p))
    rows = list(csv.reader(open(p)))
    assert len(rows[0]) == len(rows[1]) == 16 + 4
    assert rows[1][0] == "cuda-bucket" and rows[1][6] == "" and rows[1][7] == "0.001000000"


def test_strong_scaling_efficiency_table5():
    # acceptance.cpp:115-129 / PAPER Table 5: p=2, 10.28 s -> 7.67 s = 67.01 %
    assert round(H.strong_scaling_efficiency(10.28, 7.67, 2), 2) == 67.01
    with pytest.raises(ValueError):
        H.strong_scaling_efficiency(0, 1, 1)


@pytest.mark.gpu
def test_timed_run_validates_on_device(gpu, oracle_c):
    g = gpu.generate_dense(2000, 9)
    rec, res = H.timed_run(g, 3, reps=2, graph_id="dense:2000:9", seed=9)
    d, p = oracle_c.serial(g.adj, g.n, 3)
    assert np.array_equal(res.dist, d) and np.array_equal(res.pred, p)
    assert rec.engine == "cuda-bucket" and rec.m == 2000 * 1999 // 2
    assert H.csv_row(rec).startswith("cuda-bucket,dense:2000:9,2000,")
    # a corrupted result is caught by the device validator
    with gpu.DeviceGraph(g) as dg:
        r = dg.solve(3)
        assert dg.validate(r) == 0
        r.dist[17] += 1
        assert dg.validate(r) > 0
        r.dist[17] -= 1
        r.pred[25] = 1999 if r.pred[25] != 1999 else 1998
        assert dg.validate(r) > 0
