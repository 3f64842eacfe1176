"""One data-parallel solve for ncu capture: python tools/prof_dp.py [n]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03667_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
g = P.generate_dense(n, 32768)
with P.DeviceGraph(g) as dg:
    for _ in range(2):
        r = dg.solve_dataparallel(0)
    print(r.stats)
