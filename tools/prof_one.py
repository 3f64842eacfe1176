"""One solve per engine for ncu capture: python tools/prof_one.py [n] [engine] [warps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03667_b200 as P
n = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
engine = sys.argv[2] if len(sys.argv) > 2 else "cluster"
warps = int(sys.argv[3]) if len(sys.argv) > 3 else 0
flags = int(sys.argv[4]) if len(sys.argv) > 4 else None
g = P.generate_dense(n, 32768)
with P.DeviceGraph(g, engine=engine, warps=warps, flags=flags) as dg:
    for _ in range(2):
        r = dg.solve(0)
    print(r.stats)
