"""One config-4 solve per launch for ncu capture (n=65536 Bernoulli 0.001 directed):
python tools/prof_cfg4.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2504_03667_b200 as P
g = P.generate_bernoulli(65536, 0.001, 65536, directed=True)
with P.DeviceGraph(g, engine="bucket") as dg:
    for _ in range(2):
        r = dg.solve(0)
    print(r.stats)
