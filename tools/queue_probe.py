import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2504_03667_b200 as P
g = P.generate_dense(32768, 32768)
dg = P.DeviceGraph(g, engine="bucket", max_batch=64)
stream = torch.cuda.ExternalStream(dg.stream_ptr())
for _ in range(3):
    dg.enqueue([0]); dg.finish()
def timeit(fn, K):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream); t = time.perf_counter(); fn(); th = time.perf_counter() - t; e1.record(stream)
    st = dg.finish(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3, th / K * 1e6
for K in (20, 200):
    print("python loop K=%d: %.2f us/solve (host %.2f us/enqueue)" % ((K,) + timeit(lambda: [dg.enqueue([0]) for _ in range(K)], K)))
for K in (20, 64):
    print("one enqueue k=%d: %.2f us/solve (host %.2f us)" % ((K,) + timeit(lambda: dg.enqueue([0] * K), K)))
