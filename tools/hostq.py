"""Is the back-to-back solve loop host-bound?  Times the host side of K
enqueue calls (perf_counter) against the device time of the same K solves
(CUDA events), config 3 bucket engine.   python tools/hostq.py [K]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2504_03667_b200 as P
K = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sampler = None
if os.environ.get("HOSTQ_SAMPLER"):  # bench.py's nvidia-smi clock sampler running meanwhile
    import bench
    sampler = bench.ClockSampler(0)
    sampler.start()
g = P.generate_dense(32768, 32768)
srcs = [(7919 * i) % 32768 for i in range(K)]
with P.DeviceGraph(g) as dg:
    stream = torch.cuda.ExternalStream(dg.stream_ptr())
    for s in srcs[:3]:
        dg.enqueue([s]); dg.finish()
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        t0 = time.perf_counter()
        for s in srcs:
            dg.enqueue([s])
        t1 = time.perf_counter()
        e1.record(stream)
        st = dg.finish()
        torch.cuda.synchronize()
        print(f"K={K} host enqueue {1e6 * (t1 - t0) / K:.2f} us/solve, device {1e3 * e0.elapsed_time(e1) / K:.2f} us/solve, "
              f"lib kernel {st['rounds_s'] * 1e6:.2f} us", flush=True)
    # the same with a long GPU job queued first: the host runs ahead, the device time is launch-limited
    for rep in range(2):
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            torch.cuda._sleep(50_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in srcs:
            dg.enqueue([s])
        e1.record(stream)
        st = dg.finish()
        torch.cuda.synchronize()
        print(f"K={K} pre-queued: device {1e3 * e0.elapsed_time(e1) / K:.2f} us/solve", flush=True)
if sampler:
    print("clocks", sampler.stop())
