"""Calibration: cost of writing C1's output (6.4 MB) per step with torch
kernels, timed like bench.py (CUDA graph of K steps, rotating buffers)."""
import torch
dev = torch.device("cuda", 0)
K, SETS = 200, 6
n_out = 8 * 64 * 56 * 56
outs = [torch.empty(n_out, device=dev) for _ in range(SETS)]
ins = [torch.rand(8 * 64 * 112 * 112, device=dev) for _ in range(SETS)]
def timed(fn):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        for i in range(K): fn(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3
print("fill 6.4MB us", round(timed(lambda i: outs[i % SETS].fill_(1.0)), 2))
print("empty-ish fill 4KB us", round(timed(lambda i: outs[i % SETS][:1024].fill_(1.0)), 2))
print("copy 25.7MB->6.4MB (strided read 1/4) us", round(timed(lambda i: outs[i % SETS].copy_(ins[i % SETS][::4])), 2))
