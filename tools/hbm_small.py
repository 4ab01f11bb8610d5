"""Achievable HBM rate for C1-sized transfers (25.7 MB in, 6.4 MB out):
torch copies of the same byte counts, timed like bench.py (CUDA graph of K
steps, rotating buffers larger than L2)."""
import torch, json
dev = torch.device("cuda", 0)
K, SETS = 50, 6
def timed(fn):
    for i in range(3): fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.graph(g, stream=s):
        for i in range(K): fn(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()  # the first replay uploads the graph
    torch.cuda.synchronize(); e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3
n_in, n_out = 8 * 64 * 112 * 112, 8 * 64 * 56 * 56
ins = [torch.rand(n_in, device=dev) for _ in range(SETS)]
outs = [torch.empty(n_out, device=dev) for _ in range(SETS)]
big = [torch.empty(n_in, device=dev) for _ in range(SETS)]
res = {}
res["copy_in_to_in_us"] = timed(lambda i: big[i % SETS].copy_(ins[i % SETS]))
res["copy_out_us"] = timed(lambda i: outs[i % SETS].copy_(ins[i % SETS][:n_out]))
res["maxpool_torch_us"] = timed(lambda i: torch.nn.functional.max_pool2d(ins[i % SETS].view(8, 64, 112, 112), 3, 2, 1))
v = [x.view(8, 64, 112, 112) for x in ins]
res["strided_read_sum_us"] = timed(lambda i: torch.sum(ins[i % SETS]))
for k, t in list(res.items()):
    print(k, round(t, 2))
print("copy_in rate GB/s", round(2 * n_in * 4 / res["copy_in_to_in_us"] / 1e3, 1))
print("read+write C1 bytes at copy_in rate -> us", round((n_in + n_out) * 4 / (2 * n_in * 4 / res["copy_in_to_in_us"]), 2))
