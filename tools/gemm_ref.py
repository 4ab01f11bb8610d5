"""Calibration: cuBLAS bf16 GEMM time for C4's implicit-GEMM shape
(M = 256*28*28 = 200704 output pixels, N = 256 output channels, K = 1152),
the same FLOPs as the C4 convolution without the im2col gather.  Reference
point only (the product path never calls cuBLAS)."""
import torch

M, N, K = 256 * 28 * 28, 256, 128 * 9
a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
for out_dtype in (torch.bfloat16, torch.float32):
    c = torch.empty(M, N, device="cuda", dtype=out_dtype)
    f = (lambda: torch.matmul(a, b, out=c)) if out_dtype == torch.bfloat16 else \
        (lambda: torch.mm(a, b, out_dtype=torch.float32, out=c))
    try:
        for _ in range(10):
            f()
    except Exception as e:  # out_dtype overload missing in this torch
        print("skip", out_dtype, e)
        continue
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    print(f"cuBLAS bf16 {M}x{N}x{K} -> {out_dtype}: {us:.1f} us  {2 * M * N * K / us / 1e6:.0f} TFLOP/s")


# cuDNN convolutions of the C3 / C4 shapes (library reference points)
def t(f, n=30):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


torch.backends.cudnn.benchmark = True
F = torch.nn.functional
for tf32 in (False, True):
    torch.backends.cudnn.allow_tf32 = tf32
    torch.backends.cuda.matmul.allow_tf32 = tf32
    x = torch.rand(32, 64, 56, 56, device="cuda") * 2 - 1
    w = torch.randn(64, 64, 3, 3, device="cuda") * 0.0589
    us = t(lambda: F.conv2d(x, w, padding=1))
    print(f"cuDNN C3 conv fp32 (tf32={tf32}): {us:.1f} us  {2 * 32 * 64 * 56 * 56 * 576 / us / 1e6:.0f} TFLOP/s")
x = (torch.rand(256, 128, 56, 56, device="cuda") * 2 - 1).bfloat16()
w = (torch.randn(256, 128, 3, 3, device="cuda") * 0.0417).bfloat16()
us = t(lambda: F.conv2d(x, w, stride=2, padding=1))
print(f"cuDNN C4 conv bf16 NCHW (bf16 out): {us:.1f} us  {118380036096 / us / 1e6:.0f} TFLOP/s")
xc, wc = x.to(memory_format=torch.channels_last), w.to(memory_format=torch.channels_last)
us = t(lambda: F.conv2d(xc, wc, stride=2, padding=1))
print(f"cuDNN C4 conv bf16 NHWC (bf16 out): {us:.1f} us  {118380036096 / us / 1e6:.0f} TFLOP/s")
