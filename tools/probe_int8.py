"""Probe: int8 tensor-core GEMM throughput on this B200 (cuBLASLt via
torch._int_mm) at the shapes an Ozaki-sliced sketch would issue."""
import torch, time
from torch.profiler import profile, ProfilerActivity
dev = "cuda"
def bench(M, K, N, reps=10):
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev).t()  # column-major B
    for _ in range(3):
        c = torch._int_mm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c = torch._int_mm(a, b)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"int8 {M}x{K}x{N}: {ms:.3f} ms  {2*M*K*N/ms/1e9:.1f} TOPS", flush=True)
    return a, b
for shp in [(8192, 8192, 8192), (16384, 16384, 16384), (4096, 27136, 3584), (4096, 27136, 512), (7168, 4096, 27136), (1024, 4096, 27136), (31360, 27136, 512)]:
    try:
        bench(*shp)
    except Exception as ex:
        print("fail", shp, ex)
a, b = bench(8192, 8192, 8192, 2)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    torch._int_mm(a, b); torch.cuda.synchronize()
print(set(e.name for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA))
x = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
for _ in range(3): y = x @ x
torch.cuda.synchronize(); t = time.time()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): y = x @ x
e1.record(); torch.cuda.synchronize()
print("bf16 8192^3 TFLOPS", 2*8192**3/(e0.elapsed_time(e1)/10)/1e9)
