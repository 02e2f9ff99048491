"""One-off probe of the GPU box: device props, host cores, cuBLAS fp64/fp32 GEMM peaks, copy bandwidth."""
import json, os, platform, subprocess, time
import torch

out = {}
p = torch.cuda.get_device_properties(0)
out["name"] = p.name
out["sms"] = p.multi_processor_count
out["l2_bytes"] = getattr(p, "L2_cache_size", None)
out["mem_bytes"] = p.total_memory
out["cpu_count"] = os.cpu_count()
try:
    out["cpu_model"] = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
except Exception as e:
    out["cpu_model"] = str(e)
out["sched_affinity"] = len(os.sched_getaffinity(0))

def bench(fn, iters=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(iters):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    return best

for dt, n in ((torch.float64, 8192), (torch.float32, 8192)):
    a = torch.randn(n, n, device="cuda", dtype=dt); b = torch.randn(n, n, device="cuda", dtype=dt)
    torch.backends.cuda.matmul.allow_tf32 = False
    t = bench(lambda: a @ b)
    out[f"gemm_{dt}_{n}_tflops"] = 2 * n**3 / t / 1e12
for n in (4000,):
    a = torch.randn(n, n, device="cuda", dtype=torch.float64); b = torch.randn(n, n, device="cuda", dtype=torch.float64)
    t = bench(lambda: a @ b)
    out[f"dgemm_{n}_tflops"] = 2 * n**3 / t / 1e12
    out[f"dgemm_{n}_ms"] = t * 1e3
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda"); y = torch.empty_like(x)
t = bench(lambda: y.copy_(x))
out["copy_1GiB_GBs"] = 2 * (1 << 30) / t / 1e9
x = torch.empty(64 << 20, dtype=torch.uint8, device="cuda"); y = torch.empty_like(x)
t = bench(lambda: y.copy_(x), 50)
out["copy_64MiB_GBs(L2)"] = 2 * (64 << 20) / t / 1e9
print(json.dumps(out, indent=1))
print(subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout)
