import torch, time
n = 1 << 30  # 2 GB bf16
a = torch.empty(n, dtype=torch.bfloat16).pin_memory()
b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
for chunk in (4 << 20, 64 << 20, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(0, n, chunk):
        b[i:i + chunk].copy_(a[i:i + chunk], non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    print("1 stream chunk", chunk * 2 >> 20, "MB:", round(n * 2 / e0.elapsed_time(e1) / 1e6, 1), "GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
h = n // 2
with torch.cuda.stream(s1):
    for i in range(0, h, 4 << 20): b[i:i + (4 << 20)].copy_(a[i:i + (4 << 20)], non_blocking=True)
with torch.cuda.stream(s2):
    for i in range(h, n, 4 << 20): b[i:i + (4 << 20)].copy_(a[i:i + (4 << 20)], non_blocking=True)
torch.cuda.synchronize()
print("2 streams:", round(n * 2 / (time.perf_counter() - t0) / 1e9, 1), "GB/s")
