import torch, time
for mb in (1, 4, 12, 64, 256):
    n = mb * 1024 * 1024 // 4
    h = torch.empty(n, dtype=torch.int32, pin_memory=True)
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    for direction in ("h2d", "d2h"):
        s = torch.cuda.current_stream()
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"{direction} {mb} MB: {ms*1000:.1f} us, {mb*1.048576/ms:.1f} GB/s")
# zero-copy kernel read of host memory (12 MB)
n = 3 * 1024 * 1024
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
d = torch.empty(n, dtype=torch.int32, device="cuda")
print(torch.cuda.get_device_properties(0))
