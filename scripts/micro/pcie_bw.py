"""Host<->device copy bandwidth with pinned host buffers (developer diagnostic):
the e2e leg moves 7.86 MB of energies per capture back to the host."""
import torch, time
dev = torch.device("cuda:0")
for mb in (8, 126, 1024):
    n = mb * 1024 * 1024 // 4
    d = torch.empty(n, dtype=torch.float32, device=dev)
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    for name, fn in (("D2H", lambda: h.copy_(d, non_blocking=True)), ("H2D", lambda: d.copy_(h, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = max(3, 2048 // mb)
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{name} {mb:5d} MB: {mb * 1.048576 / ms:7.1f} GB/s ({ms:.3f} ms)")
