"""Times the GPU load generator (sn_synthesize_device) for N hemisphere3000 captures (developer diagnostic)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2208_10839_b200 as sn
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
cfg = sn.default_pipeline_config(sn.GridKind.hemisphere3000)
ws = sn.Workspace(cfg, device=-1)
scenes = [sn.Scene([sn.Reflector(1.0 + 0.001 * (i % 1000), 0.1, 0.0, 0.8)], 0.01, 100 + i) for i in range(n)]
d = torch.empty(n * ws.packed_bytes, dtype=torch.uint8, device="cuda")
sn.synthesize_device(cfg, scenes[:2], d.data_ptr(), device=0)
torch.cuda.synchronize()
t0 = time.perf_counter()
sn.synthesize_device(cfg, scenes, d.data_ptr(), device=0)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"{n} captures in {dt:.3f} s: {n / dt:.1f} captures/s")
