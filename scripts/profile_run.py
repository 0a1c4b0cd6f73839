"""Small driver for ncu captures: builds a workspace and runs the device path."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2208_10839_b200 as sn
p = argparse.ArgumentParser()
p.add_argument("--grid", default="hemisphere3000"); p.add_argument("--batch", type=int, default=1)
p.add_argument("--iters", type=int, default=3); p.add_argument("--precision", default="f64")
p.add_argument("--max-range", type=float, default=5.0)
p.add_argument("--lib", default=None)
a = p.parse_args()
if a.lib:
    sn.load_library(a.lib)
kind = {"horizontal90": 0, "box1850": 1, "hemisphere3000": 2}[a.grid]
cfg = sn.default_pipeline_config(kind).copy(precision=0 if a.precision == "f64" else 1, max_range=a.max_range)
ws = sn.Workspace(cfg, device=0, max_batch=a.batch)
scene = sn.Scene([sn.Reflector(min(1.5, 0.6 * a.max_range), 0.2, 0.0, 0.8), sn.Reflector(min(3.0, 0.8 * a.max_range), -0.4, 0.1, 0.5)], 0.01, 7)
pk = sn.synthesize_measurement(cfg, scene).packed
dp = torch.from_numpy(np.tile(pk, a.batch)).cuda()
out = torch.empty(a.batch * ws.n_dirs * ws.bins, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
for _ in range(a.iters):
    ws.process_device(dp.data_ptr(), a.batch, out.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
print("done", out.view(a.batch, ws.n_dirs, ws.bins)[0].max().item())
