"""Per-CTA busy time of k_beamform_tc (developer diagnostic; needs a library
built with -DSNB_TC_EXP_TIMES: scripts/ab_build.sh tct -DSNB_TC_EXP_TIMES)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2208_10839_b200 as sn
lib_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2208_10839_b200/_lib/ab/libtct.so")
sn.load_library(lib_path)
lib = ctypes.CDLL(lib_path)
cfg = sn.default_pipeline_config(2)
ws = sn.Workspace(cfg, device=0, max_batch=16)
scene = sn.Scene([sn.Reflector(1.5, 0.2, 0.0, 0.8), sn.Reflector(3.0, -0.4, 0.1, 0.5)], 0.01, 7)
pk = sn.synthesize_measurement(cfg, scene).packed
dp = torch.from_numpy(np.tile(pk, 16)).cuda()
out = torch.empty(16 * ws.n_dirs * ws.bins, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
iters = 20
for _ in range(iters):
    ws.process_device(dp.data_ptr(), 16, out.data_ptr(), s.cuda_stream)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 4096)()
assert lib.sn_debug_tc_times(buf, 4096) == 0
a = np.frombuffer(buf, dtype=np.uint64)[:2048].reshape(-1, 4)
full = np.frombuffer(buf, dtype=np.uint64)
bb = full[2048:2048 + 2 * 512].reshape(-1, 2)
keep = (a[:, 1] > 0) & (bb[:len(a), 0] > 0)
print("CTAs with a launch:", int((a[:, 1] > 0).sum()), "with tiles:", int(keep.sum()))
a = a[keep]
bsel = bb[:len(keep)][keep]
np.save(os.environ.get("TC_NPY", "gpurun_out/tc_times.npy"), np.concatenate([a, bsel], 1))
mma = a[:, 0] / a[:, 1] / 1e3
all_ = a[:, 2] / a[:, 1] / 1e3
print(f"CTAs {len(a)}, launches {int(a[0,1])}")
print(f"MMA-warp busy us per launch: min {mma.min():.1f} mean {mma.mean():.1f} max {mma.max():.1f}")
print(f"epilogue (thread 0) us per launch: min {all_.min():.1f} mean {all_.mean():.1f} max {all_.max():.1f}")
print("imbalance max/mean:", round(all_.max() / all_.mean(), 3))
print("sorted (us):", np.round(np.sort(all_)[::10], 1).tolist())
n = len(a)
b = bsel.astype(float) / a[:, 1:2]
sumR = a[:, 3] / a[:, 1]
tiles, sw = b[:, 0], b[:, 1]
X = np.stack([tiles, sumR, sw], 1)
coef, res, *_ = np.linalg.lstsq(X, all_, rcond=None)
pred = X @ coef
print("fit us = %.3f*tiles + %.4f*sumR + %.2f*switches; rms resid %.2f us" % (coef[0], coef[1], coef[2], np.sqrt(np.mean((pred - all_) ** 2))))
print("per tile at R: " + ", ".join(f"R={r}: {coef[0] + coef[1] * r:.2f}" for r in (5, 10, 15, 20, 25, 30)))
order = np.argsort(all_)
for i in list(order[:5]) + list(order[-5:]):
    print(f"  cta {i:3d} t={all_[i]:7.1f} tiles={tiles[i]:.0f} sumR={sumR[i]:.0f} avgR={sumR[i]/max(tiles[i],1):.1f} switches={sw[i]:.0f}")
