"""Developer check: tensor-core beamformer vs the CUDA-core tiled kernel and the
reference oracle, several configs (run on the GPU box)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle")); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2208_10839_b200 as sn
import pyoracle as po
from conftest import az181, TINY, to_oracle

def rel(a, b):
    a = a.astype(np.float64); b = b.astype(np.float64)
    return float(np.sqrt(((a - b) ** 2).sum() / max((b ** 2).sum(), 1e-300)))

def ulp_ok(got, want):
    w32 = want.astype(np.float32)
    tol = np.spacing(np.abs(w32)).astype(np.float64) + 1e-12 * max(float(want.max()), 1e-30)
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    return int((d > tol).sum()), float(np.mean(got == w32))

ref = po.Ref()
base = sn.default_pipeline_config(sn.GridKind.horizontal90)
cfgs = {"tiny": base.copy(**TINY), "small": base.copy(max_range=1.5), "h90": base,
        "az181": base.copy(directions=az181(), grid_kind=3),
        "box1850": sn.default_pipeline_config(sn.GridKind.box1850),
        "hemi3000": sn.default_pipeline_config(sn.GridKind.hemisphere3000)}
for name, cfg in cfgs.items():
    for prec in (0, 1):
        c = cfg.copy(precision=prec)
        m = sn.synthesize_measurement(c, sn.Scene([sn.Reflector(0.8 if name == "tiny" else 1.4, 0.2, 0.1, 0.8)], 0.01, 3))
        e_tc = sn.Workspace(c, device=0).process(m).energies
        e_ti = sn.Workspace(c, device=0, beamformer=sn.Beamformer.cuda_core).process(m).energies
        want = ref.workspace(to_oracle(po, c)).process(m.packed)
        bad, same = ulp_ok(e_tc, want)
        print(f"{name:9s} prec={prec} tc-vs-ref rel {rel(e_tc, want):.2e} beyond1ulp {bad} same {same:.4f} | "
              f"tiles-vs-ref rel {rel(e_ti, want):.2e} | tc-vs-tiles rel {rel(e_tc, e_ti):.2e} argmax {np.unravel_index(e_tc.argmax(), e_tc.shape)} {np.unravel_index(want.argmax(), want.shape)}", flush=True)
