"""Small invocations of every device path for compute-sanitizer (developer
diagnostic): python scripts/sanitize_run.py; run under
  compute-sanitizer --tool memcheck|racecheck|synccheck python scripts/sanitize_run.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2208_10839_b200 as sn

base = sn.default_pipeline_config(sn.GridKind.horizontal90)
cfgs = {
    "h90_1.5m (pair2048)": base.copy(max_range=1.5),
    "h90_5m (FFT FIR, TC N=64)": base,
    "box_5m (TC N=96)": sn.default_pipeline_config(sn.GridKind.box1850).copy(
        directions=sn.direction_grid(sn.GridKind.box1850)[:300], grid_kind=3),
    "h90_10m (split8192)": base.copy(max_range=10.0),
    "h90_5m f32": base.copy(precision=1),
}
for name, cfg in cfgs.items():
    m = [sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(0.9 + 0.2 * i, 0.1, 0.0, 0.6)], 0.01, 3 + i), seq=i)
         for i in range(3)]
    ws = sn.Workspace(cfg, device=0, max_batch=2, beam_budget_bytes=1)  # ring of one capture
    e = [im.energies for im in ws.process_batch(m)]
    d = torch.from_numpy(np.stack([x.packed for x in m[:2]])).cuda()
    out = torch.empty((2, ws.n_dirs, ws.bins), dtype=torch.float32, device="cuda")
    ws.process_device(d.data_ptr(), 2, out.data_ptr())
    ws.process_device(d.data_ptr(), 2, out.data_ptr(), graph=True)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy()[0], e[0])
    beams = ws.stage(3, 1)
    fr = ws.process_frames([sn.measurement_frame(x) for x in m])
    tr = torch.empty_like(out)
    sn.energyscape_transform(out.data_ptr(), tr.data_ptr(), 2, ws.n_dirs * ws.bins)
    torch.cuda.synchronize()
    print(name, "ok", float(np.max(e[2])), beams.shape, [s for s, _ in fr])
