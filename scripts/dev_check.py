"""Developer diagnostic: stage-by-stage GPU vs reference-oracle comparison + rough timing."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import pyoracle as po
import paper_2208_10839_b200 as sn

r = po.Ref()

def rel_rms(a, b):
    a = a.astype(np.float64); b = b.astype(np.float64)
    return float(np.sqrt(((a - b) ** 2).sum() / max((b ** 2).sum(), 1e-300)))

def check(kind, max_range=5.0, precision=0, custom=None):
    cfg = sn.default_pipeline_config(kind if custom is None else 0)
    rc = r.default_config(kind if custom is None else 0)
    if custom is not None:
        cfg = cfg.copy(directions=custom, grid_kind=3); rc = rc.copy(directions=custom, grid_kind=3)
    cfg = cfg.copy(max_range=max_range, precision=precision); rc = rc.copy(max_range=max_range)
    rws = r.workspace(rc)
    refl = [(1.5 if max_range >= 2 else 0.6, 0.2, 0.0, 0.8), (min(3.0, max_range*0.6), -0.4, 0.1, 0.5)]
    pk = r.synthesize(rc, refl, 0.01, 7)
    t = time.time(); e_ref = rws.process(pk); t_ref = time.time() - t
    ws = sn.Workspace(cfg, device=0, max_batch=4)
    m = sn.RawMeasurement(1, 0, 0, 32, ws.frames, cfg.pdm_rate, pk)
    img = ws.process(m)
    print(f"== kind={kind} max_range={max_range} prec={precision} dims={ws.n_dirs}x{ws.bins} ref {t_ref*1e3:.1f} ms")
    for st in range(3):
        a = ws.stage(st); b = rws.stage(st)
        print(f"  stage {st}: bit-exact={np.array_equal(a, b)} maxabs={np.abs(a-b).max():.3e} relrms={rel_rms(a, b):.3e}")
    e = img.energies
    print(f"  energies: bit-exact={np.array_equal(e, e_ref)} relrms={rel_rms(e, e_ref):.3e} "
          f"maxabs/peak={np.abs(e-e_ref).max()/e_ref.max():.3e} argmax {img.argmax()} vs {np.unravel_index(e_ref.argmax(), e_ref.shape)}")
    # timing (host path)
    import torch
    for B in (1, 4):
        ms = [m] * B
        ws.process_batch(ms)
        torch.cuda.synchronize()
        t = time.time(); n = 5
        for _ in range(n): ws.process_batch(ms)
        dt = (time.time() - t) / n
        print(f"  host path B={B}: {dt*1e3:.3f} ms/call -> {B/dt:.1f} energyscapes/s")
    # device path
    dp = torch.from_numpy(np.tile(pk, 4)).cuda()
    de = torch.empty(4 * ws.n_dirs * ws.bins, dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): ws.process_device(dp.data_ptr(), 4, de.data_ptr(), s)
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(); n = 10
    for _ in range(n): ws.process_device(dp.data_ptr(), 4, de.data_ptr(), s)
    ev1.record(); torch.cuda.synchronize()
    ms_ = ev0.elapsed_time(ev1) / n
    print(f"  device path B=4: {ms_:.3f} ms -> {4/ms_*1e3:.1f} energyscapes/s")
    d = de.view(4, ws.n_dirs, ws.bins).cpu().numpy()
    print(f"  device result == host result: {np.array_equal(d[3], e)}")

check(0)
check(0, max_range=1.5)
check(2)
check(2, precision=1)
check(0, custom=po.az181_directions())
