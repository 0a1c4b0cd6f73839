import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2208_10839_b200 as sn
cfg = sn.default_pipeline_config(sn.GridKind.hemisphere3000)
ws = sn.Workspace(cfg, device=0, max_batch=16)
pk = sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(1.5, 0.2, 0.0, 0.8)], 0.01, 7)).packed
for EB in (16, 64, 128):
    pin_in = torch.from_numpy(np.tile(pk, (EB, 1))).pin_memory(); pin_out = torch.empty((EB, ws.n_dirs, ws.bins), dtype=torch.float32).pin_memory()
    a, b = pin_in.numpy(), pin_out.numpy()
    ws.process_packed_host(a, b); torch.cuda.synchronize()
    # host-side struct building cost alone
    import ctypes as C
    t0 = time.perf_counter()
    for _ in range(20):
        structs = (sn._Measurement * EB)()
        base = a.ctypes.data
        for i in range(EB):
            structs[i] = sn._Measurement(1, 0, i, 32, ws.frames, cfg.pdm_rate, C.cast(base + i * ws.packed_bytes, C.POINTER(C.c_uint8)), ws.packed_bytes)
    tb = (time.perf_counter() - t0) / 20
    t0 = time.perf_counter()
    n = 5
    for _ in range(n): ws.process_packed_host(a, b)
    te = (time.perf_counter() - t0) / n
    print(f"EB={EB}: call {te*1e3:.2f} ms ({EB/te:.0f}/s), python structs {tb*1e3:.3f} ms")
