"""ncu driver for the wire path: sn_workspace_process_frames on 16 frames (developer diagnostic)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2208_10839_b200 as sn
B = 16
cfg = sn.default_pipeline_config(2)
ws = sn.Workspace(cfg, device=0, max_batch=B)
scene = sn.Scene([sn.Reflector(1.5, 0.2, 0.0, 0.8)], 0.01, 7)
pk = sn.synthesize_measurement(cfg, scene).packed
fr = [sn.measurement_frame(sn.RawMeasurement(1, k, k, 32, ws.frames, cfg.pdm_rate, pk)) for k in range(B)]
fin = torch.empty((B, len(fr[0])), dtype=torch.uint8).pin_memory()
for k in range(B):
    fin.numpy()[k] = np.frombuffer(fr[k], np.uint8)
slot = ws.image_frame_bytes
fout = torch.empty((B, slot), dtype=torch.uint8).pin_memory()
ptrs = (C.c_void_p * B)(*[fin.numpy()[i].ctypes.data for i in range(B)])
lens = (C.c_uint64 * B)(*([len(fr[0])] * B))
olen, ost = (C.c_uint64 * B)(), (C.c_int32 * B)()
L = sn.lib()
for _ in range(2):
    rc = L.sn_workspace_process_frames(ws._h, ptrs, lens, B, fout.numpy().ctypes.data, slot, olen, ost)
    assert rc == 0 and all(ost[i] == 0 for i in range(B)), (rc, list(ost))
print("ok")
