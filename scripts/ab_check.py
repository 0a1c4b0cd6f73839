"""A/B parity check (developer diagnostic): energies of two captures of
hemisphere3000 through each library, compared bit for bit.
    python scripts/ab_check.py lib_a.so lib_b.so   (each in its own process)"""
import subprocess, sys
import numpy as np

if len(sys.argv) == 3 and sys.argv[1] == "--one":
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
    import paper_2208_10839_b200 as sn
    sn.load_library(sys.argv[2])
    cfg = sn.default_pipeline_config(sn.GridKind.hemisphere3000)
    ws = sn.Workspace(cfg, device=0, max_batch=2)
    ms = [sn.synthesize_measurement(cfg, sn.Scene([sn.Reflector(1.2 + 0.3 * i, 0.2, 0.1, 0.8)], 0.01, 5 + i), seq=i)
          for i in range(2)]
    np.save(sys.stdout.buffer, np.stack([a.energies for a in ws.process_batch(ms)]))
    sys.exit(0)
import io
outs = [np.load(io.BytesIO(subprocess.run([sys.executable, __file__, "--one", lib], check=True,
                                          capture_output=True).stdout)) for lib in sys.argv[1:]]
print("identical:", all(np.array_equal(outs[0], o) for o in outs[1:]), outs[0].shape, float(outs[0].max()))
