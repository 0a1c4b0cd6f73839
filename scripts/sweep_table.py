"""Print the configs[4] sweep of a bench JSON line as a table (developer helper).
    python scripts/sweep_table.py gpurun_out/bench.log"""
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")][-1]
j = json.loads(l)
for p in j["sweep"]["points"]:
    st = p["stage_ms_per_capture"]
    print(f"{p['grid']:15s} {p['max_range_m']:5.1f} B={p['batch']:2d} {p['value']:9.1f}/s  {p['ms_per_capture']:.4f} ms  "
          f"bf {st['beamform']:.4f} env {st['envelope']:.4f} frac {p['envelope_frac']:.3f}")
