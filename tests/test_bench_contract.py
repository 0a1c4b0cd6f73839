"""bench.py contract pieces that run without a GPU: the FLOP model matches
SURVEY.md §8(d) and the reference arm prints one well-formed JSON line."""
import json
import os
import subprocess
import sys

from conftest import ROOT

sys.path.insert(0, ROOT)


def test_flop_model_matches_survey(sn):
    import bench
    d = sn.default_pipeline_config(sn.GridKind.hemisphere3000).dims()
    fe, per_dir = bench.flops_per_energyscape(d)
    assert round(fe / 1e6, 3) == 284.258          # 284.258 MFLOP
    assert round(per_dir / 1e6, 6) == 1.385930    # 1.385930 MFLOP per direction
    kf = bench.kernel_flops(d)
    assert abs(sum(kf.values()) / 1e6 - 4442.05) < 0.01  # hemi3000 4,442.1 MFLOP


def test_reference_arm_json_line(ref):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--grid", "horizontal90"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
