"""Summarise ncu captures (gpurun_out/) into committed profiles/ files.

    python scripts/summarize_ncu.py <round-tag> <full.ncu-rep> <launches.csv> <config-key> [...]

Writes profiles/<tag>_<config>_ncu.md (per-kernel metrics from the --set full
capture + launch-list shares) and merges the per-launch DRAM traffic of each
kernel into profiles/traffic.json (read by bench.py for `roofline.traffic`).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_bank_conflicts"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_throughput_pct"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_throughput_pct"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_pipe_pct"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved_occupancy_pct"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "smem_per_block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp_instructions"),
]


def to_bytes(v, unit):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def read_full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        k = {"kernel": d.get("Kernel Name", "?")}
        for m, name in METRICS:
            if m in d and d[m] not in ("", "n/a"):
                try:
                    if "bytes" in m and "pct" not in m and "per_second" not in m:
                        k[name] = to_bytes(d[m], u[m])
                    elif m == "gpu__time_duration.sum":
                        k[name] = float(d[m]) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1}[u[m]]
                    else:
                        k[name] = float(d[m])
                except ValueError:
                    k[name] = d[m]
        stalls = {}
        for key in d:
            if key.startswith("smsp__average_warps_issue_stalled_") and key.endswith("_per_issue_active.ratio"):
                try:
                    v = float(d[key])
                except ValueError:
                    continue
                if v >= 0.25:
                    stalls[key[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = v
        k["stalls"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
        kernels.append(k)
    return kernels


def read_launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    out = []
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            out.append((d["Kernel Name"], float(d["Metric Value"]) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(d["Metric Unit"], 1e-9)))
    return out


def short(name):
    for k in ("k_demod", "k_premf", "k_matched_filter", "k_beamform_tiles", "k_beamform_tc", "k_digit_words",
              "k_digits", "k_envelope", "k_rfft_forward"):
        if k in name:
            return k
    return name.split("(")[0][-40:]


def main():
    tag = sys.argv[1]
    items = sys.argv[2:]
    os.makedirs(PROF, exist_ok=True)
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    stage_of = {"k_demod": "demod", "k_premf": "premf", "k_matched_filter": "matched_filter",
                "k_beamform_tiles": "beamform", "k_digit_words": "beamform", "k_digits": "beamform", "k_beamform_tc": "beamform",
                "k_envelope": "envelope"}
    for i in range(0, len(items), 3):
        rep, launches, key = items[i], items[i + 1], items[i + 2]
        ks = read_full(rep)
        ls = read_launches(launches)
        md = [f"# ncu summary {tag} — {key}", "",
              f"Source: `{os.path.basename(rep)}` (ncu --set full --clock-control none) and "
              f"`{os.path.basename(launches)}` (gpu__time_duration.sum launch list; cold-cache, "
              "serialised: compare shares, not absolutes).", "", "## Launch list (one process() step)", "",
              "| kernel | grid launches | time (us) | share |", "|---|---|---|---|"]
        ours = [(short(n), t) for n, t in ls if short(n) in stage_of]
        # last complete pipeline pass (from the last k_demod on)
        starts = [i for i, (n, _) in enumerate(ours) if n == "k_demod"]
        last = ours[starts[-1]:] if starts else ours
        tot = sum(t for _, t in last)
        for n, t in last:
            md.append(f"| {n} | 1 | {t * 1e6:.1f} | {t / tot * 100:.1f}% |")
        md += ["", "## Per-kernel metrics (full capture)", ""]
        seen = {}
        for k in ks:
            name = short(k["kernel"])
            md.append(f"### {name}")
            md.append("")
            for m, lab in METRICS:
                if lab in k:
                    v = k[lab]
                    md.append(f"- {lab}: {v:.4g}" if isinstance(v, float) else f"- {lab}: {v}")
            md.append(f"- top stalls (warps per issue): " +
                      ", ".join(f"{s} {v:.2f}" for s, v in list(k['stalls'].items())[:6]))
            md.append("")
            if name in stage_of and "dram_read" in k:
                tk = f"{key}/{stage_of[name]}"
                seen.setdefault(tk, 0.0)
                seen[tk] += k.get("dram_read", 0) + k.get("dram_write", 0)
                traffic[tk] = seen[tk]
        open(os.path.join(PROF, f"{tag}_{key.replace('/', '_')}_ncu.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    print("wrote", tpath)


if __name__ == "__main__":
    main()
