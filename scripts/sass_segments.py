"""Per-barrier-segment breakdown of an ncu source page (SASS): samples and
instructions between consecutive BAR instructions (developer diagnostic).
    python scripts/sass_segments.py rep.ncu-rep kernel_regex"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = [i for i, r in enumerate(rows) if r and r[0] == "Address"]
h = rows[hdr[0]]
end = hdr[1] if len(hdr) > 1 else len(rows)
data = [r for r in rows[hdr[0] + 1:end] if r and r[0] not in ("Address", "Kernel Name")]
iS, iN, iE = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
f = lambda x: float(x) if x not in ("", None) else 0.0
tot = sum(f(r[iN]) for r in data)
print(f"total samples {tot:.0f}, warp instructions {sum(f(r[iE]) for r in data):.4g}")
seg, cur = [], None
for k, r in enumerate(data):
    if cur is None:
        cur = {"a": k, "n": 0.0, "e": 0.0, "st": {c: 0.0 for c in stalls}, "ops": {}}
    cur["n"] += f(r[iN]); cur["e"] += f(r[iE])
    for c in stalls: cur["st"][c] += f(r[h.index(c)])
    op = r[iS].split()[0] if r[iS].split() else ""
    if op.startswith("@"): op = r[iS].split()[1]
    op = op.split(".")[0]
    cur["ops"][op] = cur["ops"].get(op, 0) + f(r[iE])
    if "BAR" in r[iS] or "EXIT" in r[iS] or k == len(data) - 1:
        cur["b"] = k; seg.append(cur); cur = None
for s in seg:
    if s["n"] / tot < 0.01: continue
    top = sorted(s["st"].items(), key=lambda x: -x[1])[:4]
    ops = sorted(s["ops"].items(), key=lambda x: -x[1])[:6]
    print(f"{s['a']:5d}-{s['b']:5d} {100*s['n']/tot:5.1f}% instr {s['e']/1e6:8.1f}M | "
          + " ".join(f"{c[6:]}={100*v/tot:.1f}" for c, v in top) + " | " + " ".join(f"{o}:{v/1e6:.0f}M" for o, v in ops))
