"""SASS evidence per kernel of the built library (tcgen05 / TMA / FP64 pipe
mnemonics and ptxas register/spill figures), written to profiles/<tag>_sass.md.
    python scripts/sass_summary.py r02"""
import collections, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_2208_10839_b200", "_lib", "libsonarnet_b200.so")
LOG = os.path.join(ROOT, "paper_2208_10839_b200", "_lib", "build.log")
OPS = ["UTCIMMA", "UTCHMMA", "LDTM", "STTM", "UBLKCP", "UBLKPF", "UTMALDG", "SYNCS", "DFMA", "DADD", "DMUL",
       "MUFU", "SHFL", "BAR", "LDS", "STS", "LDG", "STG", "LDL", "STL"]
tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
kern, counts = None, collections.OrderedDict()
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        kern = m.group(1)
        counts[kern] = collections.Counter()
        continue
    if kern is None:
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m:
        op = m.group(2)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                counts[kern][o] += 1
regs = {}
res = subprocess.run(["cuobjdump", "-res-usage", SO], capture_output=True, text=True).stdout
cur = None
for line in res.splitlines():
    m = re.match(r"\s*Function (\S+):", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", line)
    if m and cur:
        regs[cur] = {"regs": int(m.group(1)), "stack": int(m.group(2))}


def demangle(n):
    out = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    return out.replace("snb::", "")


lines = [f"# SASS summary {tag} — libsonarnet_b200.so (sm_100a)", "",
         "Static instruction counts per kernel (cuobjdump -sass) and ptxas registers / spill stores "
         "(cuobjdump -res-usage: registers, stack bytes = spill + local arrays). UTCIMMA = tcgen05.mma kind::i8, LDTM = tcgen05.ld, UBLKCP / UBLKPF = "
         "cp.async.bulk copy / L2 prefetch, SYNCS = mbarrier ops.", "",
         "| kernel | regs | stack B | " + " | ".join(OPS) + " |", "|---|---|---|" + "---|" * len(OPS)]
for k, c in counts.items():
    if not (k.startswith("_ZN3snb") and sum(c.values())):
        continue
    r = regs.get(k, {})
    lines.append(f"| `{demangle(k)}` | {r.get('regs', '')} | {r.get('stack', '')} | " +
                 " | ".join(str(c[o]) for o in OPS) + " |")
out = os.path.join(ROOT, "profiles", f"{tag}_sass.md")
open(out, "w").write("\n".join(lines) + "\n")
print(out)
