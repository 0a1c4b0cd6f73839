#!/bin/bash
# run the short bench for each A/B library: scripts/ab_run.sh name1 name2 ...
for n in "$@"; do
  timeout 300 python bench.py --lib paper_2208_10839_b200/_lib/ab/lib${n%%:*}.so $([[ $n == *:* ]] && echo --tc-tile-n ${n##*:}) --steps 20 --warmup 3 --no-cpu-baseline --latency-samples 5 --no-sweep --stream-frames 0 --cpu-latency-calls 0 > gpurun_out/ab_${n/:/_}.log 2>&1
  python - "$n" <<'PY'
import json,sys
n=sys.argv[1]
l=[x for x in open(f"gpurun_out/ab_{n.replace(':','_')}.log") if x.startswith("{")]
if not l: print(n,"FAILED", open(f"gpurun_out/ab_{n}.log").read()[-800:]); sys.exit()
j=json.loads(l[-1]); k=j["roofline"]["kernels"]
print(f"{n:12s} {j['value']:8.1f}/s e2e {j['e2e']['value']:8.1f} ", " ".join(f"{a}={b['ms']:.3f}" for a,b in k.items()))
PY
done
