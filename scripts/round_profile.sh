#!/bin/bash
# One GPU call: bench lines (f64, f32), launch list and a full ncu capture of
# one pipeline step (hemisphere3000, 16 captures) -> gpurun_out/
set -x
TAG=${1:-r01}
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}_f64.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --precision f32 --no-cpu-baseline > gpurun_out/bench_${TAG}_f32.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_f64.csv python scripts/profile_run.py --batch 16 --iters 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_" -s 8 -c 7 -o gpurun_out/full_${TAG}_f64 python scripts/profile_run.py --batch 16 --iters 2 > /dev/null 2>&1
ls -la gpurun_out
