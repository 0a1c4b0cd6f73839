#!/bin/bash
# Developer A/B builds: scripts/ab_build.sh NAME "-DMACRO=..." -> paper_2208_10839_b200/_lib/ab/libNAME.so
# (same sources and flags as paper_2208_10839_b200/build.py plus the extra defines;
#  select at run time with bench.py --lib ...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
C=$ROOT/paper_2208_10839_b200/csrc
O=$ROOT/paper_2208_10839_b200/_lib/ab/$1
mkdir -p $O
ARCH="-gencode arch=compute_100a,code=sm_100a"
for f in plan cluster pool gather; do g++ -O2 -std=c++17 -fPIC -ffp-contract=off -I $ROOT/include -I $C -I /usr/local/cuda/include -c $C/$f.cpp -o $O/$f.o; done
pids=()
for f in kernels beamform_tc frames synth sn_api; do
  nvcc $ARCH -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off $2 -I $ROOT/include -I $C -c $C/$f.cu -o $O/$f.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "ab_build: compile failed" >&2; exit 1; }; done
nvcc $ARCH -shared -o $ROOT/paper_2208_10839_b200/_lib/ab/lib$1.so $O/*.o -lpthread -ldl
echo built lib$1.so
