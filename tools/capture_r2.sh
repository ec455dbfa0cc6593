#!/usr/bin/env bash
# Round-2 captures (run on the GPU box through gpurun):
#   bash tools/capture_r2.sh
# 1. launch list of the bench step (per-launch times, cold and serialised:
#    the kernel's SHARE of the step is what must agree with bench.py);
# 2. ncu --set full of the bench's dominant kernel (row march, k = 3) and
#    of the stage-algebra pass, CSV exports under gpurun_out/prof/.
set -u
out=gpurun_out/prof
mkdir -p $out
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $out/r2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline \
    > $out/r2_launches.log 2>&1
cap() {  # name, kernel regex, skip, command...
  local name=$1 regex=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$regex" -s "$skip" -c 1 -o /tmp/$name -f "$@" > $out/r2_${name}.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $out/r2_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_src.csv 2>/dev/null
  python tools/sass_summary.py /tmp/${name}_src.csv > $out/r2_${name}_sass.txt 2>&1
}
cap march2d_k3 'k_march2d<.*\(int\)1, \(int\)1, \(int\)3' 12 python tools/kernel_bench.py --k 3 --iters 20 --reps 1
cap march2d_k1 'k_march2d<.*\(int\)1, \(int\)1, \(int\)1' 12 python tools/kernel_bench.py --k 1 --iters 20 --reps 1
cap leja3d_k1 'k_tma3d<.*\(int\)2, \(int\)1, \(int\)1' 12 python tools/kernel_bench.py --problem advdiff3d --n 512 --k 1 --iters 20 --reps 1
cap lincomb2 'k_lincomb<\(int\)2' 8 python bench.py --steps 1 --warmup 3 --no-e2e --no-configs --no-cpu-baseline
cap leja_begin 'k_leja_begin' 8 python bench.py --steps 1 --warmup 3 --no-e2e --no-configs --no-cpu-baseline
