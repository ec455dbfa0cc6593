#!/usr/bin/env bash
# Run on the GPU box (gpurun): one `ncu --set full` capture per kernel of
# interest, exported to CSV under gpurun_out/prof/ (the .ncu-rep files stay
# in /tmp on the box; they are too large to bring back together).
#   usage: bash tools/capture_profiles.sh <tag>
set -u
tag=${1:-r1}
out=gpurun_out/prof
mkdir -p $out
cap() {  # name, kernel regex, skip, command...
  local name=$1 regex=$2 skip=$3; shift 3
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$regex" -s "$skip" -c 1 -o /tmp/$name -f "$@" > $out/${tag}_${name}.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $out/${tag}_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page details --csv > $out/${tag}_${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_src.csv 2>/dev/null
  python tools/sass_summary.py /tmp/${name}_src.csv > $out/${tag}_${name}_sass.txt 2>&1
}
# steady-state fused FD Leja iterations, config-4 geometry (k = 1 and k = 3)
cap leja2d_k1 '\(int\)1, \(int\)1, \(int\)1, \(int\)4' 12 python tools/kernel_bench.py --k 1 --iters 20 --reps 1
# 3-D TMA Leja iteration (config 5, 512^3, linear Jacobian)
cap leja3d_k1 'k_tma3d<ek::PAdvDiff3, \(int\)2, \(int\)1, \(int\)1' 12 python tools/kernel_bench.py --problem advdiff3d --n 512 --k 1 --iters 20 --reps 1
cap leja3d_k3 'k_tma3d<ek::PAdvDiff3, \(int\)2, \(int\)1, \(int\)3' 12 python tools/kernel_bench.py --problem advdiff3d --n 512 --k 3 --iters 20 --reps 1
# the bench step's dominant kernel: bulk-copy row march, k = 3 active
cap march2d_k3 'k_march2d<.*\(int\)1, \(int\)1, \(int\)3' 12 python tools/kernel_bench.py --k 3 --iters 20 --reps 1
# KIOPS Arnoldi fused pass A and the orthogonalisation pass
cap arnoldi_passA '\(int\)1, \(int\)3, \(int\)3, \(int\)4' 3 python tools/kiops_bench.py
cap arnoldi_orth 'k_arn_orth' 3 python tools/kiops_bench.py
