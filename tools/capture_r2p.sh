#!/usr/bin/env bash
# Round-2 final captures (r2p: deferred accumulation of the Leja sums on top
# of r2n). Run on the GPU box through gpurun: `bash tools/capture_r2p.sh`.
# Every profiled command first exits 0 without ncu; numbers printed under ncu
# are never bench values.
#   1. the driver-contract bench line (and the same line with per-iteration
#      accumulation, EK_LEJA_DEFER=0) and the reference arm;
#   2. ncu launch list of the bench step (cold, serialised: read the SHARES);
#   3. ncu --set full of the dominant kernel (row march, K = 0), the combine
#      pass, the 3-D plane march with and without accumulators;
#   4. kernel timings (CUDA events) for both modes, 2-D and 3-D.
set -u
out=gpurun_out/prof
mkdir -p $out
python bench.py > $out/r2p_bench.json 2> $out/r2p_bench.err
EK_LEJA_DEFER=0 python bench.py --no-e2e --no-configs --no-cpu-baseline > $out/r2p_bench_defer0.json 2> $out/r2p_bench_defer0.err
python bench.py --impl reference --steps 2 --warmup 0 > $out/r2p_reference_arm.json 2> $out/r2p_reference_arm.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline > $out/r2p_launches_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $out/r2p_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline \
    > $out/r2p_launches.log 2>&1
python tools/launch_summary.py $out/r2p_launches.csv > $out/r2p_launches.txt 2>&1
cap() {  # name, kernel regex, skip, command...
  local name=$1 regex=$2 skip=$3; shift 3
  "$@" > $out/r2p_${name}_plain.log 2>&1 || { echo "$name: plain run failed"; return; }
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$regex" -s "$skip" -c 1 -o /tmp/$name -f "$@" > $out/r2p_${name}.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $out/r2p_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_src.csv 2>/dev/null
  python tools/sass_summary.py /tmp/${name}_src.csv > $out/r2p_${name}_sass.txt 2>&1
}
cap march2d_k0 'k_march2d<.*\(int\)1, \(int\)1, \(int\)0, ' 12 python tools/kernel_bench.py --k 3 --iters 20 --reps 1 --defer 1
cap combine 'k_leja_combine' 4 python bench.py --steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline
cap leja3d_k1 'k_tma3d<.*\(int\)2, \(int\)1, \(int\)1, \(int\)5, \(int\)0>' 12 python tools/kernel_bench.py --problem advdiff3d --n 512 --k 1 --iters 20 --reps 1 --defer 0
cap leja3d_k0 'k_tma3d<.*\(int\)2, \(int\)1, \(int\)0, ' 12 python tools/kernel_bench.py --problem advdiff3d --n 512 --k 2 --iters 20 --reps 1 --defer 1
for d in 0 1; do
  for k in 1 2 3; do python tools/kernel_bench.py --k $k --iters 30 --defer $d; done
  for k in 1 2 3; do python tools/kernel_bench.py --problem advdiff3d --n 512 --k $k --iters 30 --defer $d; done
done > $out/r2p_kernels.jsonl 2>/dev/null
python tools/phi_bench.py > $out/r2p_phi_window.jsonl 2>$out/r2p_phi_window.err
ls -la $out | grep r2p | tail -30
