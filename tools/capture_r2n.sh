#!/usr/bin/env bash
# Round-2 captures after the 3-D plane-loop rework (r2n) (run on the GPU box through
# gpurun: `bash tools/capture_r2n.sh`). Every profiled command first exits 0
# without ncu; numbers printed under ncu are never bench values.
#   1. the driver-contract bench line and the reference arm;
#   2. ncu launch list of the bench step (cold, serialised: read the SHARES);
#   3. ncu --set full of the dominant kernel (row march, k = 3), its
#      repro-mode instance (integer accumulators) and the 3-D plane march;
#   4. repro-mode kernel overhead and graph-loop A/B (CUDA events).
set -u
out=gpurun_out/prof
mkdir -p $out
python bench.py > $out/r2n_bench.json 2> $out/r2n_bench.err
python bench.py --impl reference --steps 2 --warmup 0 > $out/r2n_reference_arm.json 2> $out/r2n_reference_arm.err
python bench.py --steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline > $out/r2n_launches_plain.log 2>&1 || exit 1
# the Leja iterations run inside CUDA graphs (device-side WHILE loop):
# --graph-profiling node lists their kernel nodes; the second list is the
# same step with the graph loop off (EK_LEJA_GRAPH=0: launch batches)
ncu --metrics gpu__time_duration.sum --clock-control none --graph-profiling node -c 600 --csv \
    --log-file $out/r2n_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline \
    > $out/r2n_launches.log 2>&1
python tools/launch_summary.py $out/r2n_launches.csv > $out/r2n_launches.txt 2>&1
EK_LEJA_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $out/r2n_launches_nograph.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline \
    > $out/r2n_launches_nograph.log 2>&1
python tools/launch_summary.py $out/r2n_launches_nograph.csv > $out/r2n_launches_nograph.txt 2>&1
cap() {  # name, kernel regex, skip, command...
  local name=$1 regex=$2 skip=$3; shift 3
  export EK_LEJA_GRAPH=0  # the same kernels as plain launches (ncu -k / -s count launches)
  "$@" > $out/r2n_${name}_plain.log 2>&1 || { echo "$name: plain run failed"; return; }
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
      -k "regex:$regex" -s "$skip" -c 1 -o /tmp/$name -f "$@" > $out/r2n_${name}.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > $out/r2n_${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_src.csv 2>/dev/null
  python tools/sass_summary.py /tmp/${name}_src.csv > $out/r2n_${name}_sass.txt 2>&1
  unset EK_LEJA_GRAPH
}
cap march2d_k3 'k_march2d<.*\(int\)1, \(int\)1, \(int\)3, \(int\)5, \(int\)0>' 12 python tools/kernel_bench.py --k 3 --iters 20 --reps 1
cap leja3d_k1 'k_tma3d<.*\(int\)2, \(int\)1, \(int\)1, \(int\)5, \(int\)0>' 12 python tools/kernel_bench.py --problem advdiff3d --n 512 --k 1 --iters 20 --reps 1
for r in "" "--repro"; do
  for k in 1 2 3; do python tools/kernel_bench.py --k $k --iters 30 $r; done
  for k in 1 2; do python tools/kernel_bench.py --problem advdiff3d --n 512 --k $k --iters 30 $r; done
done > $out/r2n_repro_overhead.jsonl 2>/dev/null
python tools/idle_profile.py 10 > $out/r2n_idle.txt 2>&1
for k in 1 2 3; do python tools/kernel_bench.py --problem advdiff3d --n 512 --k $k --iters 20; done > $out/r2n_leja3d_kernel.jsonl 2>/dev/null
python tools/phi_bench.py > $out/r2n_phi_window.jsonl 2>$out/r2n_phi_window.err
ls -la $out | tail -30
