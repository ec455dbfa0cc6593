kb() { timeout 120 python tools/kernel_bench.py "$@" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['problem'], d['n'], d['k'], d['tma_mode'], round(d['ms_per_launch'],4), round(d['GBps']))"; }
kb --k 2 --tma-mode 1; kb --k 2 --tma-mode 2
for m in 1 2 3; do echo "mode $m"; EK_TMA_MODE=$m timeout 300 python bench.py --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['roofline']['share_of_step'])"; done
