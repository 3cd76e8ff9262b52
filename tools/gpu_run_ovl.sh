python -m pytest tests/test_gpu_tma.py tests/test_gpu_parity.py -q -x -k "tma or config_full_size or golden" > gpurun_out/gpu_ovl.log 2>&1; echo "exit $?" >> gpurun_out/gpu_ovl.log
b() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_ovl.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2; do
FP_OVERLAP=1 b seq >> gpurun_out/ab_ovl.txt
FP_OVERLAP=2 b ovl2 >> gpurun_out/ab_ovl.txt
FP_OVERLAP=4 b ovl4 >> gpurun_out/ab_ovl.txt
FP_OVERLAP=8 b ovl8 >> gpurun_out/ab_ovl.txt
done
