python -m pytest tests/test_gpu_tma.py tests/test_gpu_guard.py -q -x > gpurun_out/gpu_z.log 2>&1; echo "exit $?" >> gpurun_out/gpu_z.log
python -m pytest tests/test_gpu_parity.py -q -x -k "config_full_size or golden" >> gpurun_out/gpu_z.log 2>&1; echo "exit full $?" >> gpurun_out/gpu_z.log
b() { python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_z.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2; do b z_tma >> gpurun_out/ab_z.txt; FP_TMA_Z=0 b z_regular >> gpurun_out/ab_z.txt; done
