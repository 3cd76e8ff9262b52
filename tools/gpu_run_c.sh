python -m pytest tests/test_gpu_tma.py -q -x > gpurun_out/gpu_c.log 2>&1; echo "exit $?" >> gpurun_out/gpu_c.log
python -m pytest tests/test_gpu_parity.py -q -x -k "c4_full or reduced or golden" >> gpurun_out/gpu_c.log 2>&1; echo "exit c4 $?" >> gpurun_out/gpu_c.log
b() { python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_c.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2; do b c4_tma >> gpurun_out/ab_c.txt; FP_TMA_CMID=0 b c4_nocmid >> gpurun_out/ab_c.txt; done
