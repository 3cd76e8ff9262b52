python -m pytest tests/test_gpu_tma.py -q -x > gpurun_out/gpu_c5.log 2>&1; echo "exit $?" >> gpurun_out/gpu_c5.log
python -m pytest tests/test_gpu_parity.py -q -x -k "c5" >> gpurun_out/gpu_c5.log 2>&1; echo "exit c5 $?" >> gpurun_out/gpu_c5.log
b() { python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_c5.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2; do b c5_tma >> gpurun_out/ab_c5.txt; FP_TMA_CP=0 b c5_notma >> gpurun_out/ab_c5.txt; done
