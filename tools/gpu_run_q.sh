python -m pytest tests/test_gpu_tma.py tests/test_gpu_guard.py -q -x > gpurun_out/gpu_q.log 2>&1; echo "exit $?" >> gpurun_out/gpu_q.log
b() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_q.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2 3; do b main >> gpurun_out/ab_q.txt; done
