python -m pytest tests -m gpu -q -x > gpurun_out/gpu_q2.log 2>&1; echo "exit $?" >> gpurun_out/gpu_q2.log
b() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_q.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2 3; do b c3 >> gpurun_out/ab_q2.txt; done
python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_q.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('c2', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'])" >> gpurun_out/ab_q2.txt
