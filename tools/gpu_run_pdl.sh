python -m pytest tests -m gpu -q -x > gpurun_out/gpu_pdl.log 2>&1; echo "exit $?" >> gpurun_out/gpu_pdl.log
b() { python bench.py --config $2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_pdl.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1 $2', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2; do for c in c1 c3 c2; do b pdl $c >> gpurun_out/ab_pdl.txt; FP_PDL=0 b nopdl $c >> gpurun_out/ab_pdl.txt; done; done
