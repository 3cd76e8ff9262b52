python -m pytest tests/test_gpu_tma.py -q -x > gpurun_out/gpu_tma.log 2>&1; echo "exit $?" >> gpurun_out/gpu_tma.log
FP_TMA_FWD=1 python -m pytest tests/test_gpu_tma.py -q -x >> gpurun_out/gpu_tma.log 2>&1; echo "exit fwd1 $?" >> gpurun_out/gpu_tma.log
for v in 2 1; do FP_TMA_FWD=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_tma_fwd$v.json 2>>gpurun_out/bench_tma.err; done
FP_TMA=0 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_notma.json 2>>gpurun_out/bench_tma.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_tma_fwd2b.json 2>>gpurun_out/bench_tma.err
