python -m pytest tests/test_gpu_tma.py -q -x > gpurun_out/gpu_tma2.log 2>&1; echo "exit main $?" >> gpurun_out/gpu_tma2.log
FP_TMA_MID=2 FP_TMA_INV=2 FP_NATIVE_LIB=abvar/minb3/libfastpoisson_b200.so python -m pytest tests/test_gpu_tma.py -q -x >> gpurun_out/gpu_tma2.log 2>&1; echo "exit minb3 $?" >> gpurun_out/gpu_tma2.log
b() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>>gpurun_out/bench_tma.err | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$1', round(d['ms_per_step'],4), d['roofline']['per_pass_ms'], round(d['roofline']['solve']['frac'],3))"; }
for rep in 1 2; do
b main >> gpurun_out/ab_tma2.txt
FP_TMA_MID=2 b main_mid2 >> gpurun_out/ab_tma2.txt
FP_TMA_MID=2 FP_TMA_INV=2 FP_NATIVE_LIB=abvar/minb3/libfastpoisson_b200.so b minb3_mid2_inv2 >> gpurun_out/ab_tma2.txt
FP_TMA_MID=2 FP_NATIVE_LIB=abvar/minb3/libfastpoisson_b200.so b minb3_mid2 >> gpurun_out/ab_tma2.txt
FP_TMA_INV=2 FP_NATIVE_LIB=abvar/minb3/libfastpoisson_b200.so b minb3_inv2 >> gpurun_out/ab_tma2.txt
done
