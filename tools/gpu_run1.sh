set -x
./tools/rcp_probe.bin > gpurun_out/rcp_probe.txt 2>&1
python -m pytest tests -m gpu -x -q -k "not c5_full_size_seeded" > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
for c in c3 c2 c4; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$c.json 2>>gpurun_out/bench.err; done
python -m pytest tests/test_gpu_parity.py -x -q -s -k "c5_full_size_seeded" > gpurun_out/c5_full.log 2>&1; echo "exit $?" >> gpurun_out/c5_full.log
