# cubic reciprocal: parity subset + c3/c2/c4 timing + ncu full capture of c3's strided passes (y fwd, MID, y inv)
python -m pytest tests/test_gpu_parity.py tests/test_gpu_regular_fft.py tests/test_gpu_mr.py -x -q > gpurun_out/gpu_tests2.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests2.log
for c in c3 c2 c4; do python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench2_$c.json 2>>gpurun_out/bench.err; done
python tools/one_solve.py --config c3 --repeat 1 && ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'fft_pass_kernelIdLi8ELb1' -c 3 -o gpurun_out/full_c3_r2v2 -f python tools/one_solve.py --config c3 --repeat 1 > gpurun_out/ncu_c3_r2v2.log 2>&1
tail -3 gpurun_out/ncu_c3_r2v2.log
