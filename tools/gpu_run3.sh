# Bluestein engine: new tests + mixed-radix + transform parity
python -m pytest tests/test_gpu_blue.py tests/test_gpu_mr.py -x -q > gpurun_out/gpu_tests3.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests3.log
python -m pytest tests/test_gpu_blue.py -q -x --durations=8 2>&1 | tail -12 >> gpurun_out/gpu_tests3.log
