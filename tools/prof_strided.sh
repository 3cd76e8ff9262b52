set -x
export FP_SPIPE=0
python tools/one_solve.py --config c5 --repeat 1 || exit 1
python tools/one_solve.py --config c4 --repeat 1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:'_ZN3fpb15fft_pass_kernelIfLi11ELb1ELi[02]E' -c 2 -o gpurun_out/c5_strided -f python tools/one_solve.py --config c5 --repeat 1 > gpurun_out/ncu_c5.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:'_ZN3fpb15fft_pass_kernelIdLi(10|9)ELb1ELi[012]E' -c 3 -o gpurun_out/c4_strided -f python tools/one_solve.py --config c4 --repeat 1 > gpurun_out/ncu_c4.log 2>&1
ls -la gpurun_out
