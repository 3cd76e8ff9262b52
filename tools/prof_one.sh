# ncu --set full of selected pass kernels of one config:  bash tools/prof_one.sh c5 '<mangled-regex>' <count> <name>
set -x
cfg=$1; rx=$2; cnt=$3; name=$4
python tools/one_solve.py --config $cfg --repeat 1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled \
  -k regex:"$rx" -c $cnt -o gpurun_out/$name -f python tools/one_solve.py --config $cfg --repeat 1 > gpurun_out/ncu_$name.log 2>&1
tail -3 gpurun_out/ncu_$name.log
