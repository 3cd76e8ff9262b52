# A/B of variant libraries: bash tools/ab_lib.sh "<configs>" <lib dir or "main"> ...
cfgs=$1; shift
for c in $cfgs; do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=""; else lib="$v/libfastpoisson_b200.so"; fi
    FP_NATIVE_LIB=$lib python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$c [$v]', round(d['ms_per_step'],3), round(d['roofline']['solve']['frac'],3), d['roofline']['per_pass_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
