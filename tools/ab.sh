# A/B of tuning env knobs: bash tools/ab.sh "<configs>" "<env setting 1>" "<env setting 2>" ...
cfgs=$1; shift
for c in $cfgs; do
  for s in "$@"; do
    env $s python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$c [$s]', round(d['ms_per_step'],3), round(d['roofline']['solve']['frac'],3), d['roofline']['per_pass_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
