# chunked pass pairs (L2-resident intermediate) A/B: bash tools/chunk_ab.sh
for c in c3 c4 c5; do
  for s in "FP_CHUNK_MB=0" "FP_CHUNK_MB=8" "FP_CHUNK_MB=16" "FP_CHUNK_MB=32" "FP_CHUNK_MB=48"; do
    env $s python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.readlines()[-1]); print('$c [$s]', round(d['ms_per_step'],3), round(d['roofline']['solve']['frac'],3), d['roofline']['per_pass_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
