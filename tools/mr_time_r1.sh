# regular-grid (DCT-I / DST-I) mixed-radix timings: bash tools/mr_time_r1.sh
for ax in "501:1:neumann:regular,501:1:neumann:regular,501:1:neumann:regular" \
          "499:1:dirichlet:regular,499:1:dirichlet:regular,499:1:dirichlet:regular" \
          "3001:1:neumann:regular,3001:1:neumann:regular"; do
  for h in 0 1; do echo "FP_MR_HALF=$h $(FP_MR_HALF=$h timeout 300 python tools/time_solve.py --axes $ax --steps 5 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d[\"axes\"][:24], d[\"ms\"])")"; done
done
