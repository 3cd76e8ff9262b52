# mixed-radix engine timings (device-resident solves): bash tools/mr_time.sh
for ax in "500:1:neumann:staggered,500:1:neumann:staggered,500:1:neumann:staggered" \
          "384:1:neumann:staggered,384:1:neumann:staggered,384:1:neumann:staggered" \
          "1000:1:dirichlet:staggered,1000:1:dirichlet:staggered" \
          "3000:1:neumann:staggered,3000:1:neumann:staggered" \
          "1000:1:neumann:staggered,1000:1:neumann:staggered,1000:1:neumann:staggered"; do
  echo "$(timeout 300 python tools/time_solve.py --axes $ax --steps 5 2>&1 | tail -1)"
done
