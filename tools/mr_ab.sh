# dense engine vs mixed-radix engine on non-power-of-two grids (device-resident solves)
for ax in "500:1:neumann:staggered,500:1:neumann:staggered,500:1:neumann:staggered" \
          "384:1:neumann:staggered,384:1:neumann:staggered,384:1:neumann:staggered" \
          "100:1:neumann:staggered,100:1:neumann:staggered,100:1:neumann:staggered" \
          "1000:1:dirichlet:staggered,1000:1:dirichlet:staggered" \
          "3000:1:neumann:staggered,3000:1:neumann:staggered" \
          "768:6.283185307179586:periodic:staggered,768:6.283185307179586:periodic:staggered,384:2:neumann:staggered" \
          "513:1:neumann:regular,513:1:neumann:regular,513:1:neumann:regular" \
          "1000:1:neumann:staggered,1000:1:neumann:staggered,1000:1:neumann:staggered"; do
  for mr in 0 1; do
    echo "FP_MR=$mr $(FP_MR=$mr timeout 300 python tools/time_solve.py --axes $ax --steps 5 2>&1 | tail -1)"
  done
done
