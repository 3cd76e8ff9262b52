for ax in "500:1:neumann:staggered,500:1:neumann:staggered,500:1:neumann:staggered" \
          "384:1:dirichlet:staggered,384:1:dirichlet:staggered,384:1:dirichlet:staggered" \
          "1000:1:neumann:staggered,1000:1:neumann:staggered" \
          "3000:1:neumann:staggered,3000:1:neumann:staggered" \
          "100:1:neumann:staggered,100:1:neumann:staggered,100:1:neumann:staggered"; do
  python tools/time_solve.py --axes $ax --steps 3
  FP_NATIVE_LIB=variants/olddense/libfastpoisson_b200.so timeout 300 python tools/time_solve.py --axes $ax --steps 2
done
