for ax in "513:1:neumann:regular,513:1:neumann:regular,513:1:neumann:regular" \
          "511:1:dirichlet:regular,511:1:dirichlet:regular,511:1:dirichlet:regular" \
          "4097:1:neumann:regular,4097:1:neumann:regular" \
          "1024:6.283185307179586:periodic:regular,1024:6.283185307179586:periodic:regular,513:2:neumann:regular"; do
  python tools/time_solve.py --axes $ax
  FP_NATIVE_LIB=variants/dense_r1/libfastpoisson_b200.so python tools/time_solve.py --axes $ax
done
