# mixed-radix kernel variants: bash tools/mr_ab3.sh
for ax in "500:1:neumann:staggered,500:1:neumann:staggered,500:1:neumann:staggered" \
          "384:1:neumann:staggered,384:1:neumann:staggered,384:1:neumann:staggered" \
          "1000:1:neumann:staggered,1000:1:neumann:staggered,1000:1:neumann:staggered" \
          "3000:1:neumann:staggered,3000:1:neumann:staggered"; do
  for v in main variants/mrb3 variants/mrb4; do
    for s in "FP_MR_MAXPOW2=16" "FP_MR_MAXPOW2=8"; do
      lib=""; [ $v = main ] || lib=$v/libfastpoisson_b200.so
      echo "$v $s $(FP_NATIVE_LIB=$lib env $s timeout 300 python tools/time_solve.py --axes $ax --steps 5 2>&1 | tail -1 | cut -c1-14,70-)"
    done
  done
done
