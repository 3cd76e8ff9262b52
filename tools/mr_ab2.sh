# mixed-radix tile shape A/B (lines per CTA): bash tools/mr_ab2.sh
for ax in "500:1:neumann:staggered,500:1:neumann:staggered,500:1:neumann:staggered" \
          "384:1:neumann:staggered,384:1:neumann:staggered,384:1:neumann:staggered" \
          "3000:1:neumann:staggered,3000:1:neumann:staggered" \
          "1000:1:neumann:staggered,1000:1:neumann:staggered,1000:1:neumann:staggered"; do
  for s in "FP_MR_STRIDED_BYTES=16" "FP_MR_STRIDED_BYTES=64" "FP_MR_STRIDED_BYTES=128" "FP_MR_STRIDED_BYTES=128 FP_MR_CONTIG_KB=24" "FP_MR_STRIDED_BYTES=128 FP_MR_CONTIG_KB=96"; do
    echo "$s $(env $s timeout 300 python tools/time_solve.py --axes $ax --steps 5 2>&1 | tail -1)"
  done
done
