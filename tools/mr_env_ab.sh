# mixed-radix tile-shape knobs (env) on a few non-power-of-two grids: bash tools/mr_env_ab.sh
for s in "FP_MR_CONTIG_KB=48" "FP_MR_CONTIG_KB=24" "FP_MR_CONTIG_KB=96" "FP_MR_STRIDED_KB=36" "FP_MR_STRIDED_KB=140" "FP_MR_STRIDED_BYTES=64"; do
  echo "== $s"; env $s bash tools/mr_time.sh | cut -c1-30,88-
done
