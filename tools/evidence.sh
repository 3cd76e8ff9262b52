# Round evidence: bench lines, ncu launch list, ncu --set full of each config's pass kernels.
#   bash tools/evidence.sh <tag>
tag=${1:-v9}
out=gpurun_out/ev_$tag; mkdir -p $out
python bench.py > $out/bench_c3_default.json 2> $out/bench_c3_default.err || exit 1
for c in c1 c2 c4; do python bench.py --config $c --no-cpu-baseline > $out/bench_$c.json 2>> $out/bench.err; done
python bench.py --config c5 --no-cpu-baseline --no-e2e > $out/bench_c5.json 2>> $out/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $out/bench_ref.json 2>> $out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1
cp profiles/ncu_traffic.json $out/ncu_traffic.json
for c in c3 c2 c4 c5; do
  ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'fft_pass|dense_pass' \
      -c 8 -o $out/full_$c -f python tools/one_solve.py --config $c --repeat 1 > $out/ncu_full_$c.log 2>&1
  python profiles/summarize_ncu.py $out/full_$c.ncu-rep $c $out/ncu_full_$c.md $out/ncu_traffic.json > /dev/null
  ncu -i $out/full_$c.ncu-rep --page raw --csv > $out/ncu_full_${c}_raw.csv 2>/dev/null
  [ $c = c3 ] || rm -f $out/full_$c.ncu-rep   # (gpurun returns at most 64 MiB)
done
ls -la $out
