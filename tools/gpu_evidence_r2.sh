# round-2 evidence: GPU tests + smoke, bench lines (c3 default with cpu_baseline/e2e; c1 c2 c4 c5 with
# cpu baselines), the reference arm, ncu launch list and a full capture of c3's passes.
#   bash tools/gpu_evidence_r2.sh <tag>
tag=${1:-v3}
out=gpurun_out/ev_$tag; mkdir -p $out
python -m pytest tests -m gpu -q -x > $out/gpu_tests.log 2>&1; echo "exit $?" >> $out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.log 2>&1; echo "exit $?" >> $out/smoke.log
python bench.py > $out/bench_c3_default.json 2> $out/bench_c3_default.err
for c in c1 c2 c4; do python bench.py --config $c > $out/bench_$c.json 2>> $out/bench.err; done
python bench.py --config c5 --no-e2e > $out/bench_c5.json 2>> $out/bench.err   # (e2e: 2 x 34 GB pinned + device buffers)
python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref_c3.json 2>> $out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/launches_c3.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:'fft_pass' \
    -c 5 -o $out/full_c3 -f python tools/one_solve.py --config c3 --repeat 1 > $out/ncu_full_c3.log 2>&1
ls -la $out
