# Round-2 final evidence at the final code: GPU tests + smoke, default bench
# (ours + reference arm), the headline's ncu launch list, and full captures of
# the late-changed kernels summarised on the box (gpurun_out/ is capped).
bash tools/gpu_tests.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke rc=$?
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench rc=$?
python bench.py --impl reference > gpurun_out/bench_ref_final.json 2> gpurun_out/bench_ref_final.err; echo ref rc=$?
B="python bench.py --steps 5 --warmup 3 --no-extra --no-cpu --no-e2e"
$B > gpurun_out/plain_headline.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch_final.log 2>&1; echo launches rc=$?
for c in halton integrate; do
  P="python tools/profile_fill.py --config $c"
  $P > gpurun_out/plain_$c.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 1 -c 1 -o /tmp/fin_$c $P > gpurun_out/ncu_fin_$c.log 2>&1; echo $c rc=$?
  (python tools/ncu_summary.py /tmp/fin_$c.ncu-rep; echo; python tools/ncu_hot.py /tmp/fin_$c.ncu-rep 0.004 | head -12) > gpurun_out/fin_${c}_summary.txt 2>&1
done
