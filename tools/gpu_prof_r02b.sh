# Round-2 late evidence: default bench at the final code and full ncu captures
# of the kernels changed late in the round (each after its command ran
# without ncu): the level-table Halton fill and the Halton-kind renders.
# The reports are summarised on the box (tools/ncu_summary.py, ncu_hot.py)
# and only the summaries come back (gpurun_out/ is capped at 64 MiB).
python bench.py > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err; echo bench rc=$?
for c in halton c5iph c5hh; do
  P="python tools/profile_fill.py --config $c"
  $P > gpurun_out/plain_$c.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ -s 1 -c 1 -o /tmp/r02b_$c $P > gpurun_out/ncu_r02b_$c.log 2>&1; echo $c rc=$?
  (python tools/ncu_summary.py /tmp/r02b_$c.ncu-rep; echo; python tools/ncu_hot.py /tmp/r02b_$c.ncu-rep 0.004 | head -12) > gpurun_out/r02b_${c}_summary.txt 2>&1
done
