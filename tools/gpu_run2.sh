timeout 1500 python -m pytest tests -m gpu -q -rA --timeout 900 -p no:cacheprovider -s > gpurun_out/gputests2.log 2>&1; echo tests rc=$?
grep -E "passed|failed|error" gpurun_out/gputests2.log | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/bench2_ref.json 2> gpurun_out/bench2_ref.err; echo ref rc=$?
P="python tools/profile_fill.py --config c3owen"
$P > gpurun_out/plain_owen.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_sobol_fast -s 1 -c 1 -o gpurun_out/prof_c3owen $P > gpurun_out/ncu_owen.log 2>&1; echo owen rc=$?
R="python tools/profile_fill.py --config c564"
$R > gpurun_out/plain_r.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_render -s 1 -c 1 -o gpurun_out/prof_c5 $R > gpurun_out/ncu_c5.log 2>&1; echo c5 rc=$?
