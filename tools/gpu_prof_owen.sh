P="python tools/profile_fill.py --config c3owen"
$P > gpurun_out/plain_owen.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on --replay-mode application -k regex:k_sobol_fast -s 1 -c 1 -o gpurun_out/prof_c3owen2 $P > gpurun_out/ncu_owen2.log 2>&1; echo owen rc=$?
