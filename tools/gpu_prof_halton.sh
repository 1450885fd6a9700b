timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "halton or radical or misaligned" 2>&1 | tail -2
python tools/exp_halton_runs.py QMC_HALTON_TMA=1 2>&1
P="python tools/profile_fill.py --config halton"
$P > gpurun_out/plain_halton.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_halton -s 1 -c 1 -o gpurun_out/prof_halton_tma $P > gpurun_out/ncu_halton.log 2>&1; echo halton rc=$?
