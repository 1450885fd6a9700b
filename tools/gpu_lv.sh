# k_halton_lv A/B, Halton parity subset and an ncu capture of the level-table fill
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/exp_halton_lv.py 2>&1 | tee gpurun_out/lv_ab.log
P="python tools/profile_fill.py --config halton"
$P > gpurun_out/plain_halton.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_halton_lv -s 1 -c 1 -o gpurun_out/prof_halton_lv $P > gpurun_out/ncu_halton.log 2>&1; echo ncu rc=$?
[ -n "$LVTEST" ] && timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "halton" 2>&1 | tail -3
