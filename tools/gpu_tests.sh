timeout 1200 python -m pytest tests -m gpu -q -rA --timeout 600 -p no:cacheprovider -s > gpurun_out/gputests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|error" gpurun_out/gputests.log | tail -3
