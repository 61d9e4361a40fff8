set -u
timeout 1200 python -m pytest tests/test_gpu_pmap.py -q -x -p no:cacheprovider > gpurun_out/j10_pmap.log 2>&1; echo "pmap rc=$? $(tail -1 gpurun_out/j10_pmap.log)"
grep -E "^FAILED|^E  " gpurun_out/j10_pmap.log | head -10
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_pmap.py > gpurun_out/j10_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j10_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/j10_pytest.log | head -20
