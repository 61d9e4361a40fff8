set -u
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j5_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j5_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/j5_pytest.log | head -20
