set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j2_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j2_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/j2_pytest.log | head -20
