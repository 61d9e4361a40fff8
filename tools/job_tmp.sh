set -u
bash tools/sanitize.sh
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j15_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j15_pytest.log)"
grep -E "^FAILED|^ERROR" gpurun_out/j15_pytest.log | head -20
