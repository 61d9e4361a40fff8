timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j25.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j25.log)"; grep -E "^FAILED" gpurun_out/j25.log | head
