timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/j17.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j17.log)"; grep -E "^FAILED" gpurun_out/j17.log | head
timeout 600 python -m pytest tests/test_gpu_pmap.py -q -p no:cacheprovider -k model_guided --count 1 > /dev/null 2>&1
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_pmap.py -q -p no:cacheprovider -k model_guided 2>&1 | tail -1; done
