set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider -k "sepconv" > gpurun_out/j23.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j23.log)"; grep -E "^FAILED|^E  " gpurun_out/j23.log | head -5
for r in 7 8 9 10 12 15; do echo "== r=$r"; python tools/time_variants.py sepconv --size 16384 --batch 1 --param $r --reps 10 stream_nt64_s128_v4 tile64p_v4 tile128p_v4 2>&1 | tail -3; done
