set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py -q -x -p no:cacheprovider -k "sepconv" > gpurun_out/j14_pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/j14_pytest.log)"
grep -E "^FAILED|^E  " gpurun_out/j14_pytest.log | head -5
for r in 3 5 6 7 8 10; do echo "== r=$r"; python tools/time_variants.py sepconv --size 16384 --batch 1 --param $r --reps 10 stream_nt64_s64_v4 stream_nt64_s128_v4 stream_nt128_s64_v4 dstream_nt64_s32_v4 dstream_nt64_s64_v4 dstream_nt64_s128_v4 dstream_nt128_s64_v4 tile64p_v4 2>&1 | tail -8; done
