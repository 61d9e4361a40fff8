set -u
mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
bash tools/ncu_capture.sh r02b
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$?"
ICL_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-small > gpurun_out/final/bench2.json 2> gpurun_out/final/bench2.err; echo "bench2 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err; echo "ref rc=$?"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/final/pytest.log)"
