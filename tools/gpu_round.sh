#!/bin/bash
# One gpurun job: GPU tests, smoke, the default bench line, the ncu
# launch list + one --set full capture per hot kernel.   tools/gpu_round.sh <tag>
set -u
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu_$TAG.log)"
grep -E "^FAILED" gpurun_out/pytest_gpu_$TAG.log | head -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; tail -1 gpurun_out/bench_$TAG.json | cut -c1-400
bash tools/ncu_capture.sh $TAG
