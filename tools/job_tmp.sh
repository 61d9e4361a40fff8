set -u
bash tools/ncu_capture.sh r02a
ls -la gpurun_out/ncu_r02a/
