timeout 2400 python tools/variant_sweep.py --all --reps 5 > gpurun_out/r02_variant_sweep.jsonl 2> gpurun_out/r02_variant_sweep.err; echo "rc=$? $(wc -l < gpurun_out/r02_variant_sweep.jsonl)"
