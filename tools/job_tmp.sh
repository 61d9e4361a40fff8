mkdir -p gpurun_out/j26
ncu --set full --clock-control none --import-source on -k regex:harris_slide -s 3 -c 1 -o gpurun_out/j26/s2 python tools/time_variants.py harris --batch 8 --reps 2 slide2_nw2_s32 > gpurun_out/j26/s2.log 2>&1; echo rc=$?
