#!/bin/bash
# Build the NCCL symmetric-window probe against the NCCL >= 2.28 torch ships; run it on a GPU box.
D=$(python -c "import importlib.util,os; s=importlib.util.find_spec('nvidia'); print([os.path.join(p,'nccl') for p in s.submodule_search_locations][0])")
cd "$(dirname "$0")" && nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I "$D/include" probe.cu -o probe \
  -L "$D/lib" -l:libnccl.so.2 -Xlinker -rpath="$D/lib"
