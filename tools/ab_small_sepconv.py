"""A/B of sepconv variants at 512^2 r=2 (BASELINE configs[0]) as replayed 20-call CUDA graphs, interleaved rounds.
    tools/ab_small_sepconv.py variant..."""
import sys, statistics
import torch
sys.path.insert(0, ".")
import os
import paper_1605_06399_b200 as icl
if os.environ.get("ICL_LIB"):  # an alternative build of the library (A/B of two builds)
    icl.load_library(os.environ["ICL_LIB"])
import synth
dev = torch.device("cuda:0"); st = torch.cuda.Stream(device=dev)
a = torch.from_numpy(synth.uniform_image(1, 512, 512)).to(dev); oa = torch.empty_like(a)
fx = synth.gaussian_taps(2)
def fn(): icl.sepconv(a, oa, fx, fx, "constant", stream=st)
res = {}
for rnd in range(6):
    for name in sys.argv[1:]:
        icl.force_variant("sepconv", name)
        with torch.cuda.stream(st):
            for _ in range(3): fn()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(20): fn()
        g.replay(); torch.cuda.synchronize()
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st): g.replay()
            e1.record(st); st.synchronize()
            res.setdefault(name, []).append(e0.elapsed_time(e1) * 1000 / 20)
for n, v in res.items(): print(f"{n:28s} median {statistics.median(v):.3f} us  min {min(v):.3f}")
