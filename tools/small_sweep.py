"""Per-call time of every variant at BASELINE.json configs[0..2] (latency-bound sizes), as a
replayed CUDA graph of 20 calls (bench.py small_configs' method).  tools/small_sweep.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

dev = torch.device("cuda:0")
st = torch.cuda.Stream(device=dev)
a = torch.from_numpy(synth.uniform_image(1, 512, 512)).to(dev)
h = torch.from_numpy(synth.rect_scene(2, 2048, 2048, noise=0.01)).to(dev)
n = torch.from_numpy(synth.rect_scene(3, 1024, 1024, noise=0.0866)).to(dev)
fx = synth.gaussian_taps(2)
oa, oh, on = torch.empty_like(a), torch.empty_like(h), torch.empty_like(n)
mk = torch.empty(2048, 2048, dtype=torch.uint8, device=dev)
calls = {
    "sepconv": lambda: icl.sepconv(a, oa, fx, fx, "constant", stream=st),
    "harris": lambda: icl.harris(h, oh, 5, 0.04, "clamp", mask=mk, threshold=1.0, stream=st),
    "nlm": lambda: icl.nlm(n, on, 2, 5, 0.1, "clamp", stream=st),
}
only = sys.argv[1:] or list(calls)
reps = 20
for f in only:
    fn = calls[f]
    res = []
    for name in icl.variant_names(f):
        if name == "naive_direct" and f == "nlm":
            continue
        icl.force_variant(f, name)
        try:
            with torch.cuda.stream(st):
                for _ in range(3):
                    fn()
            st.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for _ in range(reps):
                    fn()
        except Exception:  # noqa: BLE001 -- ineligible variant
            torch.cuda.synchronize()
            continue
        g.replay()
        torch.cuda.synchronize(dev)
        best = 1e9
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                g.replay()
            e1.record(st)
            st.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1000 / reps)
        res.append((best, name))
    icl.force_variant(f, None)
    for t, name in sorted(res)[:8]:
        print(f"{f:8s} {name:24s} {t:8.2f} us/call (graph)", flush=True)
