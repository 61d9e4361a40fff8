"""Two-rank native sharded sepconv/Harris/conv2d (icl_*_sharded over NCCL) vs the unsharded call.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/comm_2rank.py [--same-gpu]

With --same-gpu both ranks use cuda:0 (whether NCCL accepts two ranks on one device is printed)."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_1605_06399_b200 as icl  # noqa: E402
import synth  # noqa: E402

rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
same = "--same-gpu" in sys.argv
dev = torch.device("cuda", 0 if same else int(os.environ.get("LOCAL_RANK", rank)))
torch.cuda.set_device(dev)
dist.init_process_group("gloo")
try:
    comm = icl.Comm(ws, rank)
except icl.IclError as e:
    print(f"rank {rank}: icl_comm_init failed: {e}", flush=True)
    sys.exit(3)
ok = True
H, W = 523, 384
img = synth.uniform_image(81, H, W)
fx = synth.gaussian_taps(4)
full = torch.from_numpy(img).to(dev)
ref = torch.empty_like(full)
icl.sepconv(full, ref, fx, fx, "clamp")
up, down = icl.halo_rows_of("sepconv", 4)
r0, r1, s0, s1 = comm.band(H, up, down)
buf = torch.full((s1 - s0, W), float("nan"), device=dev)
buf[r0 - s0:r1 - s0] = full[r0:r1]  # own rows only; halos come from the neighbour
out = torch.empty(r1 - r0, W, device=dev)
comm.sepconv(buf, out, H, fx, fx, "clamp")
torch.cuda.synchronize()
ok &= bool(np.array_equal(out.cpu().numpy(), ref[r0:r1].cpu().numpy()))
u8 = torch.from_numpy(synth.uniform_u8(82, H, W)).to(dev)
f2 = synth.filter2d(82, 3)
ref2 = torch.empty(H, W, device=dev)
icl.conv2d_u8(u8, ref2, f2, "constant", 3.0)
r0, r1, s0, s1 = comm.band(H, 3, 3)
b2 = torch.zeros(s1 - s0, W, dtype=torch.uint8, device=dev)
b2[r0 - s0:r1 - s0] = u8[r0:r1]
o2 = torch.empty(r1 - r0, W, device=dev)
comm.conv2d_u8(b2, o2, H, f2, "constant", 3.0)
torch.cuda.synchronize()
ok &= bool(np.array_equal(o2.cpu().numpy(), ref2[r0:r1].cpu().numpy()))
print(f"rank {rank}: native sharded {'OK' if ok else 'MISMATCH'} rows [{r0},{r1})", flush=True)
comm.close()
dist.destroy_process_group()
sys.exit(0 if ok else 1)
