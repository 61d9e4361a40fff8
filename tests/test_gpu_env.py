"""Environment switches of the library (include/icl.h "Environment"; SURVEY.md §5 auxiliaries):
ICL_LOG dispatch logging, ICL_FORCE_VARIANT process-wide forcing, ICL_TUNE_CACHE persistence
across processes (with ICL_TUNE_POLICY=require proving the second process dispatches from the
loaded cache).  Each case runs in a fresh interpreter (the variables are read once)."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROG = """
import sys, torch
sys.path.insert(0, {root!r})
import paper_1605_06399_b200 as icl, synth
x = torch.from_numpy(synth.uniform_image(3, 300, 256)).cuda()
y = torch.empty_like(x)
f = synth.gaussian_taps(2)
if {tune}:
    print("TUNED", icl.tune("sepconv", x, y, taps_x=f, taps_y=f, border="constant")["name"])
icl.sepconv(x, y, f, f, "constant")
torch.cuda.synchronize()
print("LAST", icl.variant_names("sepconv")[icl.last_variant("sepconv")])
"""


def run(env, tune=False):
    e = dict(os.environ)
    for k in ("ICL_LOG", "ICL_FORCE_VARIANT", "ICL_TUNE_CACHE", "ICL_TUNE_POLICY"):
        e.pop(k, None)
    e.update(env)
    r = subprocess.run([sys.executable, "-c", PROG.format(root=ROOT, tune=tune)], env=e, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return r


def last(r):
    return [ln.split()[1] for ln in r.stdout.splitlines() if ln.startswith("LAST")][0]


def test_icl_log_prints_the_dispatch_decision():
    r = run({"ICL_LOG": "1"})
    assert "[icl] sepconv:W256:H300" in r.stderr and last(r) in r.stderr and "(default)" in r.stderr


def test_force_variant_from_the_environment():
    assert last(run({"ICL_FORCE_VARIANT": "sepconv=naive_direct"})) == "naive_direct"
    assert last(run({"ICL_FORCE_VARIANT": "harris=naive_direct,sepconv=pm_w32x4_c2x2_blk_l1_u4"})) == \
        "pm_w32x4_c2x2_blk_l1_u4"
    r = run({"ICL_FORCE_VARIANT": "sepconv=no_such_variant"})  # reported, ignored
    assert "no variant no_such_variant" in r.stderr and last(r) != "no_such_variant"


def test_tune_cache_persists_across_processes(tmp_path):
    path = str(tmp_path / "cache.json")
    r1 = run({"ICL_TUNE_CACHE": path}, tune=True)
    won = [ln.split()[1] for ln in r1.stdout.splitlines() if ln.startswith("TUNED")][0]
    assert os.path.exists(path) and won in open(path).read()
    # a new process with ICL_TUNE_POLICY=require fails on a miss: it dispatches from the loaded cache
    r2 = run({"ICL_TUNE_CACHE": path, "ICL_TUNE_POLICY": "require", "ICL_LOG": "1"})
    assert last(r2) == won and "(tune cache)" in r2.stderr
