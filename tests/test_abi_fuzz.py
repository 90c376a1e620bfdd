"""Random (including hostile) conv descriptors through the planner entry points of the C-ABI --
wf_plan_fold, wf_plan_unfolded, wf_packed_filter_bytes, wf_schedule_describe -- return a status (or a
plan) and never crash. CPU only; one child process, so a crash fails the test instead of the runner."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import ctypes, random, sys
sys.path.insert(0, {root!r})
from paper_2601_11608_b200 import _abi as A
L = A.lib()
rng = random.Random(1608)
vals = [0, 1, 2, 3, 7, 8, 11, 16, 31, 64, 224, 227, 4096, -1, -7, 2**31 - 1, 2**40, -2**40]
ok = err = 0
buf = ctypes.create_string_buffer(1 << 16)
for i in range(4000):
    pick = lambda: rng.choice(vals) if rng.random() < 0.3 else rng.randint(1, 64)
    d = A.ConvDesc(*[pick() for _ in range(11)])
    plan = A.FoldPlan()
    dt = rng.choice([A.WF_BF16, A.WF_F16, A.WF_TF32, 99])
    st = L.wf_plan_fold(ctypes.byref(d), rng.choice([0, 1, 2, 8, 16, -3, 1 << 20]), rng.choice([0, 1, 2, -1, 64]),
                        dt, ctypes.byref(plan))
    if st == A.WF_OK:
        ok += 1
        L.wf_packed_filter_bytes(ctypes.byref(plan))
        L.wf_schedule_describe(ctypes.byref(d), 0, 0, dt, buf, len(buf))
    else:
        err += 1
        assert L.wf_last_error() is not None
    st2 = L.wf_plan_unfolded(ctypes.byref(d), dt, ctypes.byref(plan))
print("DONE", ok, err)
"""


def test_planner_entry_points_survive_random_descriptors():
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout[-400:], r.stderr[-800:])
    done = [ln for ln in r.stdout.splitlines() if ln.startswith("DONE")]
    assert done, r.stdout[-400:]
    _, ok, err = done[0].split()
    assert int(ok) > 0 and int(err) > 0


WIDE_CHILD = r"""
import resource, sys, time
resource.setrlimit(resource.RLIMIT_AS, (8 << 30, 8 << 30))  # a runaway search fails here instead of eating the host
sys.path.insert(0, {root!r})
import random
from paper_2601_11608_b200 import _core
# geometries the device soak (tools/fuzz_soak.py) and a 2490-geometry plan dump found: wide folded pixels
# (C = 6 / 8, fp32 4-byte elements, W stride 1 -> many groups) made the minimal-cover enumeration grow as
# 2^(window/2) (std::bad_alloc after ~200 GB) or the automatic factor search take minutes
cases = [([4, 27, 181, 8], [11, 2, 8, 32], 2, 4, 1, 0, "tf32"),
         ([381, 181, 174, 8], [11, 11, 8, 64], 2, 1, 4, 3, "tf32"),
         ([335, 74, 160, 8], [11, 11, 8, 32], 2, 1, 5, 0, "tf32"),
         ([121, 230, 175, 8], [11, 5, 8, 32], 2, 1, 0, 0, "tf32"),
         ([213, 14, 211, 6], [11, 5, 6, 16], 4, 3, 3, 1, "bf16"),
         ([75, 161, 252, 6], [1, 2, 6, 64], 3, 1, 0, 0, "f16")]
rng = random.Random(77)
for _ in range(300):
    n, h, w = rng.randint(1, 512), rng.randint(4, 240), rng.randint(4, 260)
    c, kh, kw = rng.choice([3, 4, 6, 8]), rng.choice([1, 3, 5, 7, 11]), rng.choice([1, 2, 3, 5, 7, 11])
    sh, sw = rng.randint(1, 4), rng.randint(1, 4)
    ph, pw = rng.randint(0, kh // 2), rng.randint(0, kw // 2)
    if (h + 2 * ph - kh) // sh + 1 >= 1 and (w + 2 * pw - kw) // sw + 1 >= 1:
        cases.append(([n, h, w, c], [kh, kw, c, rng.choice([16, 32, 64, 96, 128])], sh, sw, ph, pw,
                      rng.choice(["bf16", "f16", "tf32"])))
worst = 0.0
t0 = time.time()
for x, wt, sh, sw, ph, pw, dt in cases:
    t = time.time()
    try:
        _core.FoldedConv(x, wt, sh, sw, ph, pw, dt, 0, 0, "fold")
    except Exception as e:
        assert type(e).__name__ == "UnsupportedError", (x, wt, sh, sw, ph, pw, dt, repr(e))
    worst = max(worst, time.time() - t)
print("DONE", len(cases), round(worst, 3), round(time.time() - t0, 3))
"""


def test_wide_pixel_planning_is_bounded():
    """Automatic planning of wide-pixel geometries finishes quickly in bounded memory and either applies
    or reports the planner's fallback reason."""
    r = subprocess.run([sys.executable, "-c", WIDE_CHILD.format(root=ROOT)], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout[-400:], r.stderr[-800:])
    done = [ln for ln in r.stdout.splitlines() if ln.startswith("DONE")]
    assert done, r.stdout[-400:]
    _, n, worst, total = done[0].split()
    assert float(worst) < 5.0 and float(total) < 60.0, done[0]
