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
