"""Hostile graphs through the host graph layer -- shape inference and the width-fold pass -- raise the
graph's errors (ShapeInferenceFailure, MissingInput, ValueError family) and never crash. CPU only
(interpret runs on the device and is covered by tests/test_graph_pass.py); one child process."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import random, sys
sys.path.insert(0, {root!r})
import numpy as np
import paper_2601_11608_b200 as wf
rng = random.Random(42)
ops = ["input", "output", "constant", "conv2d", "matmul", "bias_add", "reshape", "folded_conv2d", "bogus"]
weird = [0, 1, 2, 3, 7, -1, -5, 2**31, 10**12]
outcome = {{"ok": 0, "raised": 0}}
for i in range(600):
    g = wf.Graph()
    ids = []
    for j in range(rng.randint(1, 7)):
        op = rng.choice(ops)
        nid = f"n{{j}}"
        ins = [rng.choice(ids) if ids and rng.random() < 0.8 else "missing" for _ in range(rng.randint(0, 3))]
        attrs = {{}}
        if op == "input":
            attrs["shape"] = [rng.choice(weird) if rng.random() < 0.2 else rng.randint(1, 9) for _ in range(rng.randint(0, 5))]
        if op in ("conv2d", "folded_conv2d"):
            attrs["stride"] = [rng.choice(weird), rng.choice(weird)] if rng.random() < 0.3 else [1, 1]
            attrs["groups"] = rng.choice(weird) if rng.random() < 0.3 else 1
        if op == "reshape":
            attrs["shape"] = [rng.choice(weird) for _ in range(rng.randint(0, 4))]
        if op == "constant":
            shp = [rng.randint(1, 4) for _ in range(rng.randint(1, 4))]
            g.constant(nid, np.ones(shp, np.float32))
            ids.append(nid)
            continue
        g.add(nid, op, ins, **attrs)
        ids.append(nid)
    try:
        g.infer_shapes()
        wf.width_fold_pass(g, factor=rng.choice([None, 1, 2, 4, 8, 0, -2]))
        outcome["ok"] += 1
    except Exception as e:
        outcome["raised"] += 1
print("DONE", outcome["ok"], outcome["raised"], flush=True)
"""


def test_hostile_graphs_do_not_crash():
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.returncode, r.stdout[-400:], r.stderr[-800:])
    done = [ln for ln in r.stdout.splitlines() if ln.startswith("DONE")]
    assert done, (r.stdout[-400:], r.stderr[-800:])
    _, ok, raised = done[0].split()
    assert int(ok) + int(raised) == 600 and int(raised) > 0
