"""Corrupted model files never crash the C++ readers: every mutation of a valid bundle / graph either
loads or raises one of the format's exceptions (ManifestParse / BlobSizeMismatch / IoFailure /
ShapeInferenceFailure / ValueError family). Each case runs in a child process so a segfault or an
abort is a test failure, not a dead test runner. CPU only."""
import json
import os
import random
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys
sys.path.insert(0, {root!r})
import paper_2601_11608_b200 as wf
for arg in sys.argv[1:]:
    kind, path = arg.split(":", 1)
    try:
        (wf.read_bundle if kind == "bundle" else wf.read_graph)(path)
        print("LOADED", flush=True)
    except Exception as e:  # any Python-visible error is fine; crashes are not
        print("RAISED", type(e).__name__, flush=True)
"""


def _mutations(data: bytes, rng: random.Random, count: int):
    out = []
    for _ in range(count):
        b = bytearray(data)
        op = rng.randrange(5)
        if op == 0 and len(b) > 1:      # truncate
            b = b[:rng.randrange(len(b))]
        elif op == 1:                   # flip bytes
            for _ in range(rng.randint(1, 8)):
                if b:
                    b[rng.randrange(len(b))] ^= 1 << rng.randrange(8)
        elif op == 2:                   # insert garbage
            pos = rng.randrange(len(b) + 1)
            b[pos:pos] = bytes(rng.randrange(256) for _ in range(rng.randint(1, 16)))
        elif op == 3:                   # replace a digit run with a huge / negative number
            s = b.decode("latin-1")
            digits = [i for i, ch in enumerate(s) if ch.isdigit()]
            if digits:
                i = rng.choice(digits)
                s = s[:i] + rng.choice(["999999999999", "-7", "0", "1e309"]) + s[i + 1:]
            b = bytearray(s.encode("latin-1"))
        else:                           # empty
            b = bytearray()
        out.append(bytes(b))
    return out


def _run(args):
    r = subprocess.run([sys.executable, "-c", CHILD.format(root=ROOT)] + args, capture_output=True, text=True,
                       timeout=300)
    return r.returncode, r.stdout.strip().splitlines(), r.stderr[-400:]


def test_corrupted_bundles_and_graphs_do_not_crash(tmp_path):
    """One child process reads every mutated file in turn (a crash ends it early and fails the test)."""
    import paper_2601_11608_b200 as wf
    rng = random.Random(2601)
    base = tmp_path / "base"
    base.mkdir()
    wf.write_bundle(base / "m.json", {"a": np.arange(12, dtype=np.float32).reshape(3, 4), "b": np.ones(5, np.float32)})
    g = wf.Graph()
    g.add("x", "input", shape=[1, 8, 8, 3])
    g.constant("w", np.ones((3, 3, 3, 8), np.float32))
    g.add("c", "conv2d", ["x", "w"], stride=[1, 1], groups=1)
    g.add("out", "output", ["c"])
    wf.write_graph(g, base / "g.json")
    args = []
    for k, (kind, target) in enumerate([("bundle", "m.json"), ("bundle", "m.bin"), ("graph", "g.json")]):
        data = (base / target).read_bytes()
        for i, mutated in enumerate(_mutations(data, rng, 40)):
            d = tmp_path / f"c{k}_{i}"
            d.mkdir()
            for f in base.iterdir():  # every case in its own directory: the manifest names its blob
                (d / f.name).write_bytes(f.read_bytes())
            (d / target).write_bytes(mutated)
            args.append(f"{kind}:{d / ('g.json' if kind == 'graph' else 'm.json')}")
    rc, lines, err = _run(args)
    assert rc == 0, (rc, len(lines), err)
    assert len(lines) == len(args)
    assert all(ln == "LOADED" or ln.startswith("RAISED") for ln in lines)
    assert sum(ln.startswith("RAISED") for ln in lines) > 0
