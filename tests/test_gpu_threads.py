"""Host threads launching concurrently (the C-ABI's schedule and launch caches are shared, guarded by a
mutex + a per-thread last-hit slot; pybind releases the GIL around the launch). Each thread drives its
own plans on its own stream; every result is compared bitwise with a launch made up front."""
import threading

import pytest
import torch

import paper_2601_11608_b200 as wf

pytestmark = pytest.mark.gpu

GEOMS = [  # n, h, w, c, k, cout, stride, pad, dtype
    (2, 64, 64, 3, 7, 64, 2, 3, torch.bfloat16),
    (2, 67, 67, 3, 11, 96, 4, 0, torch.bfloat16),   # re-pitch workspace
    (2, 32, 32, 3, 3, 64, 1, 1, torch.bfloat16),
    (3, 40, 40, 3, 3, 32, 2, 1, torch.float16),
    (1, 48, 48, 3, 7, 64, 2, 3, torch.float32),     # TF32
]


def test_concurrent_host_threads_bitwise():
    jobs = []
    for i, (n, h, w, c, k, co, s, p, dt) in enumerate(GEOMS):
        g = torch.Generator(device="cuda").manual_seed(40 + i)
        x = torch.randint(-3, 4, (n, h, w, c), generator=g, device="cuda").to(dt)
        wt = torch.randint(-3, 4, (k, k, c, co), generator=g, device="cuda").to(dt)
        b = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
        conv = wf.FoldedConv2d(wt, b, x.shape, stride=s, padding=p, dtype=dt)
        ref = conv(x, out_dtype=torch.float32)
        jobs.append((conv, x, ref))
    torch.cuda.synchronize()
    errors = []

    def worker(ti):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                for it in range(25):
                    conv, x, ref = jobs[(ti + it) % len(jobs)]
                    # each thread gets its own workspace for plans that re-pitch (a shared one would race)
                    mine = conv.with_batch(x.shape[0])
                    y = mine(x, out_dtype=torch.float32)
                    stream.synchronize()
                    if not torch.equal(y, ref):
                        errors.append((ti, it))
        except Exception as e:  # surfaced below
            errors.append((ti, repr(e)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(6)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:5]
