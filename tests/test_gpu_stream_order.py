"""Stream order under programmatic dependent launch (PDL).

The conv kernel is launched with programmatic stream serialization: its
prologue may run while the previous kernel on the stream is still executing,
and every global access waits on griddepcontrol.wait. These tests hammer the
hazards that ordering must cover, comparing every result bitwise with a
launch made in isolation (synchronised before and after):
  - RAW on x: a torch kernel writes x, the conv reads it right after;
  - WAR on x: the conv reads x, the next torch kernel overwrites it;
  - WAW on y: consecutive convs write the same output buffer;
  - RAW on y: a torch kernel reads y right after the conv wrote it;
  - the re-pitch workspace (AlexNet W=227): re-pitch -> conv -> re-pitch ...
"""
import pytest
import torch

import paper_2601_11608_b200 as wf

pytestmark = pytest.mark.gpu


def _isolated(conv, x):
    torch.cuda.synchronize()
    y = conv(x.clone())
    torch.cuda.synchronize()
    return y.clone()


@pytest.mark.parametrize("geom", [
    # n, h, w, c, k, cout, stride, pad, dtype
    (2, 224, 224, 3, 7, 64, 2, 3, torch.bfloat16),    # R50 conv1
    (1, 224, 224, 3, 7, 64, 2, 3, torch.float32),     # R50 conv1 b1 TF32 (config 1)
    (3, 227, 227, 3, 11, 96, 4, 0, torch.bfloat16),   # AlexNet (re-pitch workspace, 2-CTA cluster)
])
def test_back_to_back_launches_keep_stream_order(geom):
    n, h, w, c, k, co, s, p, dt = geom
    g = torch.Generator(device="cuda").manual_seed(77)
    xs = [((torch.rand((n, h, w, c), generator=g, device="cuda") * 2 - 1)).to(dt) for _ in range(6)]
    wt = ((torch.rand((k, k, c, co), generator=g, device="cuda") * 2 - 1) / (k * k * c) ** 0.5).to(dt)
    b = torch.rand(co, generator=g, device="cuda") * 2 - 1
    conv = wf.FoldedConv2d(wt, b, xs[0].shape, stride=s, padding=p, dtype=dt)
    refs = [_isolated(conv, x) for x in xs]

    x = torch.empty_like(xs[0])
    y = conv(xs[0])
    sums = torch.empty(len(xs), dtype=torch.float64, device="cuda")
    outs = []
    torch.cuda.synchronize()
    for rep in range(3):
        for i, xi in enumerate(xs):
            x.copy_(xi)                    # RAW on x (torch kernel -> conv), WAR vs the previous conv
            conv(x, out=y)                 # WAW on y (previous conv wrote it too)
            sums[i] = y.double().sum()     # RAW on y (conv -> torch kernel)
            if rep == 2:
                outs.append(y.clone())
        torch.cuda.synchronize()
        for i, r in enumerate(refs):
            assert sums[i].item() == r.double().sum().item(), f"rep {rep} input {i}: checksum differs"
    for i, (o, r) in enumerate(zip(outs, refs)):
        assert torch.equal(o, r), f"input {i}: back-to-back result differs from the isolated launch"


def test_consecutive_convs_into_distinct_outputs():
    """Conv after conv with no torch kernel in between (PDL chain of our own launches)."""
    dt = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(5)
    xs = [(torch.rand((4, 224, 224, 3), generator=g, device="cuda") * 2 - 1).to(dt) for _ in range(8)]
    wt = ((torch.rand((7, 7, 3, 64), generator=g, device="cuda") * 2 - 1) / 12).to(dt)
    b = torch.rand(64, generator=g, device="cuda") * 2 - 1
    conv = wf.FoldedConv2d(wt, b, xs[0].shape, stride=2, padding=3, dtype=dt)
    refs = [_isolated(conv, x) for x in xs]
    ys = [torch.empty_like(refs[0]) for _ in xs]
    torch.cuda.synchronize()
    for x, y in zip(xs, ys):
        conv(x, out=y)
    torch.cuda.synchronize()
    for i, (y, r) in enumerate(zip(ys, refs)):
        assert torch.equal(y, r), f"launch {i} differs"


def test_repack_then_forward_sees_the_new_filter():
    """The producer loads the packed filter (B) before griddepcontrol.wait; the launch right after a pack
    (or bias replication) therefore goes without the PDL attribute. Repack different weights into the SAME
    buffers between back-to-back launches and check each launch used the filter packed just before it."""
    dt = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(11)
    x = (torch.rand((2, 224, 224, 3), generator=g, device="cuda") * 2 - 1).to(dt)
    ws = [((torch.rand((7, 7, 3, 64), generator=g, device="cuda") * 2 - 1) / 12).to(dt) for _ in range(2)]
    bs = [torch.rand(64, generator=g, device="cuda") * 2 - 1 for _ in range(2)]
    refs = [_isolated(wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=dt), x) for w, b in zip(ws, bs)]
    conv = wf.FoldedConv2d(ws[0], bs[0], x.shape, stride=2, padding=3, dtype=dt)
    y = conv(x)
    st = torch.cuda.current_stream().cuda_stream
    outs = []
    torch.cuda.synchronize()
    for i in range(12):
        k = i % 2
        conv.core.pack(ws[k].data_ptr(), bs[k].data_ptr(), conv.packed.data_ptr(), conv.b_rep.data_ptr(), st)
        conv(x, out=y)       # right after the pack: no PDL overlap
        conv(x, out=y)       # PDL again, same operands
        outs.append((k, y.clone()))
    torch.cuda.synchronize()
    for i, (k, o) in enumerate(outs):
        assert torch.equal(o, refs[k]), f"launch {i}: not the filter packed just before it"


def test_graph_captured_chain_keeps_order():
    """A CUDA graph capturing [copy x_i -> conv -> checksum of y] for several inputs: the conv nodes carry
    programmatic edges (PDL) and must still see each copy and be seen by each checksum."""
    dt = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(21)
    xs = [(torch.rand((2, 224, 224, 3), generator=g, device="cuda") * 2 - 1).to(dt) for _ in range(4)]
    wt = ((torch.rand((7, 7, 3, 64), generator=g, device="cuda") * 2 - 1) / 12).to(dt)
    b = torch.rand(64, generator=g, device="cuda") * 2 - 1
    conv = wf.FoldedConv2d(wt, b, xs[0].shape, stride=2, padding=3, dtype=dt)
    refs = [_isolated(conv, x).double().sum() for x in xs]
    x = torch.empty_like(xs[0])
    y = conv(xs[0])
    sums = torch.zeros(len(xs), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            for i, xi in enumerate(xs):
                x.copy_(xi)
                conv(x, out=y)
                sums[i] = y.double().sum()
    torch.cuda.current_stream().wait_stream(side)
    for _ in range(3):
        sums.zero_()
        graph.replay()
        torch.cuda.synchronize()
        for i, r in enumerate(refs):
            assert sums[i].item() == r.item(), f"graph replay: input {i} checksum differs"


def test_layer_chain_reads_the_previous_conv_output():
    """conv -> conv -> conv where each layer's input IS the previous layer's output buffer (no torch kernel
    in between): every layer's prologue overlaps the previous grid under PDL and only its griddepcontrol.wait
    orders the read of x after the producer's stores. Compared bitwise with the same chain synchronised
    between layers, eagerly and captured in a CUDA graph."""
    dt = torch.bfloat16
    g = torch.Generator(device="cuda").manual_seed(31)
    shapes = [  # (cin, cout, k, stride, pad, relu)
        (3, 32, 3, 1, 1, True), (32, 64, 3, 1, 1, True), (64, 32, 3, 2, 1, False), (32, 32, 1, 1, 0, True)]
    n, h = 4, 64
    convs, shape = [], (n, h, h, 3)
    for cin, cout, k, s, p, relu in shapes:
        w = ((torch.rand((k, k, cin, cout), generator=g, device="cuda") * 2 - 1) / (k * k * cin) ** 0.5).to(dt)
        b = torch.rand(cout, generator=g, device="cuda") * 0.2 - 0.1
        conv = wf.FoldedConv2d(w, b, shape, stride=s, padding=p, dtype=dt)
        convs.append((conv, relu))
        shape = conv.output_shape
    xs = [(torch.rand((n, h, h, 3), generator=g, device="cuda") * 2 - 1).to(dt) for _ in range(5)]

    def chain(x, sync):
        for conv, relu in convs:
            x = conv(x, relu=relu)
            if sync:
                torch.cuda.synchronize()
        return x

    refs = [chain(x, True).clone() for x in xs]
    torch.cuda.synchronize()
    outs = [chain(x, False) for x in xs for _ in range(2)]
    torch.cuda.synchronize()
    for i, o in enumerate(outs):
        assert torch.equal(o, refs[i // 2]), f"eager chain {i}: differs from the synchronised chain"
    # the same chain in a graph (static buffers), replayed for every input
    x_in = torch.empty_like(xs[0])
    bufs = [torch.empty(c.output_shape, dtype=dt, device="cuda") for c, _ in convs]
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            cur = x_in
            for (conv, relu), buf in zip(convs, bufs):
                conv(cur, relu=relu, out=buf)
                cur = buf
    torch.cuda.current_stream().wait_stream(side)
    for i, x in enumerate(xs):
        x_in.copy_(x)
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(bufs[-1], refs[i]), f"graph chain {i}: differs from the synchronised chain"
