"""FoldedConv2d.run_host (the e2e leg of bench.py) and with_batch.

run_host pipelines chunks over two streams: each stream has its own input /
output buffers and its own conv (with_batch), so a plan that needs a
workspace (AlexNet's re-pitch) never shares it between chunks in flight, and
a short tail chunk gets a plan of its own (its batch-dependent tiling can
differ from the parent's). Integer-valued data keeps the tensor-core results
exact, so every comparison is bitwise.
"""
import pytest
import torch

import paper_2601_11608_b200 as wf

pytestmark = pytest.mark.gpu


def _int_case(n, h, k, co, dt, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randint(-4, 5, (n, h, h, 3), generator=g, device="cuda").to(dt)
    w = torch.randint(-3, 4, (k, k, 3, co), generator=g, device="cuda").to(dt)
    b = torch.randint(-8, 9, (co,), generator=g, device="cuda").float()
    return x, w, b


@pytest.mark.parametrize("geom", [
    # n, h, k, cout, stride, pad, chunk (the last chunk is a short tail)
    (37, 227, 11, 96, 4, 0, 8),    # AlexNet rows: re-pitch workspace per stream
    (21, 224, 7, 64, 2, 3, 6),     # R50 conv1
])
@pytest.mark.parametrize("relu", [False, True])
def test_run_host_matches_device_conv(geom, relu):
    n, h, k, co, s, p, chunk = geom
    x, w, b = _int_case(n, h, k, co, torch.bfloat16, seed=n * k)
    conv = wf.FoldedConv2d(w, b, x.shape, stride=s, padding=p, dtype=torch.bfloat16)
    ref = conv(x, relu=relu, out_dtype=torch.float32)
    xh = x.cpu().pin_memory()
    yh = torch.empty(tuple(ref.shape), dtype=torch.float32).pin_memory()
    yh.fill_(float("nan"))
    conv.run_host(xh, yh, chunk=chunk, relu=relu)
    torch.cuda.synchronize()
    assert torch.equal(yh, ref.cpu())
    # and again: the per-stream convs and buffers are rebuilt per call, results identical
    yh2 = torch.zeros_like(yh).pin_memory()
    conv.run_host(xh, yh2, chunk=chunk, relu=relu)
    torch.cuda.synchronize()
    assert torch.equal(yh2, yh)


def test_run_host_rejects_device_tensors():
    x, w, b = _int_case(2, 64, 7, 64, torch.bfloat16, seed=3)
    conv = wf.FoldedConv2d(w, b, x.shape, stride=2, padding=3, dtype=torch.bfloat16)
    with pytest.raises(ValueError):
        conv.run_host(x, torch.empty((2, 32, 32, 64)))


@pytest.mark.parametrize("n_parent,n_child", [(512, 1), (512, 7), (3, 300)])
def test_with_batch_equals_fresh_plan(n_parent, n_child):
    """with_batch(m) on R50 conv1: small batches plan per-group N-tiles and one tile per stage (a
    different packed operand, so it is packed again); large ones share the parent's. Either way the
    result equals a conv planned for batch m from scratch, and each image equals the parent's result."""
    x, w, b = _int_case(max(n_parent, n_child), 224, 7, 64, torch.bfloat16, seed=n_parent + n_child)
    parent = wf.FoldedConv2d(w, b, (n_parent, 224, 224, 3), stride=2, padding=3, dtype=torch.bfloat16)
    child = parent.with_batch(n_child)
    fresh = wf.FoldedConv2d(w, b, (n_child, 224, 224, 3), stride=2, padding=3, dtype=torch.bfloat16)
    assert child.input_shape == fresh.input_shape and child.output_shape == fresh.output_shape
    mine = {k: v for k, v in child.device_plan.items()}
    theirs = {k: v for k, v in fresh.device_plan.items()}
    assert mine == theirs  # the child runs the plan a fresh conv would
    xc = x[:n_child].contiguous()
    yc = child(xc, out_dtype=torch.float32)
    assert torch.equal(yc, fresh(xc, out_dtype=torch.float32))
    m = min(n_parent, n_child)
    yp = parent(x[:n_parent].contiguous(), out_dtype=torch.float32)
    assert torch.equal(yc[:m], yp[:m])


def test_repitch_input_then_prepitched_conv_equals_one_call():
    """wf_repitch_input + WF_EPI_PREPITCHED (the re-pitch pass split from the conv) == the single call,
    bitwise, on AlexNet rows; and on a plan without a workspace the split pass is a no-op."""
    x, w, b = _int_case(16, 227, 11, 96, torch.bfloat16, seed=99)
    conv = wf.FoldedConv2d(w, b, x.shape, stride=4, padding=0, dtype=torch.bfloat16)
    assert conv.device_plan["producer"] == "repitch+tma" and conv.workspace is not None
    ref = conv(x, out_dtype=torch.float32)
    y = torch.full_like(ref, float("nan"))
    st = torch.cuda.current_stream().cuda_stream
    conv.workspace.zero_()
    conv.core.repitch(x.data_ptr(), conv.workspace.data_ptr(), st)
    conv._forward(x, out=y, out_dtype=torch.float32, flags=4)  # WF_EPI_PREPITCHED
    torch.cuda.synchronize()
    assert torch.equal(y, ref)
    x2, w2, b2 = _int_case(2, 64, 7, 64, torch.bfloat16, seed=5)
    c2 = wf.FoldedConv2d(w2, b2, x2.shape, stride=2, padding=3, dtype=torch.bfloat16)
    assert c2.workspace is None
    c2.core.repitch(x2.data_ptr(), 0, st)  # no workspace: nothing to do
