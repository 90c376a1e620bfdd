"""Random conv graphs for the pass-soundness tests, after the reference's
graph generator (tests/support/graph_gen.hpp:74-163): a mix of foldable and
unfoldable first-layer-like convs (Cin in {1, 3, 4, 8}, KW 1..7, strides,
padding), optional bias_add consumers, reshapes and several outputs, so every
skip reason occurs."""
import numpy as np

import paper_2601_11608_b200 as wf


def random_graph(seed: int, integer: bool) -> tuple[wf.Graph, dict]:
    rng = np.random.default_rng(seed)

    def data(shape, scale=1.0):
        if integer:
            return rng.integers(-4, 5, shape).astype(np.float32)
        return (rng.uniform(-1, 1, shape) * scale).astype(np.float32)

    g = wf.Graph()
    B = int(rng.integers(1, 3))
    H = int(rng.choice([8, 12, 16]))
    W = int(rng.choice([8, 16, 24, 30, 32]))
    C = int(rng.choice([1, 3, 3, 4, 8]))
    g.add("x", "input", shape=[B, H, W, C])
    inputs = {"x": data((B, H, W, C))}
    n_conv = int(rng.integers(1, 4))
    for i in range(n_conv):
        kh = int(rng.integers(1, 6))
        kw = int(rng.choice([1, 2, 3, 5, 7]))
        s = int(rng.choice([1, 1, 2]))
        p = int(rng.integers(0, 3)) if kw > 1 else 0
        if H + 2 * p < kh or W + 2 * p < kw:
            kh, kw, p = 1, 1, 0
        cout = int(rng.choice([16, 32, 64]))
        g.constant(f"w{i}", data((kh, kw, C, cout), 1.0 / np.sqrt(kh * kw * C)))
        g.add(f"c{i}", "conv2d", ["x", f"w{i}"], stride_h=s, stride_w=s, pad_h=p, pad_w=p)
        tail = f"c{i}"
        if rng.random() < 0.6:  # a sole-consumer bias_add (fused by the pass)
            g.constant(f"b{i}", data((cout,)))
            g.add(f"ba{i}", "bias_add", [tail, f"b{i}"])
            tail = f"ba{i}"
        if rng.random() < 0.3:  # a flattening reshape before the output
            out = g.infer_shapes().find(tail)["out_shape"]
            g.add(f"r{i}", "reshape", [tail], shape=[out[0], int(np.prod(out[1:]))])
            tail = f"r{i}"
        g.add(f"y{i}", "output", [tail])
    return g, inputs
