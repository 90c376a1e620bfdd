timeout 300 python -m pytest "tests/test_gpu_parity.py::test_partial_tiles_and_odd_shapes" -q -m gpu -x 2>&1 | grep -v "^\s*$" | tail -40
