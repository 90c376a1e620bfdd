"""widthfold-b200: B200-native folded first-layer convolution (arXiv 2601.11608).

Drop-in for the reference ``widthfold`` conv path (/root/reference/proj): the
fold / filter-expansion rewrite, the conv entry point and its Python binding,
re-designed for sm_100a (TMA + tcgen05 + TMEM). Same public names as
/root/reference/proj/python/widthfold/__init__.py:5-49.
"""
from .api import (  # noqa: F401
    BlobSizeMismatchError,
    DegenerateOutputError,
    IoFailureError,
    ManifestParseError,
    FoldedConv2d,
    Graph,
    MissingInputError,
    ShapeInferenceFailureError,
    IllegalFoldError,
    NotBlockDiagonalError,
    ShapeMismatchError,
    UnsupportedError,
    apply_width_fold,
    apply_width_fold_general,
    bias_add,
    check_legality,
    choose_fold_factor,
    conv1d_h,
    conv2d,
    count_macs,
    expand_filter,
    expand_filter_folded,
    expand_filter_general,
    fold_input,
    fold_input_general,
    fold_tall_skinny,
    gemm_as_conv1x1,
    gemm_ref,
    grouped_conv,
    interpret,
    mac_report,
    plan_fold,
    read_bundle,
    read_graph,
    reconstruct_output,
    replicate_bias,
    unfold_input_general,
    width_fold_pass,
    write_bundle,
    write_graph,
)
from .api import __all__  # noqa: F401

__version__ = "0.1.0"
