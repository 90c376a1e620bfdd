"""widthfold-b200: B200-native folded first-layer convolution (arXiv 2601.11608).

Drop-in for the reference ``widthfold`` conv path (/root/reference/proj):
the fold / filter-expansion rewrite, the conv entry point and its Python
binding, re-designed for sm_100a (TMA + tcgen05 + TMEM).
"""
__version__ = "0.1.0"
