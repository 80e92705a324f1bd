"""paper_2601_03187_b200 -- B200-native hot path of TaNG (arXiv 2601.03187).

libtang.so (csrc/, C ABI in include/tang.h) runs the whole classification path on the
GPU; `tang` is its ctypes binding, `train` the plain off-path trainer that emits the
model blob.  Import `paper_2601_03187_b200.tang` to load the library (fails loudly when
it is not built -- there is no CPU fallback).
"""
__all__ = ["tang", "train", "build_ext"]
