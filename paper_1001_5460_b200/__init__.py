"""paper_1001_5460_b200 -- B200-native Kronecker-structured tensor CG (arxiv 1001.5460).

The product is libtca.so (CUDA, sm_100a) behind the C ABI in include/tca.h;
`paper_1001_5460_b200.tca` is its thin ctypes binding.  Importing `tca` (or
touching any attribute below) fails loudly when the library is missing --
there is no CPU fallback.  `paper_1001_5460_b200.build` compiles it.
"""
import importlib

_EXPORTS = ("Operator", "TcaError", "generate_normal", "version", "kernel_launches")

__all__ = ["tca", *_EXPORTS]


def __getattr__(name):
    if name == "tca" or name in _EXPORTS:
        mod = importlib.import_module(__name__ + ".tca")
        return mod if name == "tca" else getattr(mod, name)
    raise AttributeError(name)
