"""B200-native direct-summation N-body hot path (arXiv 2509.19294).

The compute path is ``libnbody.so`` (C-ABI, hand-written sm_100a CUDA); this
package only marshals arguments to it.  Importing the package does not load
the library; constructing :class:`NBody` does, and fails loudly if it is
missing.
"""
__all__ = ["NBody", "NBodyError", "inputs"]


def __getattr__(name):
    if name in ("NBody", "NBodyError", "lib"):
        from . import binding
        return getattr(binding, name)
    raise AttributeError(name)
