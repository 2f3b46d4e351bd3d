"""B200-native (sm_100a) implementation of AriaNN's function-secret-sharing hot
path (arXiv 2006.04593): batched DPF/DCF key generation and evaluation with the
AES-MMO PRG, behind a drop-in of the reference's ``ariann.prg`` / ``ariann.fss``
Python API. See DESIGN.md.
"""

from . import _lib

__all__ = ["prg", "fss", "ring", "sharing", "runtime", "beaver", "nn_ops", "dealer", "keyfile", "shard"]
__version__ = "0.1.0"


def library_path() -> str:
    from ._build import LIB
    return LIB


def __getattr__(name):
    if name in __all__:
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
