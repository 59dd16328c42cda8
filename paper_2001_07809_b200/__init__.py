"""paper_2001_07809_b200 -- B200-native (sm_100a) per-frame stereo depth +
depth-masked refocus pipeline (arXiv 2001.07809), a drop-in for the
reference's stereotk::run_refocus_pipeline path.

  include/stk_b200.h          C-ABI (libstk_b200.so, built in-tree)
  include/stereotk/...        C++ drop-in of the reference's stereotk:: API
  paper_2001_07809_b200.stereotk   Python mirror of the same API (ctypes)
  paper_2001_07809_b200.synth      deterministic synthetic scenes
"""
from ._build import build  # noqa: F401

__all__ = ["build", "stereotk", "synth"]


def __getattr__(name):
    if name in ("stereotk", "synth"):
        import importlib

        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
