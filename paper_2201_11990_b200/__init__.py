"""B200-native hot path of the MT-NLG 3D-parallel training step (arXiv 2201.11990).

Host-side Python mirror of the reference's planner/partition/schedule API (`curator::` in
proj/include/curator/planner.hpp) over the C ABI of libmtnlg.so, which holds the C++ runtime
and the hand-written sm_100a kernels. There is no CPU fallback: the native library must load.
"""
from . import _native  # noqa: F401

__all__ = ["_native"]
