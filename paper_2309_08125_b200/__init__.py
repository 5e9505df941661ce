"""B200-native Oobleck planner: pipeline-template generation DP on sm_100a (PAPER §4.1)
plus host instantiation / batch distribution (§4.2), behind the C ABI of
include/oobleck_plan.h.  See DESIGN.md.

`planner` (and `_lib`) load liboobleck_plan.so and raise ImportError if it is missing —
there is no CPU fallback.  `build` compiles it and is importable without the library.
"""
import importlib

__all__ = ["planner", "build"]


def __getattr__(name):
    if name in ("planner", "_lib", "build"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
