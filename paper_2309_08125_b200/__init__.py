"""B200-native Oobleck planner: pipeline-template generation DP on sm_100a (PAPER §4.1)
plus host instantiation / batch distribution (§4.2), behind the C ABI of
include/oobleck_plan.h.  See DESIGN.md."""
from . import planner  # noqa: F401  (raises ImportError if liboobleck_plan.so is missing)

__all__ = ["planner"]
