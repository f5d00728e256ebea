"""B200-native RHS + SSP-RK3 hot path of the arXiv 2202.02319 reacting-flow
solver, behind the reference's ``ignis::Simulation`` interface (C ABI in
include/ignis_b200.h)."""
from . import abi, configs, errors  # noqa: F401
from .sim import Ensemble, SlabGroup, Simulation  # noqa: F401
