"""qfuse-b200: B200-native fused forward + adjoint gradient for batched
state-vector circuits (arXiv 2603.02804), behind a C-ABI drop-in for the
reference qfuse engine. See include/qfuse_b200.h and DESIGN.md."""
from . import circuits
from .capi import (Context, GradientResult, Group, GroupPlan, Plan, QfCapacityError, QfError,
                   QfInvalidArgument, forward_c64, gradient_c64, gradient_c64_multi, gradient_c128,
                   load,
                   LIB_PATH, SYMBOLS)

__all__ = ["circuits", "Context", "Plan", "GradientResult", "gradient_c64", "gradient_c128", "load",
           "Group", "GroupPlan", "gradient_c64_multi", "forward_c64",
           "QfError", "QfInvalidArgument", "QfCapacityError", "LIB_PATH", "SYMBOLS"]
