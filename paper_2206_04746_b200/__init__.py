"""B200-native engine for the HDTorch / hypervec hypervector hot path.

libhvb200.so (csrc/*.cu, sm_100a) behind the C ABI in include/hvb200.h;
`hypervec` mirrors the reference C++ API on host arrays, `device` runs the
HBM-resident pipeline (torch for memory, streams and NCCL plumbing).
"""
from ._native import (DomainError, HVError, InvalidArgument, LogicError, NoDevice, context, launch_count, lib)

__all__ = ["DomainError", "HVError", "InvalidArgument", "LogicError", "NoDevice", "context", "launch_count", "lib"]
