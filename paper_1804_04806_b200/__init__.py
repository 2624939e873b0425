"""B200-native micro-batched convolution (mu-cuDNN, arXiv:1804.04806).

The product is libucudnn.so (C ABI in include/ucudnn.h): sm_100a tcgen05
convolution kernels, a device benchmarker writing the reference cost-table
CSV, the reference-exact WR/WD planner and the micro-batch executor. This
package is the Python mirror of that ABI plus the data-parallel driver.
"""
from .api import (ALGOS, BACKWARD_DATA, BACKWARD_FILTER, FORWARD, MODES, OP_NAMES, POLICIES, VIRTUAL_ALGO_BASE,
                  ConvShape, Handle, algorithm_workspace, canonical_cost_table, canonical_time, kernel_hash,
                  plan_kernels, plan_network_file)
from ._lib import UcudnnError

__all__ = ["ALGOS", "BACKWARD_DATA", "BACKWARD_FILTER", "FORWARD", "MODES", "OP_NAMES", "POLICIES",
           "VIRTUAL_ALGO_BASE", "ConvShape", "Handle", "UcudnnError", "algorithm_workspace", "canonical_cost_table",
           "canonical_time", "kernel_hash", "plan_kernels", "plan_network_file"]
