"""winomem-b200: memory-efficient Strassen-Winograd schedules on NVIDIA B200.

B200-native (sm_100a) re-implementation of the hot path of
Boyer, Dumas, Pernet, Zhou -- *Memory efficient scheduling of Strassen-Winograd's
matrix multiplication algorithm* (ISSAC 2009): the schedule interpreter and its
drivers (std2, acc2 and its closure, ip, ipmm, ...) behind the reference's
API, with the block additions and the classical base products as CUDA
kernels.  See DESIGN.md.
"""
from .winomem import (  # noqa: F401
    BUILTIN_NAMES, Context, CostReport, MatView, Matrix, Modulus, MultiplyOptions,
    alias_error, block_addsub, block_scale_copy, classical_mul, compare, contract_error,
    contract_violation_error, cuda_error, dimension_error, expected_costs, ipmm, ipovmm,
    kDefaultModulus, multiply, odd_dimension_error, parse_error, parse_schedule,
    partial_overlap_error, plan_report, quad_split, render_schedule, run_parsed_schedule,
    run_variant, run_variant_host, shape_error, unknown_schedule_error, unknown_slot_error,
    variant_accumulates, workspace_error, io_error, matrix_file_info, read_matrix_host,
    write_matrix_host, read_text, read_binary, write_text, write_binary, lincomb, DistContext)
