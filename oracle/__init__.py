"""CPU oracle for the SageAttention2 forward pass (arXiv 2411.10958).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The product path
(``paper_2411_10958_b200``) never imports it; the two share no code.

The arithmetic lives in ``sage2_oracle.c`` (plain C loops, fp64, OpenMP over independent rows);
this module only builds it with gcc and marshals numpy arrays through ctypes.  ``metrics`` holds
the paper's accuracy metrics.
"""
from .oracle import (  # noqa: F401
    OracleConfig,
    build,
    lib,
    e4m3_encode,
    e4m3_decode,
    fp16_round,
    fp16_decode,
    fp22_truncate,
    group_q,
    group_k,
    group_q_g,
    group_k_g,
    ngroups,
    kv_head,
    q_block,
    q_head_delta,
    delta_s,
    s_int_block,
    attn_block,
    attn_exact_tiled,
    sage2_forward_blocks,
    num_threads,
)
from .metrics import cos_sim, rel_l1, rmse  # noqa: F401
