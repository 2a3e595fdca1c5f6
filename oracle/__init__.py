"""fp64 CPU oracle for the Neptune attention hot path (arXiv 2510.08726).

TEST INFRASTRUCTURE ONLY. Nothing in the product package
(``paper_2510_08726_b200``) may import, call or link anything under
``oracle/``; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs do. The oracle shares no code
with the CUDA path: its inputs come from ``datagen`` (which holds no attention
arithmetic) and it is pinned by ``tests/test_oracle_*.py`` against hand-derived
values, closed forms, invariants and an independent library (torch CPU fp64).

Citations: ``P:n`` = line n of the paper's PAPER.md (section / figure /
equation in brackets).
"""
from .attention import (  # noqa: F401
    Problem,
    attention,
    attention_bh,
    rolling_update_bh,
    rolling_update_lazy_bh,
    splitk_local_bh,
    splitk_combine,
    splitk_merge,
    head_group,
)
from .softmax_chain import (  # noqa: F401
    softmax_denominator,
    softmax_denominator_naive_fused,
    softmax_denominator_rolling,
    softmax_denominator_privatized,
    softmax_denominator_splitk,
    repair_h,
    softmax_rows,
)
