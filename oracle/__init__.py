"""CPU float64 oracle for AutoByte's meta-network candidate scoring (arXiv 2112.13509).

TEST INFRASTRUCTURE ONLY. Only `tests/`, `__graft_entry__.smoke()` and bench.py's
`cpu_baseline` / `--impl reference` legs may import or execute anything under `oracle/`.
The product path (`paper_2112_13509_b200`, `libautobyte.so`) never imports it and shares
no code, headers, constants or helpers with it.

The oracle is the plain definition of what the method computes, written out in float64 with
numpy; a matrix product (`@`) is the only library primitive used. Each function cites the
PAPER.md line it follows (P:n) and, where the paper is silent, the DESIGN.md reading (R#n)
that fixes the choice. Pins (tests/test_oracle_*.py, `-m "not gpu"`): torch.nn.LSTM in
float64, hand-computed nets, closed forms, finite differences, brute force.
Parity unpinned: the learned function itself (the paper publishes no weights or worked
example of the meta-network); only computation-given-weights is pinned.
"""
from .metanet import (  # noqa: F401
    encode_candidate, encode_grid, encode_job, encode_jobs, lstm_step, head_forward,
    speed, score_matrix, score_pairs, argmax_rows, loss_norm, adapt, head_loss_and_grad,
    HEAD_PARAMS, train, topk_rows, encoder_grad, ENCODER_PARAMS,
)
from .trigger import trigger_decide, KEEP, RECONFIGURE, ADAPT  # noqa: F401,E402
from . import bytescheduler  # noqa: F401,E402  (NEXT 3: one ByteScheduler iteration per candidate)
