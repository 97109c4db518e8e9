"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU (NumPy, FP64 by default) implementation of
what the CUDA path computes, written from /root/reference/PAPER.md (cited as
``PAPER.md:<line>``) and the readings listed in DESIGN.md ("Readings").

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from here.
The product package ``paper_2109_08008_b200`` never imports it and shares no
code with it; the two meet only through the seeded input generators in
``synth/`` (weights, workloads) which hold none of the method's arithmetic.

Parity status per function is stated in each module header; the only
"parity unpinned" items are the readings the paper does not fix (DESIGN.md
R2-R8, R10) and end-to-end quality (BLEU), which needs trained weights.
"""
from .nn import layer_norm, softmax, log_softmax, sinusoid_pe, rel_index  # noqa: F401
from .model import OracleModel  # noqa: F401
from .batching import plan_batches, restore_order  # noqa: F401
from .search import (greedy_def, translate_fast, beam_search, exhaustive_best,  # noqa: F401
                     beam_search_nbest, exhaustive_nbest, ensemble_step_logprobs)
