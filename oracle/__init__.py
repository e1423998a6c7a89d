"""CPU oracle for the Zipage compression step — TEST INFRASTRUCTURE ONLY.

This package is the plain, slow, obviously-correct fp64 definition of what the
compression step of Compressed PagedAttention (arXiv 2603.08743) computes. It
exists to prove the CUDA path right; it is never part of the product path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import it. It imports nothing from
``paper_2603_08743_b200`` (the CUDA product) and the product imports nothing
from here; the two share no arithmetic, constants or helpers.

Parity status per function:
  plan, finalize, select, max_pool, pin, compact_*  -> pinned (SPEC examples,
      Fig. 1 toy structure, brute force, conservation invariants)
  logits_*, attention_scores                         -> pinned by closed forms
      (G=1,w=1 textbook softmax; constant keys; sum rules; GQA dominance;
      blockwise == dense). Realistic-input score VALUES beyond those closed
      forms are "parity unpinned": the paper prints no numeric score example.
"""
from .zipc_oracle import *  # noqa: F401,F403
