"""CPU oracle for the E-Tree / E-Forest ADC hot path (arXiv 1509.05186).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library, its
Python binding) may import, call, link or execute anything in this package.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs use it.

It is a plain, slow, obviously-correct numpy implementation written from
PAPER.md (cited as ``P:<line>``) with the readings listed in DESIGN.md §3
(cited as ``A<n>``, numbering from SURVEY.md §8c).  Floating point is fp64 unless
a function is explicitly the paper-faithful fp32 variant (the pseudocode at
P:234 declares ``float``).  It shares no code with the CUDA path: the only
module both sides import is ``paper_1509_05186_b200.synth`` (seeded input
generation, none of the method's arithmetic).

Modules
-------
pq       PQ training (k-means++ + Lloyd), encode, decode, distance tables, naive ADC
etree    E-Tree: plain-definition statistics, Algorithm 1 build, Hierarchical
         Memory Structure serialise / parse, Distance-Context traversal
eforest  E-Forest: T trees over disjoint byte ranges, per-id summation
topk     exact top-k by (distance, id)
ivf      IVFADC application (coarse quantizer + residual PQ + per-list trees)
shard    first-level-subtree sharding and top-k merge

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` except where its docstring says "parity unpinned".
"""
