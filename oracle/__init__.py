"""CPU oracle for the prefix-shared decode-attention path.

TEST INFRASTRUCTURE ONLY. This package restates, in plain numpy and
Python, the algorithm of the reference package `prefixdec`
(/root/reference/pkg/src/prefixdec) for the one hot path this repo
accelerates: forest indexing -> cost model / task division / LPT
schedule -> split-phase partial attention -> log-sum-exp merge.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline
legs (`cpu_baseline`, `--impl reference`) may import it, and only as the
checker or the timed CPU reference -- never as the thing measured on the
GPU and never as a fallback of the product path
(`paper_2505_17694_b200`), which fails loudly when its CUDA library is
missing.

Parity pin: every function here is checked against golden vectors that
`tests/golden/make_golden.py` produced by importing the real reference
in the build container (tests/test_oracle_golden.py). The oracle is
therefore "pinned", not a free-standing restatement.

Each function's docstring cites the reference file:line it restates.
"""
