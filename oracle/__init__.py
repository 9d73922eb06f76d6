"""CPU oracle for the memory-layer hot path of arXiv 2412.09764.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package.  The product path (`paper_2412_09764_b200`) never imports it and
shares no code with it: no kernels, helpers, tables or constants.

Everything is plain numpy in float64 on the dtype-rounded inputs, written to
be checked against the paper by eye.  Citations: `P:n` = PAPER.md line n
(section / equation noted), `S:n` = SPEC.md line n, readings `Qn` = the
ambiguity table in SURVEY.md §8(c) as restated in DESIGN.md.

Pins (tests/test_oracle_*.py, `-m "not gpu"`) tie each function to something
other than itself: the paper's additive decomposition checked against
materialised brute force, closed forms (q = 0, k = 1, equal scores), the
SPEC.md hand examples, finite differences of the forward for every gradient,
dense-matrix re-formulations of the sparse bag, and sharded == unsharded.
Parity unpinned: none of the functions here.
"""
from . import pkm, bag, gate, layer, group, optim, peer  # noqa: F401
