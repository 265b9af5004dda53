"""CPU oracle for the IKJT training hot path -- TEST INFRASTRUCTURE ONLY.

This package is a plain numpy restatement of the reference's algorithms
(`/root/reference/pkg/src/sessiondedup/tensors.py` and `trainer_sim.py`),
each function citing the file:line it follows.  It is the checker, never
the thing measured or shipped: only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import it.  The
product package `paper_2211_05239_b200` never imports this module and fails
loudly when its CUDA extension is missing.

Parity pinning: the forward restatement (dedup, jagged index select,
lookup, pooling, expansion, DP slicing) is pinned against golden vectors
produced by importing the real reference (`tests/golden/make_golden.py`
-> `tests/golden/*.npz`, checked by `tests/test_oracle_golden.py`).
The backward has no reference implementation (`SPEC.md:13` puts training
out of scope; `SURVEY.md` §8(c)) -- its oracle is our own definition,
cross-checked against torch-CPU autograd of `F.embedding_bag`
(`tests/test_oracle_backward.py`): "backward parity unpinned by the
reference, pinned by torch autograd".
"""

from .ikjt import (  # noqa: F401
    build_kjt_arrays,
    build_ikjt_arrays,
    build_ikjt_rows,
    jagged_index_select,
    ikjt_to_kjt_arrays,
    slice_ikjt_rows,
    row_lengths,
)
from .embedding import (  # noqa: F401
    embedding_lookup,
    pool,
    pooled_lookup,
    expand,
    pool_backward,
    sparse_table_grad,
    sgd_apply,
    attention_pool,
)
from .reader import apply_transform, splitmix64  # noqa: F401,E402
from . import wire  # noqa: F401,E402
