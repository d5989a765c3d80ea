"""CF-DETR coarse-to-fine encoder oracle (TEST INFRASTRUCTURE ONLY).

Plain, slow, fp64 numpy implementation of the hot path of CF-DETR
(arXiv 2505.23317, §III A1-A3).  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
leg may import or execute anything under `oracle/`.  The product path
(`paper_2505_23317_b200`) never imports it and shares no code with it; the two
meet only in `cfd_inputs` (seeded inputs, no method arithmetic).
"""
from .cfdetr_oracle import *  # noqa: F401,F403
