"""CPU oracle for the DMT / SPTT hot path -- TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference (`towersim` 0.1.0,
/root/reference/pkg/src/towersim) used purely as a *checker*:

* only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
  ``cpu_baseline`` / ``--impl reference`` legs may import it;
* the product package ``paper_2403_00877_b200`` never imports it and has no CPU
  fallback -- its ops fail loudly when the CUDA library is missing.

Parity status: the forward path (placement, step-a routing, pooled lookup,
flat baseline, SPTT a-f, realign, TM forward, widths, flops, byte accounting)
is PINNED against fixtures produced by the real reference
(tests/golden/make_golden.py -> tests/golden/*.npz, golden.json) in
tests/test_oracle_golden.py.  The backward restatement (embedding-bag grads,
SGD / row-wise Adagrad, TM backward) has no reference counterpart; the TM
weight gradients are pinned through the adjoint identity against the
reference's own ``tm_weight_jvp`` fixtures, the rest is "parity unpinned"
(restated from the forward definitions).
"""

from .towersim_port import *  # noqa: F401,F403
from .backward import *  # noqa: F401,F403
from .dlrm import *  # noqa: F401,F403
