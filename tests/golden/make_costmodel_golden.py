"""Golden cost-model values from the REAL reference (towersim.costmodel) on the
traces of the 60 acceptance configs (same generator as make_golden.py).

Test infrastructure only: imports /root/reference (this container only) and
writes tests/golden/costmodel.json, which tests/test_costmodel.py compares
paper_2403_00877_b200.costmodel against.

    python tests/golden/make_costmodel_golden.py
"""

from __future__ import annotations

import itertools
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF_SRC)

from towersim.cli import RunContext, random_config  # noqa: E402
from towersim.costmodel import CostParams, pipeline_cost, speedup_report  # noqa: E402

FLAG_COMBOS = list(itertools.product([False, True], repeat=3))
PARAMS = {
    "default": {},
    "b200": {"alpha_up": 8e-6, "alpha_out": 2.5e-5, "beta_up": 640e9, "beta_out": 45e9,
             "compute_rate": 2.25e15, "efficiency": {1: 1.0, 2: 1.0, 4: 0.9, 8: 0.75, 16: 0.6, 64: 0.5}},
}


def brk(b):
    return {"per_step": b.per_step, "exposed": b.exposed_comm, "compute": b.compute}


def main():
    rng = np.random.default_rng(2024)
    out = []
    for i in range(60):
        cfg = random_config(rng)
        swap, omit, rs = FLAG_COMBOS[i % len(FLAG_COMBOS)]
        cfg["exchange"] = {"swap_bc": swap, "omit_permute": omit, "rowwise_reducescatter": rs}
        ctx = RunContext(cfg)
        base = ctx.run_baseline()
        tower = ctx.run_tower()
        kinds = {"d": "reducescatter"} if rs else None
        rec = {"index": i, "rowwise_reducescatter": rs, "costs": {}}
        for name, kw in PARAMS.items():
            p = CostParams(**kw)
            cb = pipeline_cost(base.trace, ctx.topo, p, flops=dict(base.flops))
            ct = pipeline_cost(tower.trace, ctx.topo, p, layout=ctx.layout, flops=dict(tower.flops),
                               step_kinds=kinds)
            rec["costs"][name] = {"base": brk(cb), "tower": brk(ct), "speedup": speedup_report(cb, ct)}
        out.append(rec)
    with open(os.path.join(HERE, "costmodel.json"), "w") as fh:
        json.dump({"params": {k: {kk: ({str(a): b for a, b in vv.items()} if isinstance(vv, dict) else vv)
                                      for kk, vv in v.items()} for k, v in PARAMS.items()},
                   "configs": out}, fh, indent=1)


if __name__ == "__main__":
    main()
