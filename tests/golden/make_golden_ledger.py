"""Golden ledger columns of the reference's run_benchmark (syncsim.py:295-392),
generated in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_ledger.py

Per step: ready_bytes, grad_bytes, tokens (the byte / token definitions the
B200 run_benchmark keeps; its times are measured, the reference's modeled),
plus the summary's count columns, for config 1 (accum 1 and 2) and config 3
placed on 2 and 4 devices.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mmtplan import syncsim as R_sim  # noqa: E402

from make_golden import ref_topo, to_ref_task  # noqa: E402
from paper_2403_07544_b200 import configs  # noqa: E402


def run(tasks, topo, steps, accum, batch_tokens):
    ledger, summary = R_sim.run_benchmark([to_ref_task(t) for t in tasks], ref_topo(topo), steps,
                                          seed=0, accum_count=accum, batch_tokens=batch_tokens)
    return {"records": [[r.ready_bytes, r.grad_bytes, r.tokens] for r in ledger.records],
            "summary": {k: summary[k] for k in ("steps", "devices", "tasks", "modules",
                                                "total_tokens", "grad_allreduce_bytes",
                                                "ready_sync_bytes")}}


def main():
    out = {}
    w1 = configs.config1()
    for accum in (1, 2):
        out[f"config1_accum{accum}"] = run(w1.tasks, w1.topo, 4, accum, 256)
    for world in (2, 4):
        w3 = configs.config3(world)
        out[f"config3_w{world}"] = run(w3.tasks, w3.topo, 3, 1, 512)
    with open(os.path.join(HERE, "ledger.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote ledger.json")


if __name__ == "__main__":
    main()
