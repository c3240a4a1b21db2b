"""Golden E(k) values of the reference's scaling harness (acceptance criteria
08 / 09, mmtplan tests/test_acceptance.py:189-210), generated from the
reference itself in the build container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_scaling_golden.py

Writes tests/golden/scaling.json: for each sharing scheme the reference's
scaling_experiment(arch, [4, 8, 12, 16, 20], steps=5) (floats as hex, bit
exact) and the criterion-08 run_benchmark summary (independent scheme,
ClusterTopology(2, 4, 1), 8 tasks, 10 steps)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from mmtplan import core as R_core  # noqa: E402
from mmtplan import syncsim as R_sim  # noqa: E402

KS = [4, 8, 12, 16, 20]


def main():
    out = {"ks": KS, "steps": 5, "efficiency": {}}
    for arch in R_sim.SCALING_ARCHS:
        eff = R_sim.scaling_experiment(arch, KS, steps=5)
        out["efficiency"][arch] = {str(k): float(v).hex() for k, v in eff.items()}
    topo = R_core.ClusterTopology(2, 4, 1)
    tasks = R_sim.synthetic_uniform_tasks("independent", 8, topo)
    _, summary = R_sim.run_benchmark(tasks, topo, steps=10)
    out["criterion08"] = {k: summary[k] for k in ("grad_allreduce_bytes", "ready_sync_bytes", "total_tokens",
                                                   "devices", "tasks", "modules")}
    with open(os.path.join(HERE, "scaling.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out)[:400])


if __name__ == "__main__":
    main()
