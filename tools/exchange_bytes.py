"""Expected NVLink bytes per rank per step of the module-gradient exchange,
per transport, for configs 3 and 5 at 8 GPUs.

Uses the real plan (group map, syncsim.py:337-340) and the multiplexer's
picks (syncsim.py:190-205) over STEPS steps; module sizes are the engine's
true buckets (model.py layouts).  Bytes follow the collectives' bus
traffic per rank: ring all-reduce 2(g-1)/g * B, broadcast / reduce-scatter /
all-gather (g-1)/g * B; option B counts the remote gradient reads of the
shard owner ((n - own) / g of the bucket) and the g - 1 remote bf16 weight
stores of the owned shard.

    python tools/exchange_bytes.py [steps]
"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2403_07544_b200 import configs  # noqa: E402
from paper_2403_07544_b200.model import module_layouts  # noqa: E402
from paper_2403_07544_b200.plan import Multiplexer, build_plan, ready_counts_all, task_modules  # noqa: E402

NVLINK_GBS = 900.0


def per_rank_bytes(wl, steps):
    plan = build_plan(wl.tasks, wl.topo)
    lay = module_layouts(plan, wl.shape)
    ranks = sorted(plan.tasks_by_rank)
    mux = {r: Multiplexer(plan, r, 0) for r in ranks}
    idx = plan.index()
    out = {t: {r: [] for r in ranks} for t in ("allreduce_fp32", "partitioned", "partitioned_bf16grad",
                                                "peer_option_b")}
    for s in range(steps):
        used = {r: set(task_modules(mux[r].pick(s))) for r in ranks}
        counts = ready_counts_all(plan, used)
        for r in ranks:
            acc = {t: 0.0 for t in out}
            for k in plan.hosted[r]:
                g, n = len(plan.groups[k]), counts[idx[k]]
                if g < 2 or n < 1:
                    continue
                numel = lay[k].numel
                f = (g - 1) / g
                acc["allreduce_fp32"] += (2 * f if n >= 2 else f) * 4 * numel
                acc["partitioned"] += f * (4 + 2) * numel
                acc["partitioned_bf16grad"] += f * (2 + 2) * numel
                own = 1 if k in used[r] else 0
                acc["peer_option_b"] += (n - own) / g * 4 * numel + (g - 1) * 2 * numel / g
            for t in out:
                out[t][r].append(acc[t])
    res = {}
    for t, by_rank in out.items():
        mean_r = [statistics.mean(v) for v in by_rank.values()]
        worst_step = [max(by_rank[r][s] for r in ranks) for s in range(steps)]
        res[t] = {"mean_rank_GB": statistics.mean(mean_r) / 1e9,
                  "max_rank_mean_GB": max(mean_r) / 1e9,
                  "mean_step_max_rank_GB": statistics.mean(worst_step) / 1e9,
                  "ms_at_900GBs": statistics.mean(worst_step) / (NVLINK_GBS * 1e9) * 1e3,
                  "ms_at_60pct": statistics.mean(worst_step) / (0.6 * NVLINK_GBS * 1e9) * 1e3}
    return res


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    res = {"config3_w8": per_rank_bytes(configs.config3(8), steps),
           "config5_w8": per_rank_bytes(configs.config5(8), steps), "steps": steps}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
