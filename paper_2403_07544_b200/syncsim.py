"""Drop-in for the hot-path names of ``mmtplan.syncsim`` on B200 buffers.

* ``DeviceState`` / ``sync_step``: the literal Algorithm-1 exchange of
  ``syncsim.py:90-153`` over devices whose buffers are CUDA fp32 tensors; the
  whole exchange is ONE launch of the sm_100a kernel ``mm_sync_emulated``
  (sum over each module's hosting devices in ascending index, ``/ n`` with n =
  devices that used it, n == 0 untouched).  Results are bit-identical to the
  reference's numpy on fp32 buffers.
* ``multiplex``, ``Reservoir`` / ``reservoir_batch``,
  ``ring_allreduce_time``, ``StepRecord`` / ``CommLedger``,
  ``synthetic_uniform_tasks``: same semantics as syncsim.py:190-292, 409-458
  (host-side bookkeeping; the ledger additionally carries measured times).

The real training step (``run_benchmark``'s loop) is ``engine.Engine`` /
``cluster.EmulatedCluster``.
"""
from __future__ import annotations

import dataclasses
import random
from typing import Iterable, Mapping, Optional, Sequence

import numpy as np

import torch

from . import _native, ops
from .domain import ClusterTopology, ModuleKey, TaskSpec, task_id
from .plan import SimulationError, multiplex  # noqa: F401  (re-exported API)
from .sharing import ArchSpec, SharingPattern, build_module_sequence

GRAD_BYTES_PER_PARAM = 4
READY_ENTRY_BYTES = 4


@dataclasses.dataclass
class DeviceState:
    """One device: hosted modules, one buffer per hosted module and the set
    of modules used this step (syncsim.py:90-118).

    ``device=None`` (the reference's constructor): float64 numpy buffers on
    the host, as the reference allocates them; ``accumulate`` and
    ``sync_step`` still do every add / divide in the sm_100a kernels (the
    arrays are staged through the GPU).  ``device="cuda"``: fp32 CUDA
    buffers that stay resident.  Explicit ``buffers`` may be numpy arrays or
    CUDA tensors, float32 or float64."""

    index: int
    hosted: frozenset
    dim: int
    buffers: dict = dataclasses.field(default_factory=dict)
    used: set = dataclasses.field(default_factory=set)
    device: Optional[str] = None

    def __post_init__(self) -> None:
        if not self.buffers:
            if self.device is None:
                self.buffers = {k: np.zeros((self.dim, self.dim)) for k in sorted(self.hosted)}
            else:
                self.buffers = {k: torch.zeros(self.dim, self.dim, device=self.device)
                                for k in sorted(self.hosted)}

    def reset(self) -> None:
        for buf in self.buffers.values():
            if isinstance(buf, np.ndarray):
                buf[...] = 0.0
            else:
                ops.memset(buf, 0)
        self.used.clear()

    def accumulate(self, grads: Mapping[ModuleKey, object]) -> None:
        """buffers[key] += g for every (key, g); g may be a numpy array or a
        tensor.  The add runs on the GPU (mm_axpy_f32 / _f64)."""
        for key, g in grads.items():
            if key not in self.hosted:
                raise SimulationError(f"gradient for unhosted module {key}")
            buf = self.buffers[key]
            if tuple(np.shape(g)) != tuple(buf.shape):
                raise SimulationError(f"gradient shape {tuple(np.shape(g))} != {tuple(buf.shape)}")
            if isinstance(buf, np.ndarray):
                dt = _torch_dtype(buf.dtype)
                y = torch.from_numpy(np.ascontiguousarray(buf)).to("cuda", dt)
                ops.axpy(y.view(-1), _as_cuda(g, dt, y.device).view(-1), 1.0)
                buf[...] = y.cpu().numpy()
            else:
                ops.axpy(buf.view(-1), _as_cuda(g, buf.dtype, buf.device).view(-1), 1.0)
            self.used.add(key)


def _torch_dtype(dt) -> torch.dtype:
    if dt == np.float64:
        return torch.float64
    if dt == np.float32:
        return torch.float32
    raise SimulationError(f"buffers must be float32 or float64, got {dt}")


def _as_cuda(x, dtype: torch.dtype, device) -> torch.Tensor:
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device=device, dtype=dtype).contiguous()


def sync_step(devices: Sequence[DeviceState], only_ready: bool = False) -> dict:
    """Algorithm 1 over all devices (syncsim.py:121-153), one kernel launch
    per dtype (mm_sync_emulated / mm_sync_emulated_f64).

    Host (numpy) buffers are staged to the GPU and the results written back
    as the reference does (every member's buffer replaced by the synced
    value when n >= 1, untouched when n == 0); the returned synced values are
    numpy arrays then, CUDA tensors for CUDA buffers.  ``only_ready=True``
    skips reading the buffers of members that did not use the module (exact
    when those buffers are zero, as after ``reset``)."""
    ordered = sorted(devices, key=lambda d: d.index)
    if len({d.index for d in ordered}) != len(ordered):
        raise SimulationError("duplicate device index")
    if len({d.dim for d in ordered}) > 1:
        raise SimulationError("inconsistent module dimensions across devices")
    keys = sorted(set().union(*(d.hosted for d in ordered))) if ordered else []
    synced: dict = {}
    tables = {torch.float32: [], torch.float64: []}
    staged = {}   # (device index, key) -> CUDA tensor of a host buffer
    host_out = {}
    for key in keys:
        members = [d for d in ordered if key in d.hosted]
        if len(members) > _native.MAX_SYNC_GROUP:
            raise SimulationError(f"module {key}: {len(members)} hosts > {_native.MAX_SYNC_GROUP}")
        bufs = [d.buffers[key] for d in members]
        host = [isinstance(b, np.ndarray) for b in bufs]
        if any(host) and not all(host):
            raise SimulationError(f"module {key}: host and device buffers mixed")
        if any(host):
            dt = _torch_dtype(bufs[0].dtype)
            if any(_torch_dtype(b.dtype) != dt for b in bufs):
                raise SimulationError(f"module {key}: buffer dtypes differ across devices")
            dev_bufs = []
            for d, b in zip(members, bufs):
                t = torch.from_numpy(np.ascontiguousarray(b)).to("cuda", dt)
                staged[(d.index, key)] = t
                dev_bufs.append(t)
        else:
            dev_bufs = bufs
            dt = bufs[0].dtype
        ref = dev_bufs[0]
        for b in dev_bufs:
            if b.dtype not in (torch.float32, torch.float64) or not b.is_cuda or not b.is_contiguous():
                raise SimulationError("buffers must be contiguous float32 / float64 tensors")
            if b.dtype != ref.dtype:
                raise SimulationError(f"module {key}: buffer dtypes differ across devices")
            if b.shape != ref.shape:
                raise SimulationError(f"module {key}: buffer shapes differ across devices")
            if b.device != ref.device:
                # the one-launch exchange reads every member's buffer from the
                # launching GPU; real ranks exchange through engine.CommGroups
                # (NCCL) or peer.PeerExchange instead
                raise SimulationError(f"module {key}: buffers on different CUDA devices")
        out = torch.empty_like(ref)
        synced[key] = out
        if any(host):
            host_out[key] = members
        m = _native.SyncModule()
        for r, b in enumerate(dev_bufs):
            m.bufs[r] = b.data_ptr()
        m.out = out.data_ptr()
        m.n_elems = ref.numel()
        m.group_size = len(members)
        m.used_mask = sum(1 << r for r, d in enumerate(members) if key in d.used)
        tables[ref.dtype].append(m)
    for dt, table in tables.items():
        if table:
            ops.sync_emulated(table, only_ready, f64=dt == torch.float64)
    for key, members in host_out.items():
        val = synced[key].cpu().numpy()
        synced[key] = val
        if any(key in d.used for d in members):  # n >= 1: install on every member
            for d in members:
                d.buffers[key] = val.copy()
    return synced


class Reservoir:
    """Single-pass reservoir sample (syncsim.py:208-227)."""

    def __init__(self, capacity: int, seed: int = 0):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        self.capacity = capacity
        self._rng = random.Random(seed)
        self._seen = 0
        self.items: list = []

    def add(self, item) -> None:
        self._seen += 1
        if len(self.items) < self.capacity:
            self.items.append(item)
            return
        j = self._rng.randrange(self._seen)
        if j < self.capacity:
            self.items[j] = item


def reservoir_batch(stream: Iterable, capacity: int, seed: int = 0) -> list:
    res = Reservoir(capacity, seed)
    for item in stream:
        res.add(item)
    return res.items


def ring_allreduce_time(payload_bytes: float, group: int, alpha: float, beta: float) -> float:
    """2(g-1) alpha + 2(g-1)/g * bytes / beta (syncsim.py:237-242)."""
    if group < 2:
        return 0.0
    return 2 * (group - 1) * alpha + 2 * (group - 1) / group * payload_bytes / beta


@dataclasses.dataclass
class StepRecord:
    step: int
    ready_bytes: int
    grad_bytes: int
    comm_time: float
    compute_time: float
    tokens: int


@dataclasses.dataclass
class CommLedger:
    """Per-step accounting (syncsim.py:245-292); times here are measured
    (CUDA events), the byte columns follow the reference's definitions."""

    records: list = dataclasses.field(default_factory=list)

    @property
    def total_tokens(self) -> int:
        return sum(r.tokens for r in self.records)

    @property
    def total_time(self) -> float:
        return sum(r.comm_time + r.compute_time for r in self.records)

    @property
    def total_grad_bytes(self) -> int:
        return sum(r.grad_bytes for r in self.records)

    @property
    def total_ready_bytes(self) -> int:
        return sum(r.ready_bytes for r in self.records)

    @property
    def comm_fraction(self) -> float:
        t = self.total_time
        return sum(r.comm_time for r in self.records) / t if t > 0 else 0.0

    @property
    def tokens_per_sec(self) -> float:
        t = self.total_time
        return self.total_tokens / t if t > 0 else 0.0

    def to_tsv(self) -> str:
        rows = ["step\tready_bytes\tgrad_bytes\tcomm_time\tcompute_time\ttokens"]
        rows += [f"{r.step}\t{r.ready_bytes}\t{r.grad_bytes}\t{r.comm_time:.9e}"
                 f"\t{r.compute_time:.9e}\t{r.tokens}" for r in self.records]
        return "\n".join(rows) + "\n"


SCALING_ARCHS = ("independent", "partially_shared", "fully_shared")


def synthetic_uniform_tasks(arch_kind: str, n_gpus: int, topo: ClusterTopology) -> list[TaskSpec]:
    """One self-pair task per GPU under the paper's three sharing schemes
    (syncsim.py:412-458)."""
    SP = SharingPattern
    archs = {
        "independent": ArchSpec(((SP.LANGUAGE, 6),), ((SP.LANGUAGE, 6),)),
        "partially_shared": ArchSpec(((SP.LANGUAGE, 4), (SP.FULL, 4)), ((SP.LANGUAGE, 4),)),
        "fully_shared": ArchSpec(((SP.FULL, 9),), ((SP.FULL, 4),)),
    }
    if arch_kind not in archs:
        raise ValueError(f"unknown architecture kind: {arch_kind}")
    devices = topo.devices()
    if n_gpus > len(devices):
        raise ValueError("more tasks than GPUs in topology")
    out = []
    for i in range(n_gpus):
        lang = f"l{i:02d}"
        enc, dec, el, dl = build_module_sequence(archs[arch_kind], lang, lang)
        out.append(TaskSpec(id=task_id(lang, lang), src_lang=lang, tgt_lang=lang,
                            src_path=f"synthetic/{lang}.src", tgt_path=f"synthetic/{lang}.tgt",
                            enc_modules=enc, dec_modules=dec, enc_layers=el, dec_layers=dl,
                            device=devices[i]))
    return out


# ---------------------------------------------------------------------------
# the trainer loop and the optimizer hook behind the reference's API


def step_optimizer(module_buckets: Mapping, ready_counts: Mapping, adam=None) -> None:
    """The optimizer hook SURVEY §8(b) adds to the reference's API: one fused
    ``/ n`` + Adam + bf16-cast launch (K3, ``mm_fused_update``) over every
    module bucket whose ready count n >= 1; n == 0 leaves the module untouched
    (``grad = None`` semantics: no moment decay, no step count).  Buckets are
    ``model.ModuleState`` objects (grad, master, exp_avg, exp_avg_sq, weights,
    step) keyed by ModuleKey; the gradient must already be the group sum."""
    import math
    from .engine import AdamConfig
    a = adam or AdamConfig()
    mods = []
    for key, st in module_buckets.items():
        n = int(ready_counts.get(key, 0))
        if n < 1:
            continue
        st.step += 1
        mods.append(_native.AdamModule(
            grad=st.grad.data_ptr(), master=st.master.data_ptr(), exp_avg=st.exp_avg.data_ptr(),
            exp_avg_sq=st.exp_avg_sq.data_ptr(), param_bf16=st.weights.data_ptr(),
            n_elems=st.master.numel(), n_ready=n, ready_index=-1,
            step_size=a.lr / (1.0 - a.beta1 ** st.step),
            inv_sqrt_bc2=1.0 / math.sqrt(1.0 - a.beta2 ** st.step)))
    if mods:
        ops.fused_update(mods, _native.AdamHyper.make(beta1=a.beta1, beta2=a.beta2, eps=a.eps,
                                                      weight_decay=a.weight_decay))


def run_benchmark(tasks: Sequence[TaskSpec], topo: ClusterTopology, steps: int, seed: int = 0,
                  accum_count: int = 1, dim: int = 4, batch_tokens: int = 4096,
                  compute_coeff: float = 2e-9, shape=None, device=None, timing: str = "measured"):
    """``run_benchmark`` (syncsim.py:295-392) with the toy model replaced by
    the real modular transformer: every device of ``topo`` that holds a task
    is an emulated rank on this GPU (``cluster.EmulatedCluster``); each step
    every rank draws ``accum_count`` micro-batches of ``batch_tokens`` target
    tokens through the multiplexer (``Random(f"{seed}:{i}:mux")``, data
    ``default_rng([seed, i])``), runs forward / backward, then the Algorithm-1
    exchange and the fused update.

    Ledger columns: ``ready_bytes`` / ``grad_bytes`` / ``tokens`` follow the
    reference's definitions exactly (module sizes in the reference's
    enumerate_modules convention, syncsim.py:318, 365-379).  Times:

    * ``timing="measured"``: CUDA events.  ``compute_time`` = max over ranks
      of that rank's forward / backward plus its own K3 update (each rank
      would run on its own GPU); ``comm_time`` = the cross-rank exchange
      (one mm_sync_emulated launch over every shared module; with option B
      the fused exchange + update).  ``dim`` and ``compute_coeff`` unused.
    * ``timing="modeled"``: the reference's own cost model on the same run --
      compute = compute_coeff * batch_tokens * layers per micro-batch (max
      over devices), comm = the ring model per group with the link class it
      spans (syncsim.py:355-392) -- so E(k) equals the reference's.

    Returns (CommLedger, summary dict with the reference's keys)."""
    if timing not in ("measured", "modeled"):
        raise ValueError(f"unknown timing {timing!r}")
    import numpy as np
    from . import configs
    from .cluster import EmulatedCluster
    from .data import ZipfIds, make_batch
    from .engine import DeviceBatch
    from .plan import task_modules
    from .sharing import enumerate_modules
    tasks = sorted(tasks, key=lambda t: t.id)
    for t in tasks:
        if t.device is None:
            raise SimulationError(f"task {t.id} has no device assignment")
    shape = shape or configs.SHAPE_CFG1_GPU
    dev = torch.device(device or f"cuda:{torch.cuda.current_device()}")
    modules = enumerate_modules(tasks)
    world = max(topo.flat(t.device) for t in tasks) + 1
    cl = EmulatedCluster(tasks, topo, shape, world=world, device=dev, seed=seed)
    plan = cl.plan
    spec = configs.DataSpec(batch_tokens, 3.0, 0.5, 4, shape.max_len, 1.1)
    ids = ZipfIds(shape.vocab, spec.zipf_s)
    ranks = sorted(plan.tasks_by_rank)
    data_rngs = {i: np.random.default_rng([seed, i]) for i in ranks}
    ledger = CommLedger()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    layers = {t.id: sum(t.enc_layers) + sum(t.dec_layers) for t in tasks}
    node_of = {i: i // topo.n_gpus_per_node for i in ranks}
    for step in range(steps):
        used_by_rank, comp, modeled = {}, {}, {}
        step_tokens = 0
        for i in ranks:
            eng = cl.ranks[i]
            ops.memset(eng.loss_sum, 0)
            used: set = set()
            e0, e1 = ev(), ev()
            e0.record()
            modeled[i] = 0.0
            for _ in range(accum_count):
                task = eng.mux.pick(step)
                b = make_batch(data_rngs[i], spec, shape.vocab, ids=ids)
                fresh = [k for k in task_modules(task) if k not in used]
                eng.zero_grads(fresh)
                used.update(fresh)
                eng.forward_backward(task, DeviceBatch(b, dev), eng.loss_sum)
                step_tokens += batch_tokens
                modeled[i] += compute_coeff * batch_tokens * layers[task.id]
            e1.record()
            used_by_rank[i] = used
            comp[i] = [(e0, e1)]
        c0, c1 = ev(), ev()
        c0.record()
        counts = cl.exchange(used_by_rank)
        c1.record()
        if cl.exchange_kind != "peer":
            for i in ranks:
                u0, u1 = ev(), ev()
                u0.record()
                cl.update_rank(i, counts)
                u1.record()
                comp[i].append((u0, u1))
        torch.cuda.synchronize(dev)
        idx = plan.index()
        ready_bytes = grad_bytes = 0
        comm_model = 0.0
        for key in sorted(modules):
            group = plan.groups.get(key, [])
            g = len(group)
            if g < 2:
                continue
            spans = len({node_of[i] for i in group}) > 1
            alpha = topo.alpha_inter if spans else topo.alpha_intra
            beta = topo.beta_inter if spans else topo.beta_intra
            ready_bytes += READY_ENTRY_BYTES * g
            comm_model += ring_allreduce_time(READY_ENTRY_BYTES, g, alpha, beta)
            if counts[idx[key]] >= 1:
                payload = GRAD_BYTES_PER_PARAM * modules[key].n_params
                grad_bytes += payload
                comm_model += ring_allreduce_time(payload, g, alpha, beta)
        if timing == "modeled":
            comm_t = comm_model
            comp_t = max(modeled.values()) if modeled else 0.0
        else:
            comm_t = c0.elapsed_time(c1) * 1e-3
            comp_t = max(sum(a.elapsed_time(b) for a, b in v) for v in comp.values()) * 1e-3 if comp else 0.0
        ledger.records.append(StepRecord(step=step, ready_bytes=ready_bytes, grad_bytes=grad_bytes,
                                         comm_time=comm_t, compute_time=comp_t, tokens=step_tokens))
    summary = {
        "steps": steps, "devices": len(ranks), "tasks": len(tasks), "modules": len(modules),
        "total_tokens": ledger.total_tokens, "total_time_sec": ledger.total_time,
        "tokens_per_sec": ledger.tokens_per_sec, "comm_time_fraction": ledger.comm_fraction,
        "grad_allreduce_bytes": ledger.total_grad_bytes, "ready_sync_bytes": ledger.total_ready_bytes,
    }
    return ledger, summary



def scaling_experiment(arch_kind: str, gpu_counts: Sequence[int], n_gpus_per_node: int = 4,
                       steps: int = 5, seed: int = 0, **benchmark_kwargs) -> dict:
    """E(k) = throughput(k) / (k * throughput(1)) of the uniform workload
    (one task per GPU, ``synthetic_uniform_tasks``), syncsim.py:461-483, over
    this package's run_benchmark (the real engine; pass timing="modeled"
    for the reference's cost model, timing="measured" for CUDA-event
    times of the emulated ranks)."""

    def throughput(k: int) -> float:
        n_nodes = max(1, -(-k // n_gpus_per_node))
        topo = ClusterTopology(n_nodes=n_nodes, n_gpus_per_node=n_gpus_per_node, n_slots_per_gpu=1)
        tasks = synthetic_uniform_tasks(arch_kind, k, topo)
        ledger, _ = run_benchmark(tasks, topo, steps=steps, seed=seed, **benchmark_kwargs)
        return ledger.tokens_per_sec

    base = throughput(1)
    return {k: throughput(k) / (k * base) for k in gpu_counts}
