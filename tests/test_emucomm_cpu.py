"""The emulated communicator's matching logic on the CPU (emucomm.EmuHub):
collectives complete when every member posted them, matched per tag and
per-rank call order; the last poster executes; errors reach every member;
overlapping member sets posted in sorted order do not deadlock."""
import threading

import pytest

from paper_2403_07544_b200 import configs
from paper_2403_07544_b200.emucomm import EmuHub
from paper_2403_07544_b200.plan import build_plan


def _hub(world=3):
    w = configs.config3(world)
    return EmuHub(world, build_plan(w.tasks, w.topo))


def test_matching_and_last_poster_executes():
    hub = _hub()
    runs, got = [], {}

    def execute(reqs):
        runs.append(sorted(reqs))
        for r, box in reqs.items():
            box.append(sum(x[0] for x in reqs.values()))

    def rank(r):
        out = []
        for i in range(3):  # three calls of the same tag: matched in call order
            box = [r * 10 + i]
            hub.wait(hub.post(r, "t", (0, 1, 2), box, execute))
            out.append(box[-1])
        got[r] = out

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(10)
    assert runs == [[0, 1, 2]] * 3
    assert got[0] == got[1] == got[2] == [30, 33, 36]
    assert not hub.slots


def test_overlapping_groups_in_sorted_order_complete():
    hub = _hub(4)
    done = []
    groups = [("a", (0, 1)), ("b", (1, 2)), ("c", (2, 3)), ("d", (0, 3))]

    def rank(r):
        keys = [hub.post(r, tag, m, None, lambda reqs: None) for tag, m in groups if r in m]
        for k in keys:
            hub.wait(k)
        done.append(r)

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(10)
    assert sorted(done) == [0, 1, 2, 3]


def test_execute_error_reaches_every_member():
    hub = _hub(2)
    errs = []

    def boom(reqs):
        raise ValueError("bad collective")

    def rank(r):
        try:
            hub.wait(hub.post(r, "x", (0, 1), None, boom))
        except ValueError as e:
            errs.append((r, str(e)))

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(10)
    assert sorted(errs) == [(0, "bad collective"), (1, "bad collective")]


def test_member_set_mismatch_rejected():
    hub = _hub(3)
    hub.post(0, "y", (0, 1), None, lambda reqs: None)
    with pytest.raises(RuntimeError):
        hub.post(1, "y", (1, 2), None, lambda reqs: None)
