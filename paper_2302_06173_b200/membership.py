"""Failure detection and communicator repair (PAPER §3
"A machine failure can be detected by catching communication errors ... a
replacement machine will be added to the training job").

Plumbing around the recovery hot path, kept small:

* every rank publishes a heartbeat counter in a key-value store (the job's
  TCPStore) from a daemon thread; a detector thread declares a peer failed
  when its counter stops advancing for `timeout` seconds (the fail-stop model
  of SPEC:253: a dead process never comes back);
* on a failure the survivors abort the old process group (NCCL communicators
  are aborted, not torn down collectively: a dead peer would hang that) and
  the lowest surviving rank publishes the repair plan for the next
  generation: the same world size, survivors keep their ranks, replacements
  claim the failed ranks' slots with an atomic store counter;
* everyone then joins generation g+1 through a PrefixStore, so keys of the
  dead generation never collide with the new one.

The resolver / replication / replay entry points then run unchanged on the
new group (recovery.resolve -> recover).
"""
from __future__ import annotations

import json
import threading
import time
from dataclasses import dataclass, field

import torch.distributed as dist


def _key(*parts) -> str:
    return "/".join(str(p) for p in parts)


@dataclass
class RepairPlan:
    generation: int
    world: int
    failed: list[int]
    survivors: list[int] = field(default_factory=list)


class Membership:
    """Heartbeat + detector for one rank of generation `generation`."""

    def __init__(self, store, rank: int, world: int, generation: int = 0, interval: float = 0.05,
                 timeout: float = 1.0, grace: float = 30.0):
        self.store, self.rank, self.world, self.gen = store, rank, world, generation
        self.interval, self.timeout, self.grace = interval, timeout, grace
        self._stop = threading.Event()
        self.failure = threading.Event()
        self.failed: set[int] = set()
        self.detected_at: float | None = None
        self._beat = 0
        self.store.set(_key("hb", self.gen, self.rank), "0")
        self._threads = [threading.Thread(target=self._heartbeat, daemon=True),
                         threading.Thread(target=self._detect, daemon=True)]
        for t in self._threads:
            t.start()

    # ---- threads ----
    def _heartbeat(self):
        while not self._stop.is_set():
            self._beat += 1
            try:
                self.store.set(_key("hb", self.gen, self.rank), str(self._beat))
            except Exception:  # store gone: nothing left to report to
                return
            self._stop.wait(self.interval)

    def _detect(self):
        last = {r: (None, time.monotonic()) for r in range(self.world) if r != self.rank}
        while not self._stop.is_set():
            now = time.monotonic()
            for r in list(last):
                try:
                    v = self.store.get(_key("hb", self.gen, r)).decode() if self.store.check(
                        [_key("hb", self.gen, r)]) else None
                except Exception:
                    v = None
                prev, since = last[r]
                # a peer that never beat yet gets a start-up grace period
                limit = self.timeout if prev is not None else self.grace
                if v != prev:
                    last[r] = (v, now)
                elif now - since > limit:
                    self.failed.add(r)
                    del last[r]
                    if self.detected_at is None:
                        self.detected_at = time.time()
                    self.failure.set()
            self._stop.wait(self.interval)

    def stop(self):
        self._stop.set()
        for t in self._threads:
            t.join(timeout=2.0)

    # ---- repair ----
    def wait_failure(self, timeout: float | None = None) -> set[int]:
        self.failure.wait(timeout)
        return set(self.failed)

    def publish_plan(self, settle: float | None = None) -> RepairPlan:
        """Survivors: agree on the failed set (each publishes its view; the
        lowest surviving rank merges them after a short settle time) and
        return the plan of generation g+1."""
        settle = self.timeout if settle is None else settle
        self.store.set(_key("view", self.gen, self.rank), json.dumps(sorted(self.failed)))
        alive = [r for r in range(self.world) if r not in self.failed]
        if self.rank == min(alive):
            time.sleep(settle)  # late detections of a simultaneous second failure
            failed = set(self.failed)
            for r in alive:
                k = _key("view", self.gen, r)
                if self.store.check([k]):
                    failed |= set(json.loads(self.store.get(k)))
            plan = RepairPlan(self.gen + 1, self.world, sorted(failed),
                              [r for r in range(self.world) if r not in failed])
            self.store.set(_key("plan", self.gen), json.dumps(plan.__dict__))
        self.store.wait([_key("plan", self.gen)])
        return RepairPlan(**json.loads(self.store.get(_key("plan", self.gen))))


def abort_group(group=None) -> None:
    """Tear the old process group down without a collective (a dead peer
    would never answer): ProcessGroupNCCL aborts its communicators."""
    if not (dist.is_available() and dist.is_initialized()):
        return
    abort = getattr(dist.distributed_c10d, "_abort_process_group", None)
    try:
        if abort is not None:
            abort(group) if group is not None else abort()
        else:  # pragma: no cover - older torch
            dist.destroy_process_group(group)
    except Exception:
        pass
    if dist.is_initialized() and group is None:
        try:
            dist.destroy_process_group()
        except Exception:
            pass


def join_generation(store, plan: RepairPlan, rank: int, backend: str, timeout_s: float = 120.0, **kw):
    """Initialise the default process group of generation plan.generation."""
    import datetime
    pstore = dist.PrefixStore(f"gen{plan.generation}", store)
    dist.init_process_group(backend, store=pstore, rank=rank, world_size=plan.world,
                            timeout=datetime.timedelta(seconds=timeout_s), **kw)


def claim_slot(store, generation: int, timeout: float = 60.0) -> tuple[RepairPlan, int]:
    """Replacement: wait for the plan of `generation` (the one that failed)
    and claim one failed rank's slot (atomic counter per generation)."""
    store.wait([_key("plan", generation)], __import__("datetime").timedelta(seconds=timeout))
    plan = RepairPlan(**json.loads(store.get(_key("plan", generation))))
    i = store.add(_key("claim", plan.generation), 1) - 1
    if i >= len(plan.failed):
        raise RuntimeError("no free slot in the repair plan")
    return plan, plan.failed[i]
