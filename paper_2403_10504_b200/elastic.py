"""Elastic peers: a DHT-style progress registry, the global-batch averaging trigger, and churn
(peers failing, leaving and joining mid-run).  SURVEY NEXT-3; R36.

PAPER P:410: every peer "periodically publish[es] its status to the DHT via a heartbeat message"
carrying the number of mini-batches it processed; "once the global batch size is reached" the
peers average parameters with an allreduce; peers join and leave at any time.  P:563 kills two to
four GPUs mid-training and training completes.

B200 reading (R36).  The registry is one logical key-value store with TTL semantics (SPEC S:407:
membership / progress registry, no Kademlia routing) over a `torch.distributed.TCPStore`; a peer
is live while its newest heartbeat is younger than `ttl` seconds.  Peers train in lockstep steps;
at every step boundary each member publishes (step, sequences processed since the last averaging
round) and waits until every member has published that step or gone stale.  The lowest live
member (the leader) then writes the boundary's decision first-writer-wins (`compare_set`), so all
members apply the same one even when the leader itself dies mid-decision:

* membership: stale members are dropped (their communicator ranks excluded with
  `ncclCommShrink`, `atom_comm_shrink`); registered joiners are admitted (a fresh communicator,
  `atom_comm_reset`, then `atom_broadcast_state` from the leader: a joiner adopts the leader's
  master, AdamW moments and step count, "fetch the current model");
* trigger: when the live members' counts sum to >= the global batch the NEXT step is a sync step
  (the allreduce runs fused into its backward swap window, `atom_sync(flush=0)`); the counts restart
  after it.  Sequences processed by a peer that dies before its round is averaged are lost (the
  conservation ledger of SPEC S:393-398).

This module is host logic only: it never touches the device itself; `apply()` calls the C-ABI
through a `Peer` (atom.Peer) or any object with the same four methods.
"""
from __future__ import annotations

import dataclasses
import json
import threading
import time
from typing import Callable, List, Optional


@dataclasses.dataclass
class Decision:
    s: int                  # step boundary (after step s)
    epoch: int              # membership epoch (changes whenever the member set does)
    prev: List[int]         # members before the decision (communicator ranks = positions)
    members: List[int]      # members after it
    dead: List[int]         # stale members dropped
    joiners: List[int]      # admitted joiners
    leader: int
    sync: bool              # the next step averages parameters
    total: int              # sequences the live members processed since the last round
    counts: dict            # per live member
    nccl_id: Optional[str]  # hex id of the new communicator (joiners admitted)
    join_seen: int          # join tickets consumed so far

    def to_json(self) -> str:
        return json.dumps(dataclasses.asdict(self), sort_keys=True)

    @staticmethod
    def from_json(s: str) -> "Decision":
        d = json.loads(s)
        d["counts"] = {int(k): v for k, v in d["counts"].items()}
        return Decision(**d)


class _LockedStore:
    """The store shared by the protocol thread and the heartbeat thread: one call at a time."""

    def __init__(self, store):
        self._s, self.lock = store, threading.RLock()

    def __getattr__(self, name):
        fn = getattr(self._s, name)

        def call(*a, **k):
            with self.lock:
                return fn(*a, **k)
        return call


class Registry:
    """Heartbeats with TTL over a store (set / get / check / add / compare_set)."""

    def __init__(self, store, ttl: float, clock: Callable[[], float] = time.time):
        self.store, self.ttl, self.clock = store, ttl, clock

    def beat(self, pid: int, s: int, count: int):
        self.store.set(f"hb/{pid}", json.dumps({"s": s, "count": count, "t": self.clock()}))

    def read(self, pid: int) -> Optional[dict]:
        if not self.store.check([f"hb/{pid}"]):
            return None
        return json.loads(self.store.get(f"hb/{pid}"))

    def fresh(self, rec: Optional[dict]) -> bool:
        return rec is not None and self.clock() - rec["t"] <= self.ttl


class Coordinator:
    """One peer's side of the protocol.

    store: a torch.distributed Store shared by all peers (TCPStore on 127.0.0.1 for one box);
    pid: this peer's id (unique, never reused); global_batch: sequences per averaging round
    (512); ttl: heartbeat lifetime in seconds; make_id: returns a fresh 128-byte NCCL
    unique id (atom.atom_nccl_unique_id) -- only the leader calls it."""

    def __init__(self, store, pid: int, global_batch: int, ttl: float = 10.0, poll: float = 0.005,
                 make_id: Optional[Callable[[], bytes]] = None, clock: Callable[[], float] = time.time,
                 boot_grace: Optional[float] = None):
        self.store, self.pid, self.global_batch = _LockedStore(store), pid, global_batch
        # a member that has never heartbeated (still starting up) is declared dead only after
        # boot_grace; one whose heartbeat went stale, after ttl
        self.boot_grace = max(30.0, 4 * ttl) if boot_grace is None else boot_grace
        self.reg = Registry(self.store, ttl, clock)
        self.poll, self.make_id, self.clock = poll, make_id, clock
        self.members: List[int] = []
        self.epoch = 0
        self.count = 0
        self.join_seen = 0
        self.sync_step = False     # the step being run averages parameters
        self.s = -1                # last completed step
        # heartbeats run for the peer's whole life on a background thread ("periodically"),
        # not only between steps: a step longer than the TTL must not make a live member stale
        self._hb_stop = threading.Event()
        self._hb_thread: Optional[threading.Thread] = None

    # ---------------------------------------------------------------- heartbeats
    def _beat(self):
        # (s, count) read and published under the store lock: a beat never regresses s
        with self.store.lock:
            self.reg.beat(self.pid, self.s, self.count)

    def _start_heartbeat(self):
        if self._hb_thread is not None:
            return
        self._beat()

        def run():
            while not self._hb_stop.wait(self.reg.ttl / 4):
                self._beat()
        self._hb_thread = threading.Thread(target=run, name=f"atom-heartbeat-{self.pid}", daemon=True)
        self._hb_thread.start()

    def stop(self):
        """Stop heartbeating (graceful leave / shutdown)."""
        self._hb_stop.set()
        if self._hb_thread is not None:
            self._hb_thread.join()
            self._hb_thread = None

    # ---------------------------------------------------------------- membership bootstrap
    def start(self, members: List[int]):
        """Initial members (known to all of them, e.g. the torchrun world)."""
        self.members = sorted(members)
        self.s = -1
        self._start_heartbeat()

    def join(self, timeout: float = 600.0) -> Decision:
        """Register as a joiner and wait to be admitted at some step boundary."""
        self._start_heartbeat()
        ticket = self.store.add("join_n", 1) - 1
        self.store.set(f"join/{ticket}", str(self.pid))
        t0 = self.clock()
        while not self.store.check([f"admit/{self.pid}"]):
            if self.clock() - t0 > timeout:
                raise TimeoutError(f"peer {self.pid}: not admitted within {timeout} s")
            time.sleep(self.poll)
        d = Decision.from_json(self.store.get(f"admit/{self.pid}").decode())
        self._adopt(d)
        self.count = 0
        return d

    # ---------------------------------------------------------------- per step boundary
    def after_step(self, processed: int) -> Decision:
        """Called by every member after each step with the sequences it processed in it.

        Waits until every other member has published this step (ready) or gone stale (dead: no
        heartbeat within ttl; every live member's heartbeat thread keeps it fresh, also while it
        is still inside a long step), then the lowest ready member writes the decision unless one
        exists already.  Joiners are admitted from the STORED decision (read back after the
        first-writer-wins compare_set, by every member, idempotently): a joiner never sees a
        decision other than the canonical one, even when the leader dies right after deciding."""
        with self.store.lock:
            self.s += 1
            s = self.s
            # a sync step closes the averaging round: its samples are in the averaged parameters
            self.count = 0 if self.sync_step else self.count + processed
            self.reg.beat(self.pid, s, self.count)
        if self._hb_thread is None:
            self._start_heartbeat()
        key = f"dec/{s}"
        t0 = self.clock()
        while not self.store.check([key]):
            now = self.clock()
            recs = {m: self.reg.read(m) for m in self.members if m != self.pid}
            ready, waiting = [self.pid], False
            for m, r in recs.items():
                if r is not None and self.reg.fresh(r) and r["s"] >= s:
                    ready.append(m)
                elif not ((r is None and now - t0 > self.boot_grace) or (r is not None and not self.reg.fresh(r))):
                    waiting = True
            if not waiting and min(ready) == self.pid:
                self.store.compare_set(key, "", self._decide(s, sorted(ready), recs).to_json())
                break
            time.sleep(self.poll)
        d = Decision.from_json(self.store.get(key).decode())
        for j in d.joiners:
            self.store.set(f"admit/{j}", d.to_json())
        self._adopt(d)
        return d

    def _decide(self, s: int, alive: List[int], recs: dict) -> Decision:
        counts = {m: (self.count if m == self.pid else recs[m]["count"]) for m in alive}
        total = sum(counts.values())
        n = int(self.store.add("join_n", 0))
        joiners, seen = [], self.join_seen
        for i in range(self.join_seen, n):       # tickets in order; stop at one not yet written
            if not self.store.check([f"join/{i}"]):
                break
            joiners.append(int(self.store.get(f"join/{i}").decode()))
            seen = i + 1
        dead = [m for m in self.members if m not in alive]
        members = sorted(alive + joiners)
        changed = members != self.members
        nid = self.make_id().hex() if joiners and self.make_id else None
        d = Decision(s=s, epoch=self.epoch + (1 if changed else 0), prev=list(self.members), members=members,
                     dead=dead, joiners=joiners, leader=self.pid, sync=total >= self.global_batch, total=total,
                     counts=counts, nccl_id=nid, join_seen=seen)
        return d

    def _adopt(self, d: Decision):
        self.members, self.epoch, self.join_seen = list(d.members), d.epoch, d.join_seen
        self.s = d.s
        self.sync_step = d.sync

    # ---------------------------------------------------------------- apply to a peer
    def apply(self, d: Decision, peer, atom_sync: Optional[Callable] = None):
        """Rebuild the averaging communicator and admit joiners (collective over d.members),
        then mark the next step as a sync step when the trigger fired."""
        if self.pid not in d.members:
            raise RuntimeError(f"peer {self.pid} is not a member after step {d.s}")
        if d.joiners:
            peer.comm_reset(bytes.fromhex(d.nccl_id), len(d.members), d.members.index(self.pid))
            peer.broadcast_state(d.members.index(d.leader), self.pid in d.joiners)
        elif d.dead:
            # the dead peer may have left this peer's averaging round waiting inside the device
            # stream: abort the outstanding operations, then shrink (the guarded commit keeps the
            # local master for a round that did not complete on every rank, R36)
            peer.comm_shrink([d.prev.index(m) for m in d.dead], abort_ops=True)
        if d.sync and atom_sync is not None and len(d.members) > 1:
            atom_sync([peer], flush=False)

    def leave(self):
        """Graceful leave: stop heartbeating; the others drop this peer after one TTL."""
        self.stop()
        self.store.set(f"hb/{self.pid}", json.dumps({"s": self.s, "count": 0, "t": 0.0}))
