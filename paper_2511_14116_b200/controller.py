"""World management of a FailSafe serving cluster (host side).

The decision half of the reference's reconfiguration orchestration
(``Simulation._desired_serving`` / ``_reconfigure`` / ``_route_for`` /
``_adopt_plan`` / ``_recompute_usage`` / ``_evict_over_capacity`` /
``_preempt`` / ``_admit``, simulation.py:198-446) restated on real request
objects, so an executing cluster (``failover.EmulatedCluster``,
``cluster.ClusterRank``) takes exactly the reference's decisions:

* which GPUs serve (``ReconfigPolicy``, recovery.py:35-54, capped by the
  world limit);
* the target placement: on-demand shrink (survivors keep their state,
  recovery.py:396-427) or, when a GPU rejoins, a fresh placement of the
  expanded world that every GPU reloads from host (recovery.py:366-394);
* re-routing of residents (a request keeps its rank when it survived) and
  the router rebuilt in arrival order;
* KV capacity per GPU (HBM minus the plan's weights) and the full-lifetime
  reservations; over capacity after a shrink, the latest arrivals are
  preempted (progress reset, back to the arrival-ordered waiting line);
* admission of waiting requests under the reservation invariant.

One deliberate difference: a preempted request is also withdrawn from the
rebuilt router's prefill queue (and its pending cost from the rank's
workload).  The reference leaves it queued, and its next iteration fails
with a KeyError on the request's routing (simulation.py:255-262 vs 458-462;
pinned in tests/golden/reconfig.json).
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass
from typing import Optional

from .core import ClusterSpec, ModelSpec, Request, SimulationError
from .failover import route_for
from .placement import make_placement, weight_bytes_per_gpu
from .recovery import (BackupState, ReconfigPolicy, merge_plans, plan_kv_recovery,
                       plan_weight_recovery)
from .scheduler import DEFAULT_KAPPA, SchedulerState, request_pending_cost, route_request


@dataclass
class Decision:
    """One reconfiguration (simulation.py:323-374): the serving world, the
    target plan, the re-routing and the recovery plans to execute."""

    desired: list
    new_plan: object
    new_routing: dict
    weight_plan: object
    kv_plan: object
    merged: object


class WorldController:
    def __init__(self, model: ModelSpec, cluster: ClusterSpec, placement_mode: str = "hybrid",
                 policy: Optional[ReconfigPolicy] = None, token_budget: int = 2048,
                 kappa: float = DEFAULT_KAPPA, recovery_mode: str = "full",
                 world_limit: Optional[int] = None, backup: Optional[BackupState] = None):
        self.model, self.cluster = model, cluster
        self.placement_mode = placement_mode
        self.policy = policy or ReconfigPolicy("flexible", 1)
        self.token_budget, self.kappa = token_budget, kappa
        self.recovery_mode = recovery_mode
        self.world_limit = world_limit
        self.kv_unit = model.kv_bytes_per_head_token()
        self.alive = set(range(cluster.num_gpus))
        self.serving: list = []
        self.plan = None
        self.capacity: dict = {}
        self.tp_total: dict = {}
        self.dp_total = 0
        self.reserved: dict = {}
        self.kv_used: dict = {}
        self.pending_dp: dict = {}
        self.sched: Optional[SchedulerState] = None
        self.requests: dict = {}
        self.residents: list = []
        self.waiting: deque = deque()
        self.routing: dict = {}
        self.backup = backup if backup is not None else BackupState(
            host_memory_bytes=cluster.host_memory_bytes,
            kv_bytes_per_token=model.kv_bytes_per_token(),
            enabled=recovery_mode in ("host", "full"))
        self.preempted: list = []
        self.rejected: list = []

    # ------------------------------------------------------------ world --
    def desired_serving(self) -> Optional[list]:
        w = self.policy.world_size(len(self.alive))
        if w is None:
            return None
        if self.world_limit is not None:
            w = min(w, self.world_limit)
        return sorted(self.alive)[:w]

    @staticmethod
    def plan_arrays(plan):
        tp_total = {g: 0 for g in plan.alive}
        dp_total = 0
        for assign in plan.per_layer:
            dp_total += len(assign.dp_heads)
            for g, heads in assign.tp_heads.items():
                tp_total[g] += len(heads)
        return tp_total, dp_total

    def request_reservation(self, tokens: int, rank: int) -> dict:
        out = {}
        for g in self.serving:
            b = self.tp_total[g] * tokens * self.kv_unit
            if g == rank:
                b += self.dp_total * tokens * self.kv_unit
            out[g] = b
        return out

    def start(self) -> list:
        """Initial world: a fresh plan over the desired GPUs."""
        desired = self.desired_serving()
        if desired is None:
            raise SimulationError("no feasible serving world")
        self.plan = make_placement(self.placement_mode, self.model, desired)
        return self.adopt_plan(desired, {})

    def adopt_plan(self, serving: list, new_routing: dict) -> list:
        """``_adopt_plan`` (simulation.py:225-258): capacities, residents
        re-routed in arrival order into a rebuilt router, usage recomputed,
        over-capacity preemption.  Returns the preempted request ids."""
        self.serving = list(serving)
        if self.plan is None:
            self.plan = make_placement(self.placement_mode, self.model, serving)
        weights = weight_bytes_per_gpu(self.plan, self.model)
        self.capacity = {g: self.cluster.hbm_bytes_per_gpu - weights[g] for g in serving}
        if any(v <= 0 for v in self.capacity.values()):
            raise SimulationError("model weights exceed HBM under the adopted plan")
        self.tp_total, self.dp_total = self.plan_arrays(self.plan)
        self.sched = SchedulerState(token_budget=self.token_budget, rank_set=tuple(serving),
                                    kappa=self.kappa)
        self.routing = {}
        for rid in self.residents:
            req = self.requests[rid]
            rank = new_routing.get(rid)
            if rank is None or rank not in self.capacity:
                rank = min(self.serving, key=lambda g: (self.sched.workload[g], g))
            req.dp_rank = rank
            self.routing[rid] = rank
            self.sched._enqueue(req, rank)
        self.recompute_usage()
        first = len(self.preempted)
        self.evict_over_capacity()
        return self.preempted[first:]

    def recompute_usage(self) -> None:
        self.reserved = {g: 0 for g in self.serving}
        self.kv_used = {g: 0 for g in self.serving}
        self.pending_dp = {g: 0 for g in self.serving}
        for rid in self.residents:
            req = self.requests[rid]
            rank = self.routing[rid]
            ctx = req.context_tokens()
            for g in self.serving:
                res = self.tp_total[g] * req.final_context_tokens() * self.kv_unit
                used = self.tp_total[g] * ctx * self.kv_unit
                if g == rank:
                    res += self.dp_total * req.final_context_tokens() * self.kv_unit
                    used += self.dp_total * ctx * self.kv_unit
                self.reserved[g] += res
                self.kv_used[g] += used
            self.pending_dp[rank] += (req.input_len - req.tokens_prefilled
                                      + req.output_len - req.tokens_decoded)

    def evict_over_capacity(self) -> None:
        over = [g for g in self.serving if self.reserved[g] > self.capacity[g]]
        while over and self.residents:
            victim = max(self.residents,
                         key=lambda rid: (self.requests[rid].arrival_time, rid))
            self.preempt(victim)
            over = [g for g in self.serving if self.reserved[g] > self.capacity[g]]
        if over:
            raise SimulationError("KV capacity exceeded with no residents to preempt")

    def preempt(self, rid: int) -> None:
        """``_preempt`` (simulation.py:283-310), plus the router withdrawal
        (module doc)."""
        req = self.requests[rid]
        rank = self.routing.get(rid)
        if self.sched is not None and rank is not None:
            self.sched.workload[rank] = max(
                0.0, self.sched.workload[rank] - request_pending_cost(req, self.kappa))
            q = self.sched.schedulable[rank]
            q.spans = deque(sp for sp in q.spans if sp[0] != rid)
            self.sched.fifo_order = deque(x for x in self.sched.fifo_order if x != rid)
        self.residents.remove(rid)
        self.routing.pop(rid, None)
        self.backup.drop(rid)
        req.tokens_prefilled = 0
        req.tokens_decoded = 0
        req.dp_rank = None
        self.preempted.append(rid)
        position = 0
        for i, wid in enumerate(self.waiting):
            other = self.requests[wid]
            if (other.arrival_time, wid) > (req.arrival_time, rid):
                break
            position = i + 1
        self.waiting.insert(position, rid)
        self.recompute_usage()

    # ------------------------------------------------------- reconfigure --
    def route_for(self, serving: list) -> dict:
        return route_for(self.residents, self.requests, self.routing, serving)

    def plan_reconfigure(self) -> Optional[Decision]:
        """``_reconfigure``'s plan choice (simulation.py:323-374) for the
        current alive set; None when the world does not change or cannot
        serve."""
        desired = self.desired_serving()
        if desired is None or desired == self.serving:
            return None
        mode = "on_demand" if self.recovery_mode in ("full", "oracle") else "naive_reshard"
        wplan = plan_weight_recovery(self.model, self.plan, desired, mode)
        new_plan = wplan.target_plan(self.placement_mode, self.model)
        new_routing = self.route_for(desired)
        contexts = {rid: self.requests[rid].context_tokens() for rid in self.residents
                    if self.requests[rid].context_tokens() > 0}
        kvplan = None
        if self.recovery_mode != "oracle" and contexts:
            kv_mode = "recompute" if self.recovery_mode == "recompute" else "host_restore"
            kvplan = plan_kv_recovery(self.backup, self.plan, new_plan, self.model, contexts,
                                      self.routing, new_routing, kv_mode)
        merged = merge_plans(wplan, kvplan)
        return Decision(desired, new_plan, new_routing, wplan, kvplan, merged)

    def apply(self, decision: Decision) -> list:
        """``_handle_reconfig_done``: adopt the decided world; returns the
        preempted request ids."""
        self.plan = decision.new_plan
        return self.adopt_plan(decision.desired, decision.new_routing)

    def fail(self, gpu: int) -> Optional[Decision]:
        self.alive.discard(gpu)
        return self.plan_reconfigure()

    def rejoin(self, gpu: int) -> Optional[Decision]:
        self.alive.add(gpu)
        return self.plan_reconfigure()

    def finish(self, rid: int) -> None:
        """``_finish_request`` (simulation.py:488-513): the request leaves
        the world and releases its reservation."""
        req = self.requests[rid]
        rank = self.routing[rid]
        for g, b in self.request_reservation(req.final_context_tokens(), rank).items():
            self.reserved[g] -= b
        tb = self.request_reservation(req.context_tokens(), rank)
        for g in self.serving:
            self.kv_used[g] = self.kv_used.get(g, 0) - tb[g]
        self.pending_dp[rank] = self.pending_dp.get(rank, 0) - (
            req.input_len - req.tokens_prefilled + req.output_len - req.tokens_decoded)
        self.residents.remove(rid)
        self.routing.pop(rid, None)
        self.backup.mark_finished(rid)

    # --------------------------------------------------------- admission --
    def add_request(self, req: Request) -> None:
        self.requests[req.id] = req
        self.waiting.append(req.id)

    def admit(self) -> list:
        """``_admit`` (simulation.py:401-446, load-aware router, both
        phases): admit from the head of the waiting line while every
        serving GPU keeps its reservation under capacity."""
        admitted = []
        while self.waiting and self.serving:
            rid = self.waiting[0]
            req = self.requests[rid]
            rank = min(self.serving, key=lambda g: (self.sched.workload[g], g))
            delta = self.request_reservation(req.final_context_tokens(), rank)
            if not all(self.reserved[g] + delta[g] <= self.capacity[g] for g in self.serving):
                if not self.residents:  # can never fit: rejected, not blocking
                    self.waiting.popleft()
                    self.rejected.append(rid)
                    continue
                break
            self.waiting.popleft()
            route_request(self.sched, req)
            self.routing[rid] = req.dp_rank
            self.residents.append(rid)
            for g in self.serving:
                self.reserved[g] += delta[g]
            self.pending_dp[req.dp_rank] = self.pending_dp.get(req.dp_rank, 0) + \
                req.input_len + req.output_len
            admitted.append(rid)
        return admitted
