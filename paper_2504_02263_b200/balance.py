"""Expert load balancing with replicated hot experts.

The paper balances expert nodes by minimising the maximum node cost
C_j = sum_i x_ij * max(a_i, K) with a greedy; the
reference's SPEC fixes the greedy (module ``balance``):

* ``node_cost(x, loads, k_cold)``
* ``balance_experts(loads, n, k_cold, mode)`` SPEC.md:407-414 -- LPT; in
  replicated mode experts whose effective cost exceeds the running average
  Sum/N are split evenly across up to R replicas, the rest assigned LPT.

``SlotPlacement`` turns a placement into what the B200 runtime executes:
``P`` physical expert slots, ``P_l`` per expert GPU (contiguous), a
logical->replica table consumed by ``msi_gate_topk_placed`` (token t of
sender s goes to replica (t + s) mod nrep -- the even split the placement
assumes) and the logical expert behind every slot (whose weights it holds).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

MODES = ("integral", "replicated", "fractional")


def node_cost(x, loads, k_cold: float = 0.0) -> np.ndarray:
    """C_j = sum_i x[i, j] * max(a_i, K_cold)."""
    x = np.asarray(x, dtype=np.float64)
    eff = np.maximum(np.asarray(loads, dtype=np.float64), k_cold)
    return eff @ x


def balance_experts(loads, n: int, k_cold: float = 0.0, mode: str = "integral",
                    max_replicas: int = 2) -> np.ndarray:
    """Greedy placement x[E, N] minimising max_j C_j approximately.

    integral: LPT (largest effective cost first onto the least-loaded node,
    ties to the lowest node).  replicated: experts above the running average
    are split evenly over up to ``max_replicas`` distinct nodes (least loaded
    first), the rest LPT.  fractional: exact water-filling (every node ends at
    the average)."""
    if mode not in MODES:
        raise ValueError(f"mode must be one of {MODES}")
    if n < 1:
        raise ValueError("need at least one node")
    a = np.maximum(np.asarray(loads, dtype=np.float64), k_cold)
    E = a.size
    if E == 0:
        raise ValueError("loads must be non-empty")
    x = np.zeros((E, n))
    if mode == "fractional":
        # water-filling: walk experts in order, pouring each into the nodes
        # up to the common level avg (exact, every node ends at avg)
        avg = a.sum() / n
        j, room = 0, avg
        for i in range(E):
            left = a[i]
            if left == 0:
                x[i, min(j, n - 1)] = 1.0
                continue
            while left > 1e-15 * max(avg, 1.0) and j < n:
                take = min(left, room)
                x[i, j] += take / a[i]
                left -= take
                room -= take
                if room <= 1e-15 * max(avg, 1.0):
                    j, room = j + 1, avg
            if left > 0 and j >= n:  # rounding remainder
                x[i, n - 1] += left / a[i]
        return x / x.sum(1, keepdims=True)
    order = sorted(range(E), key=lambda i: (-a[i], i))
    cost = np.zeros(n)
    avg = a.sum() / n
    for i in order:
        split = 1
        if mode == "replicated" and a[i] > avg and n > 1:
            split = int(min(max_replicas, n, np.ceil(a[i] / avg)))
        if split == 1:
            j = int(np.argmin(cost))
            x[i, j] = 1.0
            cost[j] += a[i]
        else:
            nodes = sorted(range(n), key=lambda j: (cost[j], j))[:split]
            for j in nodes:
                x[i, j] = 1.0 / split
                cost[j] += a[i] / split
    return x


@dataclass
class SlotPlacement:
    """Physical expert slots as the runtime executes them."""

    E: int                 # logical experts
    n_e: int               # expert GPUs
    P_l: int               # slots per expert GPU (contiguous blocks)
    phys2log: np.ndarray   # [P] logical expert of each slot (-1: empty slot)
    rep: np.ndarray        # [E, R+1] int32: count, then physical slots
    R: int

    @property
    def P(self) -> int:
        return self.n_e * self.P_l

    def gpu_of_slot(self, p: int) -> int:
        return p // self.P_l

    def logical_of_local(self, q: int) -> list:
        """Logical expert held by each local slot of expert GPU q (-1 = empty)."""
        return [int(v) for v in self.phys2log[q * self.P_l:(q + 1) * self.P_l]]

    def expected_gpu_rows(self, loads) -> np.ndarray:
        """Rows per expert GPU when expert e's rows split evenly over its replicas."""
        out = np.zeros(self.n_e)
        for e in range(self.E):
            c = int(self.rep[e, 0])
            for r in range(c):
                out[self.gpu_of_slot(int(self.rep[e, 1 + r]))] += loads[e] / c
        return out


def identity_slots(E: int, n_e: int) -> SlotPlacement:
    """No replication: slot p = logical expert p, contiguous blocks (the default layout)."""
    if E % n_e:
        raise ValueError("experts must divide over expert GPUs")
    rep = np.zeros((E, 2), np.int32)
    rep[:, 0] = 1
    rep[:, 1] = np.arange(E)
    return SlotPlacement(E, n_e, E // n_e, np.arange(E, dtype=np.int32), rep, 1)


def slots_from_placement(x: np.ndarray, max_replicas: int | None = None) -> SlotPlacement:
    """Integral / replicated placement x[E, N] -> physical slots.  Each nonzero
    (expert, node) becomes a slot on that node; nodes are padded with empty
    slots (never routed to) to a common P_l."""
    x = np.asarray(x)
    E, n = x.shape
    per_node = [[i for i in range(E) if x[i, j] > 0] for j in range(n)]
    P_l = max(1, max(len(v) for v in per_node))
    phys2log = np.full(n * P_l, -1, np.int32)
    slots_of = [[] for _ in range(E)]
    for j, experts in enumerate(per_node):
        for k, i in enumerate(experts):
            p = j * P_l + k
            phys2log[p] = i
            slots_of[i].append(p)
    R = max(len(v) for v in slots_of)
    if max_replicas is not None and R > max_replicas:
        raise ValueError("placement exceeds max_replicas")
    rep = np.zeros((E, R + 1), np.int32)
    for i, s in enumerate(slots_of):
        if not s:
            raise ValueError(f"expert {i} has no slot")
        rep[i, 0] = len(s)
        rep[i, 1:1 + len(s)] = s
    return SlotPlacement(E, n, P_l, phys2log, rep, R)


def balanced_slots(loads, n_e: int, max_replicas: int = 2, k_cold: float = 0.0) -> SlotPlacement:
    """balance_experts(mode='replicated') followed by slots_from_placement."""
    x = balance_experts(loads, n_e, k_cold=k_cold, mode="replicated", max_replicas=max_replicas)
    return slots_from_placement(x, max_replicas)


def spread_slots(E: int, n_e: int) -> SlotPlacement:
    """Even load on any number of expert GPUs (PAPER.md:452-455 on-device
    redundancy; SPEC.md:407-414 replicated mode with uniform loads): the first
    (E // n_e) * n_e experts are placed whole, E // n_e per GPU; each of the
    remaining E % n_e experts is replicated on every GPU, so token t of sender
    s reaches replica (t + s) mod n_e and each GPU carries 1 / n_e of its rows.
    Every GPU then holds E / n_e experts' worth of rows (e.g. Mixtral's 8
    experts on 5 expert GPUs: 1 whole + 3 fifths each, 4 slots per GPU), so a
    disaggregated split need not divide the expert count."""
    if n_e < 1 or E < 1:
        raise ValueError("need E >= 1 experts and n_e >= 1 GPUs")
    q, r = divmod(E, n_e)
    if r == 0:
        return identity_slots(E, n_e)
    x = np.zeros((E, n_e))
    for i in range(q * n_e):
        x[i, i // q] = 1.0
    for i in range(q * n_e, E):
        x[i, :] = 1.0 / n_e
    return slots_from_placement(x)


@dataclass
class AttnBatchPlan:
    """Requests assigned to attention nodes: ``assignment[j]``
    lists the request ids of node j (in placement order), ``predicted[j]`` its
    predicted attention time in seconds (k2 + sum of request costs; 0 for an
    empty node)."""

    assignment: list
    predicted: list

    @property
    def n_a(self) -> int:
        return len(self.assignment)

    def seq_lens(self, requests) -> list:
        """Per node, the sequence lengths of its requests (the attention
        stage's ctx_lens), in assignment order."""
        length = {rid: int(s) for rid, s in requests}
        return [np.array([length[r] for r in ids], np.int32) for ids in self.assignment]


def request_cost(seq_len: float, cm) -> float:
    """alpha·seq_len + beta: one decode request's share of T_a.
    Without a fitted beta the per-token slope k1 stands in for it."""
    beta = cm.beta if cm.beta is not None else (cm.k1 if cm.alpha == 0 else 0.0)
    return cm.alpha * float(seq_len) + beta


def _spread(load, k2) -> float:
    t = [k2 + v for v in load]
    lo = min(t)
    return max(t) / lo if lo > 0 else float("inf")


def _refine(assignment, load, cost, n_a, k2, max_batch, max_iter: int = 200):
    """Best-improvement local search on max/min node time (moves + swaps)."""
    for _ in range(max_iter):
        cur = _spread(load, k2)
        best = (cur * (1 - 1e-12), None)
        for a in range(n_a):
            for b in range(n_a):
                if a == b:
                    continue
                for ia, i in enumerate(assignment[a]):
                    # move i: a -> b
                    if len(assignment[a]) > 1 and (max_batch is None or len(assignment[b]) < max_batch):
                        trial = load.copy()
                        trial[a] -= cost[i]
                        trial[b] += cost[i]
                        f = _spread(trial, k2)
                        if f < best[0]:
                            best = (f, ("move", a, ia, b, None))
                    if a < b:
                        for ib, j in enumerate(assignment[b]):  # swap i <-> j
                            trial = load.copy()
                            trial[a] += cost[j] - cost[i]
                            trial[b] += cost[i] - cost[j]
                            f = _spread(trial, k2)
                            if f < best[0]:
                                best = (f, ("swap", a, ia, b, ib))
        if best[1] is None:
            return
        kind, a, ia, b, ib = best[1]
        i = assignment[a][ia]
        if kind == "move":
            assignment[a].pop(ia)
            assignment[b].append(i)
            load[a] -= cost[i]
            load[b] += cost[i]
        else:
            j = assignment[b][ib]
            assignment[a][ia], assignment[b][ib] = j, i
            load[a] += cost[j] - cost[i]
            load[b] += cost[i] - cost[j]


def compose_attention_batches(requests, n_a: int, cm, target_time: float | None = None,
                              max_batch: int | None = None, refine_limit: int = 32,
                              mode: str = "ffd") -> AttnBatchPlan:
    """Attention batch composition (§7 / SPEC.md:415-423): per-request
    cost alpha·seq_len + beta, first-fit-decreasing into n_a bins whose
    predicted time (k2 + costs) is capped at ``target_time``; a request no
    bin can take spills to the least-loaded bin (ties: lowest node index).
    Deterministic: requests of equal cost keep their input order.

    ``target_time`` None = the balanced target k2 + total cost / n_a.
    ``max_batch`` (additive; the runtime's per-node micro-batch capacity)
    also caps the request count of a bin; spills then go to the least-loaded
    bin with room.  ``mode="lpt"`` (additive) skips the first-fit step: every
    request, largest first, goes to the least-loaded bin with room -- the
    right rule when max_batch fixes every bin's request count (the runtime's
    equal micro-batches), where first-fit would fill the first bins with the
    largest requests and leave the spill to the count cap.

    Small instances (<= ``refine_limit`` requests, where one misplaced
    request moves a node's time by a large fraction) are then refined by
    deterministic local search -- the best single move or swap between two
    nodes while it lowers max/min of the node times -- which keeps FFD's
    result within 15 % of the brute-force optimal max/min ratio
    (tests/test_balance.py).  Large batches are FFD as stated."""
    if n_a < 1:
        raise ValueError("need at least one attention node")
    if mode not in ("ffd", "lpt"):
        raise ValueError("mode must be 'ffd' or 'lpt'")
    reqs = [(rid, float(s)) for rid, s in requests]
    if max_batch is not None and len(reqs) > n_a * max_batch:
        raise ValueError("more requests than n_a * max_batch")
    cost = [request_cost(s, cm) for _, s in reqs]
    if target_time is None:
        target_time = cm.k2 + sum(cost) / n_a
    if not target_time > 0:
        raise ValueError("target_time must be > 0")
    order = sorted(range(len(reqs)), key=lambda i: (-cost[i], i))
    load = [0.0] * n_a
    assignment = [[] for _ in range(n_a)]
    eps = 1e-12 * max(target_time, 1e-30)

    def has_room(j):
        return max_batch is None or len(assignment[j]) < max_batch

    for i in order:
        dest = None
        for j in range(n_a if mode == "ffd" else 0):
            if has_room(j) and cm.k2 + load[j] + cost[i] <= target_time + eps:
                dest = j
                break
        if dest is None:
            dest = min((j for j in range(n_a) if has_room(j)), key=lambda j: (load[j], j))
        assignment[dest].append(i)
        load[dest] += cost[i]
    if len(reqs) <= refine_limit and n_a > 1:
        _refine(assignment, load, cost, n_a, cm.k2, max_batch)
    assignment = [[reqs[i][0] for i in a] for a in assignment]
    predicted = [cm.k2 + load[j] if assignment[j] else 0.0 for j in range(n_a)]
    return AttnBatchPlan(assignment, predicted)
