"""Learning the FSM batching policy by tabular N-step Q-learning (PAPER §2.3) — oracle,
test infrastructure only (the product's C++ learner is ed_fsm_learn in libedbatch.so; the two share
no code; only the SplitMix64 draws are the same counter-based generator, implemented on each side).

What the paper fixes:
  * environment = the dataflow graph; state S_t = E(G_t) (E_sort by default); action = the
    type of the next batch; after the action the batch of ALL ready type-a nodes executes (Alg. 1).
  * reward Eq. 1: r(S_t, a_t) = -1 + alpha * ratio, with the ratio read as
    |Frontier_a(G_t)| / |Frontier(G^a_t)| (SURVEY A-1: the display is inverted w.r.t. the worked
    values 5/7 and 1/1 of P:138 and Lemma 1).
  * tabular Q-learning with N-step bootstrapping; pi(S) = argmax_a Q(S, a).
  * up to 1000 trials, early stop when the batch count reaches the lower bound, checked every 50
    iterations (App. B.3 lower bound).
Readings where the paper is silent (A-26; defaults):
  * alpha 0.5, learning rate 0.1, epsilon 0.5 decayed x0.95 every 10 episodes to a floor of 0.02,
    N = 4, no discounting (gamma = 1), max 1000 episodes, check every 50.
  * episodes cycle over the training graphs (one instance graph per episode); the backup runs
    after each episode for t = 0..T-1 in order:
        Q(S_t,a_t) += lr * (sum_{i<N, t+i<T} r_{t+i} + [t+N < T] max_b Q(S_{t+N}, b) - Q(S_t,a_t))
    with b over the types present in S_{t+N} (= the ready types) and unseen pairs valued 0.
  * epsilon-greedy over the ready types (ascending type id): u = (x >> 11) * 2^-53 of one
    SplitMix64 draw; if u < epsilon the action is ready[y % len(ready)] for a second draw y, else
    the greedy argmax (ties to the lowest type id).
  * the learned FSM table maps every state seen in Q to argmax_a Q(S, a) over the actions tried
    in S ("greedy argmax over ready types with table entries"; ties to the
    lowest type id); evaluation runs that table through Alg. 1 with the A-3 fallback key[0] for
    unseen states (what ed_plan executes).
  * the returned table is the best greedy table evaluated (the checkpoints, then the final Q;
    fewest batches, earliest on ties): with an early stop, the table that reached the bound.
  * the training graphs are either the instances (one per episode, cycling) or the one merged
    minibatch graph -- the dataflow graph Alg. 1 actually runs on ("the environment
    is the dataflow graph"); the caller passes [Merged(all instances)] for the latter.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

from .graph import Merged, lower_bound
from .schedule import ENCODERS, frontier, fsm_schedule, readiness_ratio, type_counts

MASK64 = (1 << 64) - 1


class SplitMix64:
    """Steele, Lea & Flood's SplitMix64 (the product learner implements the same recurrence)."""

    def __init__(self, seed: int):
        self.state = seed & MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
        return z ^ (z >> 31)


@dataclass
class RLConfig:
    encoder: str = "sort"
    alpha: float = 0.5
    lr: float = 0.1
    eps0: float = 0.5
    eps_decay: float = 0.95
    eps_every: int = 10
    eps_floor: float = 0.02
    n_steps: int = 4
    max_episodes: int = 1000
    check_every: int = 50
    seed: int = 4000


@dataclass
class RLResult:
    q: Dict[Tuple[tuple, int], float]
    table: Dict[tuple, int]
    episodes: int
    checkpoints: List[Tuple[int, int]] = field(default_factory=list)   # (episode, total batches)
    returns: List[float] = field(default_factory=list)                 # per-episode sum of rewards
    batches: List[int] = field(default_factory=list)                   # per-episode batch count
    lower_bound: int = 0
    final_batches: int = 0                                             # batches of the returned table


def ready_types(key: tuple, encoder: str) -> List[int]:
    """Types present in an encoded state = the ready types (E_max keys carry them in key[0])."""
    return sorted(key[0]) if encoder == "max" else sorted(key)


def greedy(q: Dict[Tuple[tuple, int], float], key: tuple, ready: Sequence[int]) -> int:
    """argmax_a Q(S, a) over the ready types; unseen pairs are 0; ties to the lowest type id."""
    best, best_v = None, None
    for a in ready:
        v = q.get((key, a), 0.0)
        if best_v is None or v > best_v:
            best, best_v = a, v
    return best


def policy_table(q: Dict[Tuple[tuple, int], float], encoder: str) -> Dict[tuple, int]:
    """pi(S) = argmax_a Q(S, a) for every state that has Q entries, a over the actions with a
    Q entry in S; ties to the lowest type id."""
    table = {}
    for k in sorted({k for k, _ in q}, key=repr):
        tried = [a for a in ready_types(k, encoder) if (k, a) in q]
        table[k] = greedy(q, k, tried)
    return table


def reward(m: Merged, executed: Sequence[bool], a: int, alpha: float) -> float:
    """Eq. 1 with the A-1 ratio."""
    return -1.0 + alpha * readiness_ratio(m, executed, a)


def run_episode(m: Merged, q, cfg: RLConfig, eps: float, rng: SplitMix64):
    """One pass of Alg. 1 with epsilon-greedy actions; returns the (S, a, r) trace."""
    enc = ENCODERS[cfg.encoder]
    executed = [False] * m.n
    trace = []
    while not all(executed):
        front = frontier(m, executed)
        counts = type_counts(m, front)
        key = enc(counts)
        ready = sorted(counts)
        u = (rng.next() >> 11) * (2.0 ** -53)
        if u < eps:
            a = ready[rng.next() % len(ready)]
        else:
            a = greedy(q, key, ready)
        r = reward(m, executed, a, cfg.alpha)
        for v in front:
            if m.type[v] == a:
                executed[v] = True
        trace.append((key, a, r))
    return trace


def nstep_backup(q, trace, cfg: RLConfig) -> None:
    T = len(trace)
    n = cfg.n_steps
    for t in range(T):
        g = 0.0
        for i in range(n):
            if t + i < T:
                g += trace[t + i][2]
        if t + n < T:
            k2 = trace[t + n][0]
            g += max(q.get((k2, b), 0.0) for b in ready_types(k2, cfg.encoder))
        key, a, _ = trace[t]
        old = q.get((key, a), 0.0)
        q[(key, a)] = old + cfg.lr * (g - old)


def train(graphs: Sequence[Merged], cfg: RLConfig = RLConfig()) -> RLResult:
    """Tabular N-step Q-learning over the instance graphs (each a Merged of one instance)."""
    if not graphs or cfg.alpha < 0 or cfg.n_steps < 1 or cfg.check_every < 1:
        raise ValueError("bad RL config")
    rng = SplitMix64(cfg.seed)
    q: Dict[Tuple[tuple, int], float] = {}
    lb = sum(lower_bound(m) for m in graphs)
    res = RLResult(q=q, table={}, episodes=0, lower_bound=lb)
    best = None
    for ep in range(cfg.max_episodes):
        m = graphs[ep % len(graphs)]
        eps = max(cfg.eps_floor, cfg.eps0 * cfg.eps_decay ** (ep // cfg.eps_every))
        trace = run_episode(m, q, cfg, eps, rng)
        res.returns.append(sum(r for _, _, r in trace))
        res.batches.append(len(trace))
        nstep_backup(q, trace, cfg)
        res.episodes = ep + 1
        if (ep + 1) % cfg.check_every == 0:
            table = policy_table(q, cfg.encoder)
            total = sum(len(fsm_schedule(g, table, cfg.encoder)) for g in graphs)
            res.checkpoints.append((ep + 1, total))
            if best is None or total < best:
                best, res.table = total, table
            if total == lb:
                break
    table = policy_table(q, cfg.encoder)
    total = sum(len(fsm_schedule(g, table, cfg.encoder)) for g in graphs)
    if best is None or total < best:
        best, res.table = total, table
    res.final_batches = best
    return res
