"""ORACLE (test infrastructure only) — dynamic reconfiguration over a template set,
PAPER.md §5 and Appendix B, written out step by step.

Only `tests/` may import this module; it shares no code with paper_2309_08125_b200/.

State: a list of pipelines, each instantiated from the template of its node count
(a pipeline is "an instance of a pipeline template"), holding an ordered list of
node ids; template stage i runs on the pipeline's node `stage.node` (template-local index).

`apply_failures` follows §5.1 "in three steps: simple reinstantiation, borrowing nodes,
and merging pipelines", then §5.2 batch redistribution.  Where the
paper is silent the readings are DESIGN.md §10 (R21-R27):
  R21 affected pipelines are processed in ascending surviving node count (ties: pipeline
      index); a pipeline that lost every node disappears;
  R22 (1) a pipeline with s surviving nodes, n_lo <= s <= n_hi, is reinstantiated from the
      template of s nodes;
  R23 (2) with s < n0 it borrows one node at a time from the pipeline that can yield (more
      than n0 nodes), the largest first (ties: lowest index), which gives its LAST node and
      is reinstantiated with one node fewer; the borrowed node is appended;
  R24 (3) if no pipeline can yield, it merges with the smallest other pipeline (ties:
      lowest index) — its nodes first, then the partner's — repeatedly until >= n0 nodes
      (Appendix B: a template of the merged size exists; a merged size above n_hi is an
      error, `NoTemplate`);
  R25 survivors < (f+1) n0: training checkpoints and exits — `Exit`;
  R26 after reinstantiation the batch is redistributed with Eq.6 over the new pipelines
      (T_i = t* of the pipeline's template, reading R19); the global batch is unchanged;
  R28 if whole pipelines failed and fewer than f+1 pipelines remain although >= (f+1) n0
      nodes survive, the cluster can still hold f+1 replicas, so the pipelines
      are instantiated afresh over the survivors (§4.2: "Pipeline instantiation and batch
      distribution happens whenever a node fails"): the max-throughput plan of
      Eq.5/Eq.6 (select_plan), survivors in ascending id order filling its pipelines in
      template order — action ("replan", number of pipelines);
  R27 layer copies: every (node, layer) the new state needs and the
      node did not hold is copied from a surviving node that held the layer before, the
      one with the fewest transfers so far (ties: lowest node id), in (node id, layer)
      order; no surviving owner of a needed layer is `Unrecoverable` (§3.2).
`sync_groups` (§6.1): per layer, the (pipeline, stage) that holds it in every
pipeline — the peers of that layer's gradient all-reduce.
Pins: tests/test_reconfig.py (the three Fig. 7 cases; Appendix B's guarantee as a
property over random failure sequences; invariants: every survivor in exactly one pipeline,
>= f+1 pipelines, template conformance, batch conservation, one sync entry per pipeline).
"""
from __future__ import annotations

from .instantiate import distribute_batch_brute, select_plan_brute


class Exit(Exception):
    """Fewer than (f+1) n0 nodes survive: checkpoint and exit."""


class NoTemplate(Exception):
    """A merged pipeline above the largest template (Appendix B's premise broken)."""


class Unrecoverable(Exception):
    """A layer needed by the new state has no surviving owner."""


class State:
    def __init__(self, templates, f: int, B: int, b: int, layer_bytes=None):
        """templates: the template set (list of dicts with 'nodes', 'stages', 'tstar', ...)
        of consecutive sizes n_lo..n_hi."""
        self.tpl = {t["nodes"]: t for t in templates}
        self.n_lo = min(self.tpl)
        self.n_hi = max(self.tpl)
        self.f = f
        self.B = B
        self.b = b
        self.L = templates[0]["stages"][-1][1]
        self.layer_bytes = list(layer_bytes) if layer_bytes is not None else [0] * self.L
        self.pipes = []          # [[node ids]] (template = len)
        self.nb = []

    @classmethod
    def from_counts(cls, templates, counts, node_ids, f, B, b, layer_bytes=None):
        """Pipelines in template order (x_i pipelines of size n_lo + i), nodes consecutive."""
        st = cls(templates, f, B, b, layer_bytes)
        pos = 0
        for i, c in enumerate(counts):
            n = st.n_lo + i
            for _ in range(c):
                st.pipes.append(list(node_ids[pos:pos + n]))
                pos += n
        if pos != len(node_ids):
            raise ValueError("node count does not match the counts")
        st.nb = st.distribute()
        return st

    # -------------------------------------------------------------- views
    def owned(self):
        """node id -> set of layers it holds (its stages in its pipeline's template)."""
        own = {}
        for nodes in self.pipes:
            t = self.tpl[len(nodes)]
            for (u, v, d, node, goff) in t["stages"]:
                own.setdefault(nodes[node], set()).update(range(u, v))
        return own

    def sync_groups(self):
        """Per layer: [(pipeline, stage)] — the stage of every pipeline that holds it."""
        out = []
        for layer in range(self.L):
            g = []
            for p, nodes in enumerate(self.pipes):
                for s, (u, v, d, node, goff) in enumerate(self.tpl[len(nodes)]["stages"]):
                    if u <= layer < v:
                        g.append((p, s))
            out.append(g)
        return out

    def distribute(self):
        """Eq.6 over the current pipelines (reading R26); raises ValueError if B is not
        distributable over them."""
        T = [self.tpl[len(n)]["tstar"] for n in self.pipes]
        nb, _ = distribute_batch_brute(T, self.B, self.b)
        return list(nb)

    # -------------------------------------------------------------- §5.1
    def apply_failures(self, failed):
        failed = set(failed)
        alive = [n for nodes in self.pipes for n in nodes]
        if not failed <= set(alive):
            raise ValueError("unknown or already failed node")
        before = self.owned()
        survivors = len(alive) - len(failed)
        if survivors < (self.f + 1) * self.n_lo:                       # R25
            raise Exit()
        pipes = [[n for n in nodes if n not in failed] for nodes in self.pipes]
        affected = [i for i, nodes in enumerate(self.pipes) if any(n in failed for n in nodes)]
        live = [True] * len(pipes)
        actions = []
        for i in sorted(affected, key=lambda i: (len(pipes[i]), i)):  # R21
            if not live[i]:
                continue
            if not pipes[i]:
                live[i] = False
                actions.append(("remove", i))
                continue
            if self.n_lo <= len(pipes[i]) <= self.n_hi:               # R22
                actions.append(("reinstantiate", i, len(pipes[i])))
                continue
            while len(pipes[i]) < self.n_lo:                          # R23
                donors = [j for j in range(len(pipes)) if live[j] and j != i and len(pipes[j]) > self.n_lo]
                if not donors:
                    break
                j = min(donors, key=lambda j: (-len(pipes[j]), j))
                pipes[i].append(pipes[j].pop())
                actions.append(("borrow", j, i))
            while len(pipes[i]) < self.n_lo:                          # R24
                others = [j for j in range(len(pipes)) if live[j] and j != i]
                j = min(others, key=lambda j: (len(pipes[j]), j))
                pipes[i] = pipes[i] + pipes[j]
                live[j] = False
                actions.append(("merge", i, j))
            if len(pipes[i]) > self.n_hi:
                raise NoTemplate(len(pipes[i]))
            actions.append(("reinstantiate", i, len(pipes[i])))
        self.pipes = [p for p, ok in zip(pipes, live) if ok]
        if len(self.pipes) < self.f + 1:                                 # R28
            nodes = sorted(n for p in self.pipes for n in p)
            plan = select_plan_brute([self.tpl[n] for n in range(self.n_lo, self.n_hi + 1)], len(nodes),
                                     self.f, self.B, self.b)
            if plan is None:
                raise Exit()
            counts = plan[1]
            self.pipes = []
            pos = 0
            for i, c in enumerate(counts):
                for _ in range(c):
                    self.pipes.append(nodes[pos:pos + self.n_lo + i])
                    pos += self.n_lo + i
            actions.append(("replan", len(self.pipes)))
        after = self.owned()
        copies = copy_plan(before, after, failed, self.layer_bytes)
        self.nb = self.distribute()                                     # R26
        return actions, copies


def copy_plan(before, after, failed, layer_bytes):
    """Reading R27: (layer, donor, receiver, bytes) transfers, receivers in (node, layer) order."""
    sent = {}
    out = []
    for node in sorted(after):
        have = before.get(node, set()) if node not in failed else set()
        for layer in sorted(after[node] - have):
            owners = [n for n, ls in before.items() if n not in failed and layer in ls]
            if not owners:
                raise Unrecoverable(layer)
            donor = min(owners, key=lambda n: (sent.get(n, 0), n))
            sent[donor] = sent.get(donor, 0) + 1
            out.append((layer, donor, node, layer_bytes[layer]))
    return out
