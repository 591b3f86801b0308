"""Host-side logic of the multi-rank path (one process per GPU).

The device runtime exchanges halo messages with NCCL inside one
ncclGroupStart/End per stage; within a group NCCL matches sends and receives
per peer in issue order, so both endpoints must issue a link's messages in
the same order.  The contract (implemented in bf_runtime.cu,
remote_links_sorted) is: this rank's remote connected endpoints sorted by
(peer rank, link tag, own child id); a link's tag is its plan link id, which
both endpoints share (decomp.py:466-482).

The residual norm is the rank-ordered sum of per-rank sums, each of which is
the child-id-ordered sum of per-block sums (exchange.py:294-309,
solver.py:800-811) — deterministic for a fixed plan.
"""

from __future__ import annotations

import numpy as np

from .model import FIELD_NAMES


def remote_links(plan, rank):
    """This rank's remote endpoints in NCCL issue order:
    [(child_id, spec, peer_rank, tag)] sorted by (peer_rank, tag, child_id)."""
    out = []
    for c in plan.rank_children(rank):
        for s in plan.boundaries[c.id]:
            if s.kind != "connected":
                continue
            peer_rank = plan.child(s.neighbor_block).rank
            if peer_rank != rank:
                out.append((c.id, s, peer_rank, int(s.link_id)))
    out.sort(key=lambda e: (e[2], e[3], e[0]))
    return out


def rank_ordered_sum(parts):
    """Sum a list of per-rank 5-vectors in rank order (exchange.py:305-309)."""
    total = None
    for p in parts:
        p = np.asarray(p, dtype=float)
        total = p if total is None else total + p
    return total


def allgather_sum(local, dist):
    """All ranks' sums through torch.distributed, added in rank order."""
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, np.asarray(local, dtype=float))
    return rank_ordered_sum(parts)


def assemble_parent_fields(plan, parts):
    """Interior fields per parent from per-rank {child: {name: interior}} parts
    (exchange.py:666-676)."""
    fields = {b.id: {n: np.full(b.dims, np.nan) for n in FIELD_NAMES} for b in plan.grid.blocks}
    for part in parts:
        for cid, fl in part.items():
            c = plan.child(cid)
            (i0, i1), (j0, j1), (k0, k1) = c.cell_box()
            for n in FIELD_NAMES:
                fields[c.parent][n][i0:i1, j0:j1, k0:k1] = fl[n]
    return fields


def local_interiors(solvers):
    return {cid: {n: s.fields[n][s.block.interior()] for n in FIELD_NAMES}
            for cid, s in solvers.items()}
