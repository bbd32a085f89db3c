"""Host-side logic of the snapshot-window-sharded trainer (N > 1).

ReInc's communication-free placement (consecutive_block, ref
src/distsim.cpp:52-70) gives every rank a contiguous block of windows; the only
exchange is the sum of the flat gradient buffer once per optimizer step
(src/distsim.cpp:248-260), done here with torch.distributed (NCCL on GPUs,
gloo in the CPU tests).
"""
from __future__ import annotations


def rank_windows(total: int, world: int, rank: int, L: int, S: int, H: int):
    """[window_begin, window_end) of `rank` under consecutive_block."""
    from .api import plan
    row = plan(total, world, L, S, H)[rank]
    return row[2], row[3]


def run_sharded_epoch(sess, grad, allreduce=None):
    """One distsim epoch on this rank: per batch, local window-gradient sum ->
    all-reduce (sum over ranks) -> identical optimizer step on every rank.
    `sess` implements begin_epoch / local_grads / apply / end_epoch (the C-ABI
    session, or a test double). Returns the per-batch `applied` flags."""
    applied = []
    nb = sess.begin_epoch()
    for b in range(nb):
        sess.local_grads(b, grad)
        if allreduce is not None:
            allreduce(grad)
        applied.append(sess.apply(grad))
    sess.end_epoch()
    return applied


def torch_allreduce(world: int):
    """Sum all-reduce over the default process group (no-op for one rank)."""
    if world <= 1:
        return None
    import torch.distributed as dist

    def _ar(t):
        dist.all_reduce(t)

    return _ar
