"""Process-group plumbing for the multi-process (one GPU per process) path.

Host logic only -- handle exchange, plan agreement, timing reduction -- over
any torch.distributed backend (gloo on CPU works; the collectives themselves
never go through torch.distributed).
"""
import hashlib
import json

import paper_1910_04940_b200 as B


def exchange(group=None):
    """`exchange(blob) -> [blob_0, ..., blob_{n-1}]` over torch.distributed."""
    return B.torch_exchange(group)


def plan_digest(nranks, is_allreduce, root, count, dtype="f32", graph=None, cfg=None):
    """SHA-256 of the host-only plan (TreeGen + split + chunking)."""
    p = B.plan_json(nranks, is_allreduce, root, count, dtype, graph=graph, cfg=cfg)
    return hashlib.sha256(json.dumps(p, sort_keys=True).encode()).hexdigest()


def check_same_plan(nranks, is_allreduce, root, count, dtype="f32", graph=None, cfg=None, group=None):
    """Every rank must plan the same trees (the collective contract: same graph,
    config and call sequence on every rank).  Raises on disagreement."""
    d = plan_digest(nranks, is_allreduce, root, count, dtype, graph, cfg).encode()
    all_d = exchange(group)(d)
    if len(set(all_d)) != 1:
        bad = [i for i, x in enumerate(all_d) if x != all_d[0]]
        raise B.BlinkError(5, f"ranks {bad} planned different trees than rank 0 "
                              "(graph/config differ across ranks)")
    return d.decode()


def max_over_ranks(value, group=None):
    """Max of a host float over ranks (bench timing: max over ranks)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def init(graph=None, cfg=None, device=None, group=None):
    """Multi-process comm for this rank of the default process group."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if device is None:
        import torch
        device = torch.cuda.current_device()
    return B.init_multiprocess(world, rank, device, exchange(group), graph=graph, cfg=cfg)
