"""Row-shard plumbing for multi-GPU runs (one process per GPU).

The rows of K -- and of every n-vector block -- are split into contiguous
shards of ``ceil(n / G)`` rows.  ``torch.distributed`` only
bootstraps: rank 0 draws the NCCL unique id through the C ABI and broadcasts
its 128 bytes; from then on the collectives run inside ``librld.so`` on the
handle's stream (NCCL over NVLink / NVSwitch).
"""

from __future__ import annotations

import ctypes as C


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """[row0, row1) owned by ``rank`` (the C side uses the same formula, rld_api.cu prepare())."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    L = -(-n // world)
    r0 = min(n, rank * L)
    return r0, min(n, r0 + L)


def broadcast_nccl_id() -> bytes:
    import torch
    import torch.distributed as dist

    from ._native import load

    buf = torch.zeros(128, dtype=torch.uint8)
    if dist.get_rank() == 0:
        raw = C.create_string_buffer(128)
        rc = load().rld_nccl_unique_id(raw)
        if rc != 0:
            raise RuntimeError(f"rld_nccl_unique_id failed ({rc})")
        buf.copy_(torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8))
    if dist.get_backend() == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
        t = buf.to(dev)
        dist.broadcast(t, 0)
        buf = t.cpu()
    else:
        dist.broadcast(buf, 0)
    return bytes(buf.numpy().tobytes())
