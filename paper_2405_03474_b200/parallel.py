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


class VirtualShards:
    """G row shards of one estimate in ONE process (RLD_COMM_THREADS): one librld handle per
    rank, each driven by its own host thread, collectives through device staging slots with
    host barriers (comm.cu) -- no kernel waits on another rank.  Runs the world > 1 code paths
    of the library on a single GPU (tests, and ``bench.py --virtual-shards``); production
    multi-GPU runs use one process per GPU over NCCL instead.

        with VirtualShards(3) as vs:
            results = vs.run(lambda: rstar_logdet(M, cfg))     # one LogDetEstimate per rank
    """

    def __init__(self, world_size: int, device: int = 0):
        from . import _native as N
        from ._session import Session

        if world_size < 1:
            raise ValueError("world_size must be >= 1")
        self.world_size = world_size
        self.group = N.VirtualGroup(world_size)
        self.sessions = [Session(device, r, world_size, group=self.group) for r in range(world_size)]

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def close(self):
        for s in self.sessions:
            s.handle.close()
        self.sessions = []
        self.group.close()

    def run(self, fn, *args):
        """fn(*args) on every rank concurrently, each in a thread bound to its rank's session
        (``fn`` may take the rank's Session as a keyword ``session`` if it declares one).
        Returns the per-rank results; re-raises the first root-cause error (a rank whose
        failure aborted the group makes the others fail with 'virtual group aborted')."""
        import inspect
        import threading

        from ._session import worker_session

        out = [None] * self.world_size
        errs = [None] * self.world_size
        wants = "session" in inspect.signature(fn).parameters

        def body(r):
            try:
                with worker_session(sess=self.sessions[r]):
                    out[r] = fn(*args, session=self.sessions[r]) if wants else fn(*args)
            except BaseException as e:  # noqa: BLE001 - collected and re-raised below
                errs[r] = e

        ths = [threading.Thread(target=body, args=(r,)) for r in range(self.world_size)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        real = [e for e in errs if e is not None and "virtual group aborted" not in str(e)]
        if real:
            raise real[0]
        if any(e is not None for e in errs):
            raise next(e for e in errs if e is not None)
        return out
