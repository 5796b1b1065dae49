"""Multi-GPU sharding of a stream by block range.

Blocks are independent given their soft window, so rank r of G takes
the contiguous blocks [r*nb/G, (r+1)*nb/G) and reads the stages its forward
spans need -- its own range plus an L-stage halo on each side (replicated
reads, no halo exchange).  The only collective is the final gather of the
packed decoded bits (NCCL all_gather over NVLink on GPUs; gloo in the CPU
tests).  Byte alignment holds because D % 8 == 0.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    block0: int
    nblocks: int
    stage0: int          # first stage of the soft-value window
    stage1: int          # one past the last stage of the window
    bit0: int            # first decoded bit of the shard
    bit1: int            # one past the last decoded bit

    @property
    def nbytes(self) -> int:
        return (self.bit1 - self.bit0 + 7) // 8


def n_blocks(n_info: int, D: int) -> int:
    return -(-n_info // D)


def plan(n_info: int, D: int, L: int, K: int, terminated: bool, world: int, rank: int) -> Shard:
    """Block range and soft-value window of `rank` (P:93 geometry)."""
    assert D % 8 == 0 and 0 <= rank < world
    n_stages = n_info + ((K - 1) if terminated else 0)
    nb = n_blocks(n_info, D)
    b0 = rank * nb // world
    b1 = (rank + 1) * nb // world
    if b1 <= b0:
        return Shard(rank, world, b0, 0, 0, 0, 0, 0)
    lo = max(0, b0 * D - L)
    if b1 == nb:
        hi = n_stages
    else:
        hi = min(n_stages, min(b1 * D, n_info) + L)
    return Shard(rank, world, b0, b1 - b0, lo, hi, b0 * D, min(b1 * D, n_info))


def equal_shards(n_info: int, D: int, world: int) -> bool:
    """all_gather_into_tensor needs equal shard byte sizes."""
    nb = n_blocks(n_info, D)
    return nb % world == 0 and n_info % (D * world) == 0


def gather_bits(local, shard: Shard, n_info: int, D: int, group=None):
    """Concatenate every rank's packed bits in rank order (the a10 gather)."""
    import torch
    import torch.distributed as dist
    world = shard.world
    if world == 1:
        return local
    if equal_shards(n_info, D, world):
        out = torch.empty(local.numel() * world, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out
    # unequal last shard: pad to the largest shard then trim
    sizes = [plan(n_info, D, 0, 3, False, world, r).nbytes for r in range(world)]
    m = max(sizes)
    buf = torch.zeros(m, dtype=local.dtype, device=local.device)
    buf[:local.numel()] = local
    parts = [torch.empty(m, dtype=local.dtype, device=local.device) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


class PeerGather:
    """The final gather fused into the decode (pbvd_decode_blocks_mirrored):
    every rank allocates the whole stream's packed bits (`gbuf`, a device
    tensor), exports it with pbvd_ipc_export, and maps every other rank's
    buffer with pbvd_ipc_open (CUDA IPC, peer access over NVLink / NVSwitch).
    `mirrors(shard)` are then the device pointers, in this process, of the
    other ranks' copies of this rank's output range -- the traceback stores
    its bytes to all of them.  Raises RuntimeError (with the reason) when a
    peer is not reachable; the caller falls back to gather_bits (NCCL)."""

    def __init__(self, gbuf, group=None):
        import ctypes
        import torch
        import torch.distributed as dist
        from . import _lib
        self.L = _lib.load()
        self.gbuf = gbuf
        self.device = gbuf.device.index
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        handle = ctypes.create_string_buffer(_lib.PBVD_IPC_HANDLE_BYTES)
        off = ctypes.c_int64()
        rc = self.L.pbvd_ipc_export(ctypes.c_void_p(gbuf.data_ptr()), handle, ctypes.byref(off))
        mine = (self.device, handle.raw, off.value, rc,
                self.L.pbvd_last_error(None).decode() if rc else "")
        allv = [None] * self.world
        dist.all_gather_object(allv, mine, group=group)
        self.opened = []
        self.ptrs = [None] * self.world
        errs = [f"rank {r}: export failed: {a[4]}" for r, a in enumerate(allv) if a[3] != 0]
        if not errs:
            for r, (pdev, hraw, poff, _, _) in enumerate(allv):
                if r == self.rank:
                    self.ptrs[r] = gbuf.data_ptr()
                    continue
                if pdev != self.device and not torch.cuda.can_device_access_peer(self.device, pdev):
                    errs.append(f"no peer access cuda:{self.device} -> cuda:{pdev}")
                    break
                p = ctypes.c_void_p()
                rc = self.L.pbvd_ipc_open(hraw, poff, self.device, ctypes.byref(p))
                if rc != 0:
                    errs.append(f"rank {r}: {self.L.pbvd_last_error(None).decode()}")
                    break
                self.opened.append((p.value, poff))
                self.ptrs[r] = p.value
        ok = torch.tensor([0 if errs else 1], dtype=torch.int32,
                          device=gbuf.device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if errs or not int(ok.item()):
            self.close()
            raise RuntimeError("; ".join(errs) or "a peer rank could not map the buffers")

    def mirrors(self, shard):
        o = shard.bit0 // 8
        return [self.ptrs[r] + o for r in range(self.world) if r != self.rank]

    def close(self):
        for p, off in self.opened:
            self.L.pbvd_ipc_close(p, off, self.device)
        self.opened = []
