"""z-slab decomposition of ``total_sum`` over several GPUs.

The reference library is single-process; this is the multi-GPU layer the
north star asks for, built on the slab entry points of the C-ABI
(``fse_cuda_slab_*``, include/fse_cuda.h).  Slab ``r`` of ``G`` owns the
x-planes ``[x_lo, x_lo + nx)`` of the M~ grid (the slowest axis of the
reference layout ``(i*M~ + j)*M~ + k``) and the ky rows ``[ky_lo, ky_lo + nky)``
of the k-space pass.  Every rank holds all points (inputs are replicated, as
in the reference's API), so spreading and quadrature need no halo exchange:
a rank spreads every point's support onto its own planes and adds its planes'
share of every target's quadrature.  The exchanges per evaluation are

1. all-to-all of the y-transformed spectrum (block ``s`` -> rank ``s``),
2. all-to-all back after the fused x-FFT / multiplier / inverse x-FFT,
3. one sum of the per-rank partial velocities (the real-space sum and the
   self term of target range ``r`` are added by rank ``r`` only).

``Exchange`` implementations: ``TorchExchange`` (torch.distributed; NCCL over
NVLink on GPUs, gloo on CPU for the tests), ``PeerExchange`` (no all-to-all:
the y pass and the x pass store their blocks straight into the owning rank's
buffer, mapped over NVLink with torch symmetric memory, and a barrier orders
the phases; see ``fse_cuda_slab_forward_peers``) and the single-process
``simulate`` driver, which runs ``G`` virtual ranks one after another on one
device (no kernel ever waits on another rank) to check the decomposition --
both exchanges -- against the one-GPU result.
"""
from __future__ import annotations

import numpy as np

from .api import Context, EwaldConfig, MollifiedGreen, slab_info, strength_arity

COMPLEX_BYTES = 16


class DeviceArray:
    """__cuda_array_interface__ view of a device allocation (float64)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8",
                                         "data": (int(ptr), False), "version": 3}


def torch_view(ptr: int, n: int):
    """torch.float64 CUDA tensor aliasing n doubles at ptr (no copy)."""
    import torch
    return torch.as_tensor(DeviceArray(ptr, n), device="cuda")


class TorchExchange:
    """Block all-to-all and sum over a torch.distributed process group.

    ``all_to_all(send, recv)``: both are 1-D tensors of ``size`` equal blocks;
    block ``s`` of ``send`` goes to rank ``s`` and lands as block ``r`` (this
    rank) of its ``recv``.  Works for CUDA tensors (NCCL) and CPU tensors
    (gloo).
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def _sync(self, t):
        if t.is_cuda:
            import torch
            torch.cuda.current_stream(t.device).synchronize()

    def all_to_all(self, send, recv):
        if send.numel() % self.size or recv.numel() != send.numel():
            raise ValueError("all_to_all: buffers must hold `size` equal blocks")
        if self.dist.get_backend(self.group) == "gloo":
            # gloo has no all_to_all_single: a send/recv ring of blocks
            blk = send.numel() // self.size
            recv.view(self.size, blk)[self.rank].copy_(send.view(self.size, blk)[self.rank])
            reqs = []
            for k in range(1, self.size):
                dst = (self.rank + k) % self.size
                src = (self.rank - k) % self.size
                reqs.append(self.dist.isend(send.view(self.size, blk)[dst].contiguous(), dst,
                                            group=self.group))
                reqs.append(self.dist.irecv(recv.view(self.size, blk)[src], src,
                                            group=self.group))
            for q in reqs:
                q.wait()
        else:
            self.dist.all_to_all_single(recv, send, group=self.group)
        self._sync(recv)

    def all_reduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        self._sync(t)


class PeerExchange:
    """Peer-direct exchange buffers: two symmetric-memory allocations per rank
    (CUDA IPC mappings over NVLink), every rank's buffer addresses known to all.

    ``ptrs[0][s]`` / ``ptrs[1][s]``: rank s's forward (A) / backward (B) buffer.
    """

    def __init__(self, nelem: int, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        self.torch, self.dist = torch, dist
        self.group = group if group is not None else dist.distributed_c10d._get_default_group()
        self.rank = dist.get_rank(self.group)
        self.size = dist.get_world_size(self.group)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.tensors, self.handles, self.ptrs = [], [], []
        for _ in range(2):
            t = symm_mem.empty(int(nelem), dtype=torch.float64, device=dev)
            h = symm_mem.rendezvous(t, self.group)
            self.tensors.append(t)
            self.handles.append(h)
            self.ptrs.append([int(q) for q in h.buffer_ptrs])

    def barrier(self):
        """All ranks' previous phase done (the C-ABI calls return after their
        kernels completed; the device barrier then orders the ranks)."""
        self.torch.cuda.synchronize()
        self.handles[0].barrier()
        self.torch.cuda.synchronize()


class SlabSum:
    """One rank's side of the decomposed ``total_sum`` (device pointers).

    Buffers are allocated once per (config, kind) and reused across calls.
    """

    def __init__(self, ctx: Context, cfg: EwaldConfig, kind, rank: int, nslabs: int):
        self.ctx, self.cfg, self.kind = ctx, cfg, int(kind)
        self.rank, self.nslabs = int(rank), int(nslabs)
        self.info = slab_info(cfg, kind, rank, nslabs)
        self.block_doubles = 2 * int(self.info.block_complex)
        nbytes = 8 * self.block_doubles * self.nslabs
        self.d_send = ctx.dev_alloc(nbytes)
        self.d_recv = ctx.dev_alloc(nbytes)

    def free(self):
        for p in (self.d_send, self.d_recv):
            if p:
                self.ctx.dev_free(p)
        self.d_send = self.d_recv = 0

    # the three local phases
    def forward(self, d_pos, d_str, n):
        self.ctx.slab_forward(self.cfg, self.kind, d_pos, d_str, n, self.rank, self.nslabs,
                              self.d_send)

    def scale(self, green: MollifiedGreen):
        self.ctx.slab_scale(self.cfg, self.kind, green, self.rank, self.nslabs, self.d_recv)

    def inverse(self, d_pos, d_str, n, d_tgt, nt, tas, d_u):
        self.ctx.slab_inverse(self.cfg, self.kind, d_pos, d_str, n, self.d_send, self.rank,
                              self.nslabs, d_tgt, nt, int(tas), d_u)

    def run_peers(self, px: PeerExchange, ex: TorchExchange, green, d_pos, d_str, n, d_tgt,
                  nt, tas, d_u):
        """Full evaluation with the peer-direct exchange (buffers of ``px``; the
        final sum of the partial velocities still goes through ``ex``)."""
        fwd, bwd = px.ptrs
        r, G = self.rank, self.nslabs
        self.ctx.slab_forward_peers(self.cfg, self.kind, d_pos, d_str, n, r, G, fwd)
        px.barrier()
        self.ctx.slab_scale_peers(self.cfg, self.kind, green, r, G, fwd[r], bwd)
        px.barrier()
        self.ctx.slab_inverse(self.cfg, self.kind, d_pos, d_str, n, bwd[r], r, G, d_tgt, nt,
                              int(tas), d_u)
        ex.all_reduce_sum(torch_view(d_u, 3 * nt))

    def run(self, ex: TorchExchange, green, d_pos, d_str, n, d_tgt, nt, tas, d_u):
        """Full evaluation; on return d_u (NT x 3) holds the summed velocities."""
        send = torch_view(self.d_send, self.block_doubles * self.nslabs)
        recv = torch_view(self.d_recv, self.block_doubles * self.nslabs)
        self.forward(d_pos, d_str, n)
        ex.all_to_all(send, recv)
        self.scale(green)
        ex.all_to_all(recv, send)
        self.inverse(d_pos, d_str, n, d_tgt, nt, tas, d_u)
        ex.all_reduce_sum(torch_view(d_u, 3 * nt))


def simulate(ctx: Context, cfg: EwaldConfig, kind, positions, strengths, targets, green,
             nslabs: int, targets_are_sources: bool, peers: bool = False) -> np.ndarray:
    """Run the G-slab pipeline as G virtual ranks on one device, in sequence.

    Host arrays in, host velocities out.  ``peers=False``: the exchanges are
    device copies between the virtual ranks' buffers (what the all-to-all
    does); ``peers=True``: the peer-direct entry points store every block
    straight into the owning virtual rank's buffer, as over NVLink.  Used by
    the tests to check the decomposition against ``Context.total_sum``.
    """
    pos = np.ascontiguousarray(positions, dtype=np.float64)
    st = np.ascontiguousarray(strengths, dtype=np.float64)
    tgt = np.ascontiguousarray(targets, dtype=np.float64)
    n, nt = pos.shape[0], tgt.shape[0]
    if st.shape != (n, strength_arity(kind)):
        raise ValueError("strengths shape does not match the kernel arity")
    d_pos = ctx.dev_alloc(max(pos.nbytes, 8))
    d_str = ctx.dev_alloc(max(st.nbytes, 8))
    d_tgt = ctx.dev_alloc(max(tgt.nbytes, 8))
    d_u = ctx.dev_alloc(max(8 * 3 * nt, 8))
    ranks = []
    try:
        ctx.memcpy(d_pos, pos.ctypes.data, pos.nbytes)
        ctx.memcpy(d_str, st.ctypes.data, st.nbytes)
        ctx.memcpy(d_tgt, tgt.ctypes.data, tgt.nbytes)
        ranks = [SlabSum(ctx, cfg, kind, r, nslabs) for r in range(nslabs)]
        blk = 8 * ranks[0].block_doubles
        if peers:  # forward buffers = the d_recv's, backward buffers = the d_send's
            fwd = [rk.d_recv for rk in ranks]
            bwd = [rk.d_send for rk in ranks]
            for r in range(nslabs):
                ctx.slab_forward_peers(cfg, kind, d_pos, d_str, n, r, nslabs, fwd)
            for r in range(nslabs):
                ctx.slab_scale_peers(cfg, kind, green, r, nslabs, fwd[r], bwd)
        else:
            for rk in ranks:
                rk.forward(d_pos, d_str, n)
            for r, rk in enumerate(ranks):      # block s of rank r -> block r of rank s
                for s, dst in enumerate(ranks):
                    ctx.memcpy(dst.d_recv + r * blk, rk.d_send + s * blk, blk)
            for rk in ranks:
                rk.scale(green)
            for s, rk in enumerate(ranks):      # block r of rank s -> block s of rank r
                for r, dst in enumerate(ranks):
                    ctx.memcpy(dst.d_send + s * blk, rk.d_recv + r * blk, blk)
        u = np.zeros((nt, 3))
        part = np.empty((nt, 3))
        for rk in ranks:
            rk.inverse(d_pos, d_str, n, d_tgt, nt, targets_are_sources, d_u)
            ctx.memcpy(part.ctypes.data, d_u, part.nbytes)
            u += part
        return u
    finally:
        for rk in ranks:
            rk.free()
        for p in (d_pos, d_str, d_tgt, d_u):
            ctx.dev_free(p)
