"""PackedEmbedding: owns the torch buffers (workspace, packed tables, optimizer state) of one
rank's context and forwards to the C ABI.  Plumbing only — every step runs in libpicasso."""
from __future__ import annotations

import os

import numpy as np
import torch

from . import abi


def default_exchange():
    """PICASSO_EXCHANGE = p2p (default) | nccl: how a row-sharded step exchanges keys / rows / G."""
    import os

    return os.environ.get("PICASSO_EXCHANGE", "p2p")


class PackedEmbedding:
    """One rank of the packed multi-field embedding layer.

    field_to_table [F], table_rows [T], table_dim [T]: the model.
    The D-Packing plan comes from picasso_pack_plan (Eq. 1).  Output columns are the
    fields' dims laid side by side in field order unless field_col is given.
    """

    def __init__(self, field_to_table, table_rows, table_dim, *, max_batch, max_ids, table_salt=None,
                 field_col=None, pool=abi.POOL_SUM, id_mode=abi.IDS_HASH, opt=abi.OPT_ADAGRAD, eps=None,
                 beta1=0.9, beta2=0.999, split=False, warmup_count=None, rank=0, world=1, device="cuda",
                 init_acc=0.1, nccl_uid=None, max_recv=0, cache_max_bytes=0, exchange=None, all_gather=None,
                 max_step_unique=0, max_step_floats=0, cold_tier=False, plan=None):
        self.f2t = np.asarray(field_to_table, np.int32)
        self.rows = np.asarray(table_rows, np.int64)
        self.dims = np.asarray(table_dim, np.int32)
        # every table is stored at its kernel dim (picasso_kernel_dim: dims other than 4, 8, 16, ... 512 are
        # zero-padded); the output column block of a field is that wide, the padding columns stay 0
        self.kdims = np.array([abi.picasso_kernel_dim(int(d)) for d in self.dims], np.int32)
        fd = self.kdims[self.f2t].astype(np.int64)
        self.field_col = (np.concatenate([[0], np.cumsum(fd)[:-1]]) if field_col is None
                          else np.asarray(field_col, np.int64))
        self.out_width = int(max(self.field_col + fd)) if len(fd) else 0
        self.out_width = (self.out_width + 3) // 4 * 4
        # plan: a precomputed plan dict (e.g. picasso_pack_plan_kinterleave's, with pack_group)
        self.plan = plan if plan is not None else abi.picasso_pack_plan(self.f2t, self.rows, self.dims,
                                                                        warmup_count, split)
        self.opt = opt
        self.rank, self.world = rank, world
        self.exchange = exchange or default_exchange()
        self.device = torch.device(device)
        self.ctx = abi.picasso_ctx_create(self.plan, self.f2t, self.rows, self.dims, table_salt, self.field_col,
                                          self.out_width, rank, world, max_batch, max_ids, pool, id_mode, opt,
                                          eps, beta1, beta2, nccl_uid=nccl_uid, max_recv=max_recv,
                                          cache_max_bytes=cache_max_bytes, exchange=self.exchange,
                                          max_step_unique=max_step_unique, max_step_floats=max_step_floats,
                                          cold_tier=int(bool(cold_tier)))
        self.cold_tier = bool(cold_tier)
        P = self.plan["n_packs"]
        self.local_rows = [abi.picasso_pack_local_rows(self.ctx, p) for p in range(P)]
        ws = abi.picasso_workspace_size(self.ctx)
        self.workspace = torch.empty(ws + 256, dtype=torch.uint8, device=self.device)
        # cold tier (HybridHash with host-DRAM Cold-storage): the tables and their
        # optimizer state live in pinned host memory the GPU maps; HBM holds only the hot rows
        def table(p, r, fill):
            shape = (max(r, 1), abi.picasso_kernel_dim(int(self.plan["pack_dim"][p])))
            if self.cold_tier:
                return torch.empty(shape, dtype=torch.float32, pin_memory=True).fill_(fill)
            return torch.full(shape, fill, dtype=torch.float32, device=self.device)

        rows = list(enumerate(self.local_rows))
        self.weights = [table(p, r, 0.0) for p, r in rows]
        self.state1 = [table(p, r, init_acc if opt == abi.OPT_ADAGRAD else 0.0) for p, r in rows]
        self.state2 = None if opt == abi.OPT_ADAGRAD else [table(p, r, 0.0) for p, r in rows]
        abi.picasso_bind(self.ctx, self.workspace, self.weights, self.state1, self.state2)
        self.step = 0
        # world > 1, one process per GPU: the exchange runs over NVLink peer memory ("p2p", the
        # default) or NCCL AllToAllv ("nccl").  all_gather(bytes) -> [bytes] * world shares the
        # windows' IPC handles (default: torch.distributed.all_gather_object).
        # Without a NCCL id (nccl_uid None) the peer-memory exchange still runs when all_gather is
        # given and the cache is off: e.g. several processes sharing one GPU, where NCCL refuses
        # duplicate devices (tests/test_xproc_gpu.py).
        if world > 1 and self.exchange == "p2p" and (nccl_uid is not None or all_gather is not None):
            h = abi.picasso_p2p_handle(self.ctx)
            if all_gather is None:
                import torch.distributed as dist

                def all_gather(x):
                    out = [None] * world
                    dist.all_gather_object(out, x)
                    return out
            abi.picasso_p2p_open(self.ctx, all_gather(h))
            # HybridHash hot-row gradients over NVLS multicast (PICASSO_NVLS=0: keep NCCL's AllReduce)
            self.nvls = False
            if cache_max_bytes > 0 and nccl_uid is not None and os.environ.get("PICASSO_NVLS", "1") != "0":
                self.nvls = self._nvls_setup(all_gather)

    def _nvls_setup(self, all_gather):
        """Collective: every rank runs the same calls; any failure on any rank leaves all ranks on the
        NCCL AllReduce (the agreement goes through all_gather).  Rank 0's multicast descriptor reaches
        the other processes over an abstract Unix socket (SCM_RIGHTS)."""
        import secrets
        import socket
        import sys

        def attempt(fn, *args):
            try:
                return True, fn(self.ctx, *args)
            except abi.PicassoError as err:
                print(f"[picasso] rank {self.rank}: NVLS off ({err}); hot rows use the NCCL AllReduce",
                      file=sys.stderr)
                return False, None

        ok, fd = attempt(abi.picasso_nvls_create)
        srv, name = None, b""
        if ok and self.rank == 0:
            name = b"\0picasso-nvls-" + secrets.token_hex(8).encode()
            srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
            srv.bind(name)
            srv.listen(self.world)
        res = all_gather((ok, name))
        if not all(r[0] for r in res):
            if srv:
                srv.close()
            return False
        try:
            if self.rank == 0:
                for _ in range(self.world - 1):
                    conn, _ = srv.accept()
                    socket.send_fds(conn, [b"f"], [fd])
                    conn.close()
                srv.close()
                myfd = fd
            else:
                cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
                cli.connect(res[0][1])
                _, fds, _, _ = socket.recv_fds(cli, 1, 1)
                cli.close()
                myfd = fds[0]
        except OSError as err:
            print(f"[picasso] rank {self.rank}: NVLS off (descriptor exchange: {err})", file=sys.stderr)
            ok = False
        if not all(all_gather(ok)):
            return False
        ok, _ = attempt(abi.picasso_nvls_open, myfd)
        if self.rank != 0:
            os.close(myfd)  # the driver holds its own reference after the import
        if not all(all_gather(ok)):  # also the barrier between every rank's open and any bind
            return False
        ok, _ = attempt(abi.picasso_nvls_bind)
        return all(all_gather(ok))

    @property
    def n_packs(self):
        return self.plan["n_packs"]

    def forward(self, ids: torch.Tensor, offsets: torch.Tensor, batch: int, out: torch.Tensor | None = None,
                stream=None):
        if out is None:
            out = torch.empty(batch, self.out_width, dtype=torch.float32, device=self.device)
        abi.picasso_packed_lookup_fwd(self.ctx, ids, offsets, batch, out, stream, n_fields=len(self.f2t),
                                      out_width=self.out_width, device=self.device)
        self._batch = batch
        return out

    def backward_update(self, grad_out: torch.Tensor, lr: float, step: int | None = None, stream=None):
        self.step = self.step + 1 if step is None else step
        abi.picasso_packed_lookup_bwd_update(self.ctx, grad_out, lr, self.step, stream,
                                             batch=getattr(self, "_batch", None), out_width=self.out_width,
                                             device=self.device)

    # ---- D-Interleaving (include/picasso.h section 8)
    def dinterleave_begin(self, stream=None):
        abi.picasso_dinterleave_begin(self.ctx, stream)

    def backward_accumulate(self, grad_out: torch.Tensor, stream=None):
        """The last forward's micro-batch: its G rows added to the step accumulator."""
        abi.picasso_packed_lookup_bwd_accumulate(self.ctx, grad_out, stream, batch=getattr(self, "_batch", None),
                                                 out_width=self.out_width, device=self.device)

    def dinterleave_apply(self, lr: float, step: int | None = None, stream=None):
        self.step = self.step + 1 if step is None else step
        abi.picasso_dinterleave_apply(self.ctx, lr, self.step, stream)

    def dinterleave_stats(self):
        return abi.picasso_dinterleave_stats(self.ctx)

    def check(self):
        st, msg = abi.picasso_last_error(self.ctx)
        if st != 0:
            raise abi.PicassoError(st, "device", msg)

    def unique(self, pack):
        return abi.picasso_get_unique(self.ctx, pack, self.device)

    def inverse(self, pack):
        return abi.picasso_get_inverse(self.ctx, pack, self.device)

    def unique_offsets(self, dst=None, stream=None):
        """int32 [n_packs+1] uid prefix of the last forward, copied into dst (enqueue only)."""
        if dst is None:
            dst = torch.empty(self.n_packs + 1, dtype=torch.int32, device=self.device)
        return abi.picasso_unique_offsets(self.ctx, dst, stream)

    def unique_offsets_host(self):
        o = self.unique_offsets()
        return o.cpu().numpy()

    def launch_count(self):
        return abi.picasso_launch_count(self.ctx)

    def owner_unique(self, pack):
        return abi.picasso_get_owner_unique(self.ctx, pack, self.device)

    def hot_cache_refresh(self, capacity_bytes, stream=None):
        """Alg. 1 L514-517 (collective over the ranks in NCCL mode); returns the cache stats."""
        return abi.picasso_hot_cache_refresh(self.ctx, capacity_bytes, stream)

    def hot_keys(self):
        return abi.picasso_get_hot_keys(self.ctx)

    def send_list(self, owner, pack):
        """Local rows this rank requested from `owner` for `pack` in the last forward (send order)."""
        return abi.picasso_get_send_list(self.ctx, owner, pack)

    def send_counts(self):
        return abi.picasso_get_send_counts(self.ctx, self.world)

    def close(self):
        if self.ctx:
            abi.picasso_ctx_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class LoopbackGroup:
    """W ranks of the row-sharded layer in ONE process on one device (nccl_uid = None).  With
    exchange="p2p" the step runs the peer-memory kernels on the ranks' windows (plain pointers,
    the host ordering the phases); with "nccl" the exchanges are device copies between the ranks'
    buffers.  Used to test the sharded path at W up to 8 with a single GPU."""

    def __init__(self, world, field_to_table, table_rows, table_dim, exchange=None, **kw):
        self.world = world
        self.exchange = exchange or default_exchange()
        self.ranks = [PackedEmbedding(field_to_table, table_rows, table_dim, rank=r, world=world,
                                      exchange=self.exchange, **kw) for r in range(world)]
        self.group = abi.picasso_group_create([e.ctx for e in self.ranks])
        if self.exchange == "p2p":  # the peer-memory kernels, windows as plain pointers
            abi.picasso_group_p2p(self.group)

    def forward(self, ids, offsets, batch, outs=None, stream=None):
        if outs is None:
            outs = [torch.empty(b, e.out_width, dtype=torch.float32, device=e.device) for b, e in zip(batch, self.ranks)]
        abi.picasso_group_fwd(self.group, ids, offsets, batch, outs, stream)
        return outs

    def backward_update(self, grad_outs, lr, step, stream=None):
        abi.picasso_group_bwd_update(self.group, grad_outs, lr, step, stream)

    def hot_cache_refresh(self, capacity_bytes, stream=None):
        return abi.picasso_group_hot_cache_refresh(self.group, self.world, capacity_bytes, stream)

    def close(self):
        if self.group:
            abi.picasso_group_destroy(self.group)
            self.group = None
        for e in self.ranks:
            e.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
