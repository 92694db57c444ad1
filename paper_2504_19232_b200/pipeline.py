"""Pipeline driver: builds stages, links and executors through the C-ABI and
runs iterations under a schedule arm (1F1B / ZB / adaptive) with injected
link latencies.  Control plane only (torch for memory and streams,
torch.distributed gloo for handle exchange / schedule broadcast / barriers);
every F/B/W, transfer and the schedule itself run in libadaptra.so.

Stage -> rank placement: contiguous, stage i on rank floor(i * world / S);
one process per GPU (rank r uses cuda:local_rank).
"""
from __future__ import annotations

import ctypes as C
import os
import secrets
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from . import sched as cs
from .stage import Stage


@dataclass
class ModelCfg:
    block: str = "gpt"          # "gpt" | "mlp"
    n_layers: int = 24          # total blocks, split evenly over stages
    d: int = 2048
    d_ff: int = 8192
    n_heads: int = 16
    b: int = 1                  # sequences per microbatch
    T: int = 2048               # tokens per sequence
    dtype: int = L.BF16

    @property
    def tokens_per_mb(self):
        return self.b * self.T


@dataclass
class IterResult:
    epoch: int
    stats: dict                  # stage -> IterStats fields (+ op_times)
    loss: float | None = None


def _op_array(ops):
    arr = (L.Op * max(1, len(ops)))()
    for q, (k, mb) in enumerate(ops):
        arr[q].kind = cs.KIND_ID[k]
        arr[q].mb = mb
    return arr


class Pipeline:
    def __init__(self, model: ModelCfg, S: int, N: int, *, params=None, inputs=None, targets=None,
                 rank: int = 0, world: int = 1, device: int = 0, group=None, link_mode: int = L.LINK_DIRECT,
                 host_links: bool = True, n_slots=None, n_slots_fb=None, seed: int = 0):
        if model.n_layers % S:
            raise ValueError("n_layers must divide evenly over stages")
        self.model, self.S, self.N = model, S, N
        self.rank, self.world, self.group = rank, world, group
        self.dev = device
        torch.cuda.set_device(device)
        self.Ls = model.n_layers // S
        self.stage_rank = [i * world // S for i in range(S)]
        self.local = [i for i in range(S) if self.stage_rank[i] == rank]
        self.msg_bytes = model.tokens_per_mb * model.d * (2 if model.dtype == L.BF16 else 4)
        lib = L.lib()
        # With 8 stages sharing this GPU, persistent GEMMs take half the SMs:
        # the other stages fill the rest and each CTA amortises its prologue and
        # last epilogue over twice the tiles (8 co-located stages: +1 % tokens/s
        # at a 9 % lower SM clock under the power cap,
        # profiles/r02_gemm_sms_step_ab.txt).  $ADAPTRA_GEMM_SMS overrides.
        if "ADAPTRA_GEMM_SMS" in os.environ:
            L.check(lib.adaptra_set_tuning(L.TUNE_GEMM_SMS, int(os.environ["ADAPTRA_GEMM_SMS"])))
        elif len(self.local) >= 8:     # measured with 8 co-located stages only
            n_sm = torch.cuda.get_device_properties(device).multi_processor_count
            L.check(lib.adaptra_set_tuning(L.TUNE_GEMM_SMS, n_sm // 2))
        if "ADAPTRA_ATTN_SMS" in os.environ:
            L.check(lib.adaptra_set_tuning(L.TUNE_ATTN_SMS, int(os.environ["ADAPTRA_ATTN_SMS"])))
        block = L.BLOCK_GPT if model.block == "gpt" else L.BLOCK_MLP
        # ---------------- stages
        self.stages = {}
        for i in self.local:
            ns = n_slots[i] if isinstance(n_slots, (list, tuple)) else (n_slots or N)
            nf = n_slots_fb[i] if isinstance(n_slots_fb, (list, tuple)) else (n_slots_fb or ns)
            st = Stage(block, model.dtype, self.Ls, model.d, model.d_ff, model.n_heads, model.b, model.T,
                       i == 0, i == S - 1, N, ns, f"cuda:{device}", n_slots_fb=nf)
            if params is not None:
                st.load_params(params[i])
            else:
                self._init_params(st, i, seed)
            self.stages[i] = st
        # ---------------- io
        tdt = torch.bfloat16 if model.dtype == L.BF16 else torch.float32  # (a rank may host no stage: S < world)
        R = model.tokens_per_mb
        self.inputs, self.targets = [], []
        if 0 in self.stages:
            if inputs is not None:
                self.inputs = [torch.from_numpy(np.asarray(x, np.float32).reshape(R, model.d)).to(
                    f"cuda:{device}", tdt) for x in inputs]
            else:
                g = torch.Generator(device=f"cuda:{device}").manual_seed(seed + 1)
                self.inputs = [torch.randn(R, model.d, device=f"cuda:{device}", generator=g).to(tdt)
                               for _ in range(N)]
        if S - 1 in self.stages:
            if targets is not None:
                self.targets = [torch.from_numpy(np.asarray(t, np.float32).reshape(R, model.d)).to(
                    f"cuda:{device}") for t in targets]
            else:
                g = torch.Generator(device=f"cuda:{device}").manual_seed(seed + 2)
                self.targets = [torch.randn(R, model.d, device=f"cuda:{device}", generator=g) for _ in range(N)]
            self.loss = torch.zeros(1, device=f"cuda:{device}")
        # ---------------- links: inboxes on receivers, outboxes on senders
        token = self._bcast(secrets.token_hex(4) if rank == 0 else None)
        self._host_names = {}
        self.in_fwd, self.in_bwd, self.out_fwd, self.out_bwd = {}, {}, {}, {}
        exports = {}
        for i in self.local:
            if i > 0:
                nm = f"/adaptra_{token}_{i - 1}_f" if host_links else None
                h = C.c_void_p()
                L.check(lib.adaptra_inbox_create(device, N, self.msg_bytes, nm.encode() if nm else None,
                                                 C.byref(h)))
                self.in_fwd[i] = h
                exports[("f", i - 1)] = (self._export(h), nm)
            if i < S - 1:
                nm = f"/adaptra_{token}_{i}_b" if host_links else None
                h = C.c_void_p()
                L.check(lib.adaptra_inbox_create(device, N, self.msg_bytes, nm.encode() if nm else None,
                                                 C.byref(h)))
                self.in_bwd[i] = h
                exports[("b", i)] = (self._export(h), nm)
        all_exports = self._allgather(exports)
        for i in self.local:
            if i < S - 1:   # forward link i -> inbox of stage i+1
                self.out_fwd[i] = self._open_out(i + 1, self.in_fwd, ("f", i), all_exports, link_mode)
            if i > 0:       # backward link i-1 -> inbox of stage i-1
                self.out_bwd[i] = self._open_out(i - 1, self.in_bwd, ("b", i - 1), all_exports, link_mode)
        # ---------------- executors
        self.streams, self.execs = {}, {}
        self._keep = []
        for i in self.local:
            s = torch.cuda.Stream(device=device)
            self.streams[i] = s
            d = L.ExecDesc()
            d.stage = self.stages[i].handle
            d.stage_index, d.n_stages, d.n_microbatches = i, S, N
            d.in_fwd = self.in_fwd.get(i)
            d.in_bwd = self.in_bwd.get(i)
            d.out_fwd = self.out_fwd.get(i)
            d.out_bwd = self.out_bwd.get(i)
            d.compute_stream = s.cuda_stream
            if i == 0:
                arr = (C.c_void_p * N)(*[t.data_ptr() for t in self.inputs])
                self._keep.append(arr)
                d.inputs = arr
            if i == S - 1:
                arr = (C.c_void_p * N)(*[t.data_ptr() for t in self.targets])
                self._keep.append(arr)
                d.targets = arr
                d.loss_acc = self.loss.data_ptr()
            h = C.c_void_p()
            L.check(lib.adaptra_exec_create(C.byref(d), C.byref(h)))
            self.execs[i] = h
        # one time base for all stages of this rank (one device)
        self._base_stream = torch.cuda.Stream(device=device)
        self._base_event = torch.cuda.Event(enable_timing=True)
        for i in self.local:
            L.check(lib.adaptra_exec_set_time_base(self.execs[i], C.c_void_p(self._base_event.cuda_event)))
        self.epoch = 0
        self.latency = [0] * (S - 1)
        torch.cuda.synchronize(device)
        self._barrier()

    # ------------------------------------------------------------ setup helpers
    def _init_params(self, st: Stage, i: int, seed: int):
        """GPT-2 init drawn on the device (bench sizes): weights N(0, 0.02), output
        projections scaled by 1/sqrt(2 n_layers); LN gamma 1, beta 0; biases 0."""
        m = self.model
        g = torch.Generator(device=st.device).manual_seed(seed * 1000 + i)
        w = torch.randn(st.wts.numel(), device=st.device, generator=g) * 0.02
        if m.block == "gpt":
            D, F = m.d, m.d_ff
            per = 3 * D * D + D * D + F * D + D * F
            ro = 1.0 / (2.0 * m.n_layers) ** 0.5
            for l in range(self.Ls):
                o = l * per
                w[o + 3 * D * D:o + 4 * D * D] *= ro                       # Wo
                w[o + 4 * D * D + F * D:o + per] *= ro                     # W2
        st.wts.copy_(w.to(st.tdt))
        v = torch.zeros(st.vecs.numel(), device=st.device)
        if m.block == "gpt":
            per = 2 * m.d + 3 * m.d + m.d + 2 * m.d + m.d_ff + m.d
            for l in range(self.Ls):
                o = l * per
                v[o:o + m.d] = 1.0                            # ln1_g
                v[o + 6 * m.d:o + 7 * m.d] = 1.0              # ln2_g
        st.vecs.copy_(v)

    def _export(self, h):
        buf = (C.c_uint8 * L.IPC_BYTES)()
        L.check(L.lib().adaptra_inbox_export(h, buf))
        return bytes(buf)

    def _open_out(self, peer_stage, local_inboxes, key, all_exports, mode):
        lib = L.lib()
        h = C.c_void_p()
        if self.stage_rank[peer_stage] == self.rank:
            L.check(lib.adaptra_outbox_open_local(self.dev, local_inboxes[peer_stage], mode, C.byref(h)))
        else:
            handle, nm = all_exports[key]
            hb = (C.c_uint8 * L.IPC_BYTES)(*handle)
            L.check(lib.adaptra_outbox_open_ipc(self.dev, hb, self.N, self.msg_bytes,
                                                nm.encode() if nm else None, mode, C.byref(h)))
        return h

    def _bcast(self, obj):
        if self.world == 1:
            return obj
        import torch.distributed as dist
        lst = [obj]
        dist.broadcast_object_list(lst, src=0, group=self.group)
        return lst[0]

    def _allgather(self, d):
        if self.world == 1:
            return dict(d)
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, d, group=self.group)
        merged = {}
        for x in out:
            merged.update(x)
        return merged

    def _barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier(group=self.group)

    # ------------------------------------------------------------ control
    def set_latency(self, link: int, ns: int):
        """Inject latency c_link (ns) or L.LINK_DOWN on both directions of `link`."""
        lib = L.lib()
        self.latency[link] = ns
        if link in self.out_fwd:
            L.check(lib.adaptra_set_link_latency(self.out_fwd[link], ns))
        if link + 1 in self.out_bwd:
            L.check(lib.adaptra_set_link_latency(self.out_bwd[link + 1], ns))
        down = 1 if (ns == L.LINK_DOWN or link in getattr(self, "on_host", set())) else 0
        if link + 1 in self.in_fwd:
            L.check(lib.adaptra_inbox_set_host(self.in_fwd[link + 1], down))
        if link in self.in_bwd:
            L.check(lib.adaptra_inbox_set_host(self.in_bwd[link], down))

    def enable_nccl(self, down_ns=0):
        """N1 baseline: one NCCL communicator over all ranks for the
        ADAPTRA_EXEC_NCCL arms (one stage per rank: NCCL refuses two ranks on a
        device, and one communicator must not be driven by two stage threads)."""
        if getattr(self, "_nccl", None):
            return
        if len(self.local) != 1 or self.S != self.world:
            raise ValueError("the NCCL baseline needs exactly one stage per rank (S == world)")
        lib = L.lib()
        uid = (C.c_uint8 * L.NCCL_ID_BYTES)()
        if self.rank == 0:
            L.check(lib.adaptra_nccl_unique_id(uid))
        raw = self._bcast(bytes(uid))
        uid = (C.c_uint8 * L.NCCL_ID_BYTES)(*raw)
        comm = C.c_void_p()
        L.check(lib.adaptra_nccl_comm_init(uid, self.world, self.rank, self.dev, C.byref(comm)))
        self._nccl = comm
        i = self.local[0]
        prev = self.stage_rank[i - 1] if i > 0 else -1
        nxt = self.stage_rank[i + 1] if i < self.S - 1 else -1
        L.check(lib.adaptra_exec_set_nccl(self.execs[i], comm, prev, nxt, int(down_ns)))
        self.nccl_buffered = self._probe_nccl_buffering()

    def _probe_nccl_buffering(self, wait_s=0.5):
        """R39: how many messages of msg_bytes a link holds before a posted
        receive.  Rank 0 issues m = max(16, N) sends to rank 1 while rank 1
        posts nothing; after wait_s the sends that completed are the buffered
        count K.  Then rank 1 posts the m receives (nothing is left blocked)
        and K goes to every rank.  The NCCL arm's receive plan assumes K - 1
        (a margin), or no limit when all m completed (a link never carries
        more than N messages per iteration)."""
        import time
        m = max(16, self.N)
        lib = L.lib()
        k = 0
        if self.rank in (0, 1):
            dev = torch.device("cuda", self.dev)
            st = torch.cuda.Stream(device=dev)
            buf = [torch.empty(self.msg_bytes, dtype=torch.uint8, device=dev) for _ in range(m)]
            # one matched message first: NCCL connects peers lazily, on both sides
            L.check(lib.adaptra_nccl_p2p(self._nccl, int(self.rank == 0), C.c_void_p(buf[0].data_ptr()),
                                         self.msg_bytes, 1 - self.rank, C.c_void_p(st.cuda_stream)))
            st.synchronize()
            if self.rank == 0:
                evs = []
                for b in buf:
                    L.check(lib.adaptra_nccl_p2p(self._nccl, 1, C.c_void_p(b.data_ptr()), self.msg_bytes, 1,
                                                 C.c_void_p(st.cuda_stream)))
                    e = torch.cuda.Event()
                    e.record(st)
                    evs.append(e)
                time.sleep(wait_s)
                k = sum(1 for e in evs if e.query())
            self._barrier()
            if self.rank == 1:
                for b in buf:
                    L.check(lib.adaptra_nccl_p2p(self._nccl, 0, C.c_void_p(b.data_ptr()), self.msg_bytes, 0,
                                                 C.c_void_p(st.cuda_stream)))
            st.synchronize()
        else:
            self._barrier()
        k = int(self._bcast(k))
        self.nccl_probe = k
        return 1 << 20 if k >= m else max(0, k - 1)

    def set_path(self, link: int, host: bool):
        """Delegation policy: move both directions of `link` to
        the delegated host path while it is up (host=True) or back (False)."""
        lib = L.lib()
        self.on_host = getattr(self, "on_host", set())
        if (link in self.on_host) == bool(host):
            return
        p = L.PATH_HOST if host else L.PATH_GPU
        if link in self.out_fwd:
            L.check(lib.adaptra_link_set_path(self.out_fwd[link], p))
        if link + 1 in self.out_bwd:
            L.check(lib.adaptra_link_set_path(self.out_bwd[link + 1], p))
        on = 1 if (host or self.latency[link] == L.LINK_DOWN) else 0
        if link + 1 in self.in_fwd:
            L.check(lib.adaptra_inbox_set_host(self.in_fwd[link + 1], on))
        if link in self.in_bwd:
            L.check(lib.adaptra_inbox_set_host(self.in_bwd[link], on))
        (self.on_host.add if host else self.on_host.discard)(link)

    def run(self, orders, merge_w=False, want_times=False, inorder=False, nccl=False):
        """One iteration.  orders[i] = [(kind, mb), ...] for every stage i (only
        local stages are executed here).  Returns IterResult with local stats."""
        lib = L.lib()
        # Iteration boundary across ranks (the optimizer-step boundary of real
        # training): the receiver's W of the previous iteration still reads
        # its inbox slots (x_in / dy_in alias the mailboxes until W), so no
        # sender may start writing them for the next iteration before every
        # rank has finished the previous one (write-after-read across ranks).
        self._barrier()
        self.epoch += 1
        flags = (L.MERGE_W if merge_w else 0) | (L.EXEC_INORDER if inorder else 0) | (L.EXEC_NCCL if nccl else 0)
        self._base_event.record(self._base_stream)
        keep = []
        if nccl:
            # R39: receive-posting plan of the blocking NCCL groups, from all
            # stages' orders (adaptra_nccl_post_plan)
            post = cs.nccl_post_plan(orders, merge_w, getattr(self, "nccl_buffered", 0))
            for i in self.local:
                sl = (C.c_int32 * max(1, len(post[i])))(*post[i])
                L.check(lib.adaptra_exec_set_nccl_post(self.execs[i], sl, len(post[i])))
        for i in self.local:
            arr = _op_array(orders[i])
            keep.append(arr)
            L.check(lib.adaptra_run_iteration(self.execs[i], arr, len(orders[i]), self.epoch, flags))
        errs = []
        for i in self.local:
            rc = lib.adaptra_exec_join(self.execs[i])
            if rc != L.OK:
                errs.append((i, rc, lib.adaptra_last_error().decode()))
        if errs:
            self.abort()
            raise L.AdaptraError(errs[0][1], f"stage {errs[0][0]}: {errs[0][2]}")
        stats = {}
        for i in self.local:
            s = L.IterStats()
            n = len(orders[i])
            times = (C.c_int64 * (2 * max(1, n)))()
            rc = lib.adaptra_exec_wait(self.execs[i], C.byref(s), times)
            if rc != L.OK:
                msg = lib.adaptra_last_error().decode()
                self.abort()
                raise L.AdaptraError(rc, f"stage {i}: {msg}")
            st = {"busy_ns": s.busy_ns, "first_start_ns": s.first_start_ns, "last_end_ns": s.last_end_ns,
                  "op_ns": list(s.op_ns), "op_cnt": list(s.op_cnt), "host_enqueue_ns": s.host_enqueue_ns}
            if want_times:
                st["op_times"] = [(times[2 * q], times[2 * q + 1]) for q in range(n)]
            stats[i] = st
        if self.S - 1 not in self.stages:
            loss = None
        elif getattr(self, "_host_loss", None) is not None:
            loss = float(self._host_loss[0])          # already copied back by the executor
        else:
            loss = float(self.loss.item())
        return IterResult(self.epoch, stats, loss)

    def set_host_io(self, on=True):
        """End-to-end mode (adaptra_exec_set_host_io): the inputs come from
        pinned host memory every iteration (H2D inside the executor, overlapped
        with the pipeline) and the loss goes back to pinned host memory.
        Returns (h2d_bytes, d2h_bytes) per iteration on this rank."""
        lib = L.lib()
        self._host_in, self._host_loss = None, None
        h2d = d2h = 0
        if 0 in self.stages:
            if on:
                self._host_in = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in self.inputs]
                for h, t in zip(self._host_in, self.inputs):
                    h.copy_(t)
                arr = (C.c_void_p * self.N)(*[h.data_ptr() for h in self._host_in])
                self._keep.append(arr)
                nbytes = self.inputs[0].numel() * self.inputs[0].element_size()
                h2d = nbytes * self.N
                L.check(lib.adaptra_exec_set_host_io(self.execs[0], arr, nbytes, None))
            else:
                L.check(lib.adaptra_exec_set_host_io(self.execs[0], None, 0, None))
        if self.S - 1 in self.stages:
            if on:
                self._host_loss = torch.zeros(1, dtype=torch.float32, pin_memory=True)
                d2h = 4
            L.check(lib.adaptra_exec_set_host_io(self.execs[self.S - 1], None, 0,
                                                 C.c_void_p(self._host_loss.data_ptr()) if on else None))
        return h2d, d2h

    def enable_offload(self, host_slots, window=4):
        """N4: give every local stage a pinned host pool of `host_slots` F->W
        stash slots (adaptra_exec_set_offload); the device keeps n_slots."""
        lib = L.lib()
        self._host_pools = getattr(self, "_host_pools", {})
        for i in self.local:
            hs = host_slots[i] if isinstance(host_slots, (list, tuple)) else host_slots
            if hs > 0:
                pool = torch.empty(hs * self.stages[i].slot_bytes, dtype=torch.uint8, pin_memory=True)
                self._host_pools[i] = pool
                L.check(lib.adaptra_exec_set_offload(self.execs[i], C.c_void_p(pool.data_ptr()), hs, window))
            else:
                self._host_pools.pop(i, None)
                L.check(lib.adaptra_exec_set_offload(self.execs[i], None, 0, window))

    def offload_stats(self):
        lib = L.lib()
        out = {}
        for i in self.local:
            a, b, c = C.c_int32(), C.c_int32(), C.c_int64()
            L.check(lib.adaptra_exec_offload_stats(self.execs[i], C.byref(a), C.byref(b), C.byref(c)))
            out[i] = (a.value, b.value, c.value)
        return out

    def profile(self, k=5, quantum=1000):
        """a1: per-stage (t^F, t^B, t^W) in ns = lower median over the last k
        iterations of each stage's mean op time (adaptra_exec_profile, CUDA
        events), floored to `quantum` ns; gathered over ranks.  Kinds that did
        not run (W under 1F1B) report 0."""
        lib = L.lib()
        loc = {}
        for i in self.local:
            t = (C.c_int64 * 3)()
            L.check(lib.adaptra_exec_profile(self.execs[i], k, quantum, t))
            loc[i] = list(t)
        allp = self._allgather(loc)
        return ([allp[i][0] for i in range(self.S)], [allp[i][1] for i in range(self.S)],
                [allp[i][2] for i in range(self.S)])

    def abort(self):
        """Release every GPU-side wait of this rank (after a failure)."""
        lib = L.lib()
        for h in list(self.in_fwd.values()) + list(self.in_bwd.values()):
            lib.adaptra_inbox_poison(h)
        try:
            torch.cuda.synchronize(self.dev)
        except Exception:
            pass

    def zero_grads(self):
        for i in self.local:
            self.stages[i].zero_grads(self.streams[i])
        torch.cuda.synchronize(self.dev)

    def link_stats(self):
        out = {}
        lib = L.lib()
        for name, boxes in (("fwd", self.out_fwd), ("bwd", self.out_bwd)):
            for i, h in boxes.items():
                n, s, m = C.c_int64(), C.c_int64(), C.c_int64()
                L.check(lib.adaptra_link_stats(h, C.byref(n), C.byref(s), C.byref(m)))
                out[(name, i)] = (n.value, s.value, m.value)
        return out

    def close(self):
        lib = L.lib()
        for h in self.execs.values():
            lib.adaptra_exec_destroy(h)
        self.execs = {}
        if getattr(self, "_nccl", None):
            lib.adaptra_nccl_comm_destroy(self._nccl)
            self._nccl = None
        torch.cuda.synchronize(self.dev)
        for h in list(self.out_fwd.values()) + list(self.out_bwd.values()):
            lib.adaptra_outbox_close(h)
        self.out_fwd, self.out_bwd = {}, {}
        self._barrier()
        for h in list(self.in_fwd.values()) + list(self.in_bwd.values()):
            lib.adaptra_inbox_destroy(h)
        self.in_fwd, self.in_bwd = {}, {}
        for st in self.stages.values():
            st.close()


# ---------------------------------------------------------------- metrics
def iteration_metrics(results, orders):
    """a11 (R15): bubble rates of one executed iteration from the
    executor's per-op CUDA-event times.  results = {stage: stats with
    "op_times"} for every stage (gathered over ranks); orders[i] the stage's
    (kind, mb) list.  T = last op end - first op start over all stages;
    utilisation bubble = 1 - sum busy / (S T); interior bubble = sum of each
    stage's gaps inside its own span / sum of spans."""
    S = len(orders)
    t0 = min(st["op_times"][0][0] for st in results.values() if st["op_times"])
    busy, span = [], []
    T = 0
    for i in range(S):
        times = results[i]["op_times"]
        busy.append(sum(e - s for s, e in times))
        span.append((times[-1][1] - times[0][0]) if times else 0)
        T = max(T, max((e for _, e in times), default=0) - t0)
    util = 1.0 - sum(busy) / (S * T)
    interior = (sum(sp - b for sp, b in zip(span, busy)) / sum(span)) if sum(span) else 0.0
    return {"T_ns": T, "busy_ns": busy, "util_bubble": util, "interior_bubble": interior}


# ---------------------------------------------------------------- schedules
def orders_from(X):
    return [[(k, mb) for (k, mb, _s, _e) in ops] for ops in X]


class Arm:
    """One schedule arm: marshalling around the C planner (adaptra_planner_*,
    R18 / R21 / R26 in csrc/sched/sched.cpp).

    name: "1f1b" | "zb" | "adaptive", optionally suffixed "-inorder" (the same
    orders executed with blocking sends/receives in the compute sequence,
    SURVEY N1: the HOL-blocking baseline).  mem = (M, M^F) selects Alg. 1 for
    the adaptive arm's initial plan (R12), clamped to x_cap (R26)."""

    def __init__(self, name, S, N, tF, tB, tW, *, x_init=None, ratio=30, x_cap=None, mem=None):
        self.inorder = name.endswith("-inorder")
        self.nccl = name.endswith("-nccl")       # N1: NCCL send/recv in the compute sequence
        self.deleg = name.endswith("-deleg")     # straggling links on the delegated host path
        name = name[:-len("-deleg")] if self.deleg else name
        name = name[:-len("-inorder")] if self.inorder else name
        name = name[:-len("-nccl")] if self.nccl else name
        self.name, self.S, self.N = name, S, N
        self.merge_w = name == "1f1b"
        self.planner = cs.Planner(name, S, N, tF, tB, tW, x_init=x_init if name == "adaptive" else None,
                                  x_cap=x_cap if name == "adaptive" else None,
                                  mem=mem if name == "adaptive" else None, ratio=ratio)
        self.orders, self.x, _ = self.planner.step([0] * (S - 1))
        self.x_init = list(self.x)
        self.c = [0] * (S - 1)
        self.last = {"c": list(self.c), "x": list(self.x), "replanned": False}

    @property
    def replans(self):
        return self.planner.info.replans

    @property
    def delta(self):
        return self.planner.info.delta

    def set_profile(self, tF, tB, tW):
        """Adopted at the next re-plan (adaptra_planner_set_profile)."""
        self.planner.set_profile(tF, tB, tW)

    def plan(self, c):
        """Orders for the next iteration given the link latencies c (ns, finite)."""
        x_prev = list(self.x)
        self.orders, self.x, replanned = self.planner.step(c)
        self.c = list(c)
        tF, tB, tW = self.planner.profile
        self.last = {"c": list(c), "x_prev": x_prev, "x": list(self.x), "replanned": replanned,
                     "tF": tF, "tB": tB, "tW": tW, "delta": self.planner.info.delta,
                     "makespan": self.planner.info.makespan}
        return self.orders
