"""Public Python API of the cold-start engine (thin: buffers, streams and wiring via torch; every
step of the method runs in libpipeboost.so through the C ABI in _binding).

    plan   = Plan(model, adapters, n_gpus, policy="stage", vocab_sliced=0, chunk_bytes=32 << 20)
    eng    = RankEngine(plan, rank, host_base, host_adapters, max_batch=1, max_seq=128)
    eng.wire_local([...]) | eng.wire_ipc(blobs)          # N > 1
    toks   = eng.cold_start(epoch, tokens, adapter_id=0)  # a1..a5 for this rank; rank 0 gets the tokens

One process per GPU (torch.distributed for the handle exchange), or several ranks driven from one
process (logical ranks on one device for tests, or one process driving N devices).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _binding as B


class Plan:
    """pb_plan: immutable layer-to-GPU assignment, load and receive orders."""

    def __init__(self, model, adapters: Sequence, n_gpus: int, policy: str = "stage", vocab_sliced: int = 0,
                 chunk_bytes: int = 32 << 20, prefill_chunks: int = 1, host_alias_layers: int = 0):
        self.model = model
        self.adapters = tuple(adapters)
        self.n_gpus = n_gpus
        self.opts = B.plan_opts(policy, vocab_sliced, chunk_bytes, prefill_chunks, host_alias_layers)
        self.handle = B.pb_plan_create(model, self.adapters, n_gpus, self.opts)
        self.sizes = B.pb_plan_sizes(self.handle)

    def dump(self) -> str:
        return B.pb_plan_dump(self.handle)

    def replan(self, alive, resident) -> "Plan":
        """f1: the plan that finishes the cold start on the GPUs still alive. alive[g] 0/1 per GPU;
        resident: uint8 [n_gpus, n_chunks], 1 = GPU g already holds that chunk (never moved again).
        Rank r of the new plan runs on original GPU gpu_of_rank(r)."""
        new = Plan.__new__(Plan)
        new.model, new.adapters = self.model, self.adapters
        new.opts = self.opts
        new.handle = B.pb_plan_replan(self.handle, alive, resident)
        new.sizes = B.pb_plan_sizes(new.handle)
        new.n_gpus = new.sizes.n_gpus
        return new

    def gpu_of_rank(self, rank: int) -> int:
        return B.pb_plan_gpu_of_rank(self.handle, rank)

    def chunks(self):
        """(id, is_adapter, tensor, r0, r1, dev_off, bytes, loader) of every chunk, parsed from the canonical dump."""
        out = []
        for ln in self.dump().splitlines():
            if ln.startswith("chunk "):
                f = ln.split()
                kv = dict(x.split("=", 1) for x in f[3:])
                r0, r1 = kv["rows"][1:-1].split(",")
                out.append((int(f[1]), f[2] == "adapter", int(kv["tensor"]), int(r0), int(r1), int(kv["dev_off"]),
                            int(kv["bytes"]), int(kv["loader"])))
        return out

    def lists(self):
        """Per-rank load and receive lists (chunk ids), parsed from the canonical dump."""
        load, recv = {}, {}
        for ln in self.dump().splitlines():
            if ln.startswith("load ") or ln.startswith("recv "):
                head, _, rest = ln.partition(":")
                kind, g = head.split()
                (load if kind == "load" else recv)[int(g)] = [int(x) for x in rest.split()]
        return [load[g] for g in range(self.sizes.n_gpus)], [recv[g] for g in range(self.sizes.n_gpus)]

    def tensors(self):
        out = []
        for i in range(self.sizes.n_tensors):
            t = B.pb_plan_tensor(self.handle, i)
            out.append((t.name.decode(), t.rows, t.cols, t.host_off, t.layer, t.dev_off))
        return out

    def atensors(self):
        out = []
        for i in range(self.sizes.n_atensors):
            t = B.pb_plan_atensor(self.handle, i)
            out.append((t.name.decode(), t.rows, t.cols, t.off, t.adapter, t.is_B, t.base_tensor, t.base_row0))
        return out

    def workspace_bytes(self, batch: int, seq: int) -> int:
        return B.pb_plan_workspace_bytes(self.handle, batch, seq)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and B is not None and B.pb_plan_free is not None:
            try:
                B.pb_plan_free(h)
            except Exception:
                pass
            self.handle = None


class RankEngine:
    """One rank's pb_ctx plus the device buffers and streams it borrows."""

    def __init__(self, plan: Plan, rank: int, host_base: torch.Tensor, host_adapters: Optional[torch.Tensor],
                 max_batch: int = 1, max_seq: int = 128, device: Optional[torch.device] = None,
                 multi_adapter: bool = False, reuse: Optional["RankEngine"] = None, switchable: bool = False):
        """multi_adapter=True allocates the out-of-place per-adapter copies (PB_MERGE_ALL mode).
        reuse: a (closed or live) engine of the same GPU whose weight / adapter buffers hold what a re-plan
        (Plan.replan) marks as resident — the recovery trial continues in them instead of fresh buffers.
        switchable=True allocates the pristine-base buffer that pb_switch_adapter (f2) re-merges from."""
        self.plan = plan
        self.rank = rank
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        # host_base / host_adapters must be page-locked (torch pin_memory or cudaHostRegister'ed shared memory)
        self.host_base = host_base
        self.host_adapters = host_adapters
        s = plan.sizes
        with torch.cuda.device(self.device):
            if reuse is not None:
                self.weights, self.adapters, self.adapted = reuse.weights, reuse.adapters, reuse.adapted
            else:
                self.weights = torch.empty(s.dev_weight_bytes, dtype=torch.uint8, device=self.device)
                self.adapters = torch.empty(max(s.dev_adapter_bytes, 1), dtype=torch.uint8, device=self.device)
                self.adapted = (torch.empty(s.dev_adapted_bytes, dtype=torch.uint8, device=self.device)
                                if multi_adapter and s.dev_adapted_bytes else None)
            self.backup = (torch.empty(s.dev_backup_bytes, dtype=torch.uint8, device=self.device)
                           if switchable and s.dev_backup_bytes else None)
            ws = plan.workspace_bytes(max_batch, max_seq)
            self.workspace = torch.empty(ws, dtype=torch.uint8, device=self.device)
            # streams: NULL -> the ctx creates five distinct non-blocking streams (torch's stream pool
            # recycles 32 handles, and two ranks sharing a stream can deadlock on readiness waits)
        self.bufs = B.pb_rank_bufs()
        self.bufs.weights = self.weights.data_ptr()
        self.bufs.weights_cap = self.weights.numel()
        self.bufs.adapters = self.adapters.data_ptr() if s.dev_adapter_bytes else None
        self.bufs.adapters_cap = s.dev_adapter_bytes
        self.bufs.adapted = self.adapted.data_ptr() if self.adapted is not None else None
        self.bufs.adapted_cap = self.adapted.numel() if self.adapted is not None else 0
        self.bufs.workspace = self.workspace.data_ptr()
        self.bufs.workspace_cap = self.workspace.numel()
        self.bufs.max_batch = max_batch
        self.bufs.max_seq = max_seq
        self.bufs.stream_h2d[0] = None
        self.bufs.stream_h2d[1] = None
        self.bufs.stream_merge = None
        self.bufs.stream_nvlink = None
        self.bufs.stream_compute = None
        self.bufs.backup = self.backup.data_ptr() if self.backup is not None else None
        self.bufs.backup_cap = self.backup.numel() if self.backup is not None else 0
        ha = host_adapters.data_ptr() if (host_adapters is not None and s.host_adapter_bytes) else None
        with torch.cuda.device(self.device):
            self.ctx = B.pb_ctx_create(plan.handle, rank, host_base.data_ptr(), ha, self.bufs)
        self._out_tokens = np.zeros(max_batch, dtype=np.int32)

    # ---- wiring
    def export(self) -> bytes:
        with torch.cuda.device(self.device):
            return B.pb_ctx_export(self.ctx)

    def wire_ipc(self, blobs: List[bytes]):
        with torch.cuda.device(self.device):
            for r, blob in enumerate(blobs):
                if r != self.rank:
                    B.pb_ctx_import_peer(self.ctx, r, blob)

    def wire_local(self, engines: List["RankEngine"]):
        with torch.cuda.device(self.device):
            for e in engines:
                if e.rank != self.rank:
                    B.pb_ctx_link_local(self.ctx, e.rank, e.ctx)

    # ---- the method
    def invalidate(self):
        """Put the weights buffer in an explicit cold state (0xFF) — not part of a trial."""
        with torch.cuda.device(self.device):
            self.weights.fill_(0xFF)
            self.adapters.fill_(0xFF)
            torch.cuda.synchronize(self.device)

    def enqueue(self, epoch: int, tokens: Optional[np.ndarray], batch: int, seq: int, adapter_id: int = 0,
                adapter_of_seq=None):
        """Enqueue a1..a5 for this rank (non-blocking). tokens [batch, seq] int32 (needed on rank 0).
        adapter_id: adapter merged in place, -1 none, B.PB_MERGE_ALL: all adapters out of place, with
        adapter_of_seq[b] choosing each sequence's adapter (every rank passes the same list)."""
        self._batch = batch
        with torch.cuda.device(self.device):
            B.pb_trial_begin(self.ctx, epoch)
            B.pb_load_shard(self.ctx)
            B.pb_merge_lora(self.ctx, adapter_id)
            B.pb_gather_layers(self.ctx)
            tp = None
            if tokens is not None:
                self._tok = np.ascontiguousarray(tokens, dtype=np.int32)
                assert self._tok.shape == (batch, seq)
                tp = self._tok.ctypes.data
            if adapter_of_seq is None:
                B.pb_prefill_enqueue(self.ctx, tp, batch, seq)
            else:
                self._aos = np.ascontiguousarray(adapter_of_seq, dtype=np.int32)
                B.pb_prefill_enqueue_ex(self.ctx, tp, self._aos.ctypes.data, batch, seq)

    def wait(self, want_logits: bool = False):
        """Block until this rank's trial is done; rank 0 returns (tokens[B], logits[B, V] | None)."""
        with torch.cuda.device(self.device):
            logits, lp, tp = None, None, None
            if self.rank == 0 or getattr(self, "replica", False):
                tp = self._out_tokens.ctypes.data
                if want_logits:
                    logits = np.empty((self._batch, self.plan.model.vocab), dtype=np.float32)
                    lp = logits.ctypes.data
            B.pb_prefill_wait(self.ctx, lp, tp)
            B.pb_sync(self.ctx)
            if self.rank == 0 or getattr(self, "replica", False):
                return self._out_tokens[:self._batch].copy(), logits
            return None, None

    def cold_start(self, epoch: int, tokens: Optional[np.ndarray], batch: int = None, seq: int = None,
                   adapter_id: int = 0, want_logits: bool = False):
        """One cold start on this rank (blocking). With several ranks in ONE process use enqueue() on
        every rank first, then wait() — a rank's device work may wait on its peers' readiness words."""
        if tokens is not None:
            batch, seq = np.asarray(tokens).shape
        self.enqueue(epoch, tokens, batch, seq, adapter_id)
        return self.wait(want_logits)

    def set_file_source(self, path: Optional[str], staging_bytes: int = 256 << 20):
        """f4: read the base weights of later cold starts from the checkpoint file `path` (canonical host layout)
        through a pinned staging ring of `staging_bytes`; None returns to the pinned host image."""
        if path is None:
            B.pb_ctx_set_file_source(self.ctx, None, None, 0)
            self._staging = None
            return
        self._staging = torch.empty(staging_bytes + 4096, dtype=torch.uint8, pin_memory=True)
        base = (self._staging.data_ptr() + 4095) // 4096 * 4096
        with torch.cuda.device(self.device):
            B.pb_ctx_set_file_source(self.ctx, path, base, staging_bytes)

    def decode_enqueue(self, epoch: int):
        """f3: one decode step of the last prefilled batch (every rank, same epoch); complete with wait()."""
        with torch.cuda.device(self.device):
            B.pb_decode_step(self.ctx, epoch)

    def set_replica(self, on: bool = True):
        """f3: serve later batches with the whole model on this GPU (after T_full)."""
        with torch.cuda.device(self.device):
            B.pb_sync(self.ctx)
            B.pb_ctx_set_replica(self.ctx, 1 if on else 0)
        self.replica = on

    def switch_adapter(self, adapter_id: int):
        """f2: re-merge this rank's stage with `adapter_id` (-1: base model) behind the prefills
        already enqueued; serve the next batch with replay_enqueue."""
        with torch.cuda.device(self.device):
            B.pb_switch_adapter(self.ctx, adapter_id)

    def replay_enqueue(self, epoch: int, tokens: Optional[np.ndarray], batch: int, seq: int):
        """Warm prefill re-run on the resident weights (pb_prefill_replay); complete with wait()."""
        self._batch = batch
        with torch.cuda.device(self.device):
            tp = None
            if tokens is not None:
                self._tok = np.ascontiguousarray(tokens, dtype=np.int32)
                tp = self._tok.ctypes.data
            B.pb_prefill_replay(self.ctx, epoch, tp, batch, seq)

    def timeline(self) -> dict:
        t = B.pb_timeline(self.ctx)
        n = t.n_chunks
        return {"t_ready_ms": t.t_ready_ms, "t_full_ms": t.t_full_ms, "ttft_ms": t.ttft_ms,
                "load_done_ms": t.load_done_ms, "load_bytes": t.load_bytes, "recv_bytes": t.recv_bytes,
                "n_launches": t.n_launches,
                "chunk_landed_ms": np.ctypeslib.as_array(t.chunk_landed_ms, shape=(n,)).copy() if n else np.zeros(0),
                "chunk_gathered_ms": np.ctypeslib.as_array(t.chunk_gathered_ms, shape=(n,)).copy() if n else np.zeros(0),
                "chunk_merged_ms": np.ctypeslib.as_array(t.chunk_merged_ms, shape=(n,)).copy() if n else np.zeros(0),
                "stage_begin_ms": t.stage_begin_ms, "stage_end_ms": t.stage_end_ms, "ctx_create_ms": t.ctx_create_ms}

    def arm(self, epoch: int, adapter_id: int = 0):
        """Start a cold start with no prompt yet: a2 load, a3 merge, a4 gather are issued at once (the rank reaches
        T_full on its own); a prompt given later with post_prompt() joins the loads still in flight."""
        with torch.cuda.device(self.device):
            B.pb_trial_begin(self.ctx, epoch)
            B.pb_load_shard(self.ctx)
            B.pb_merge_lora(self.ctx, adapter_id)
            B.pb_gather_layers(self.ctx)

    def post_prompt(self, tokens: Optional[np.ndarray], batch: int, seq: int):
        """a5 for an armed trial (see arm); complete with wait()."""
        self._batch = batch
        with torch.cuda.device(self.device):
            tp = None
            if tokens is not None:
                self._tok = np.ascontiguousarray(tokens, dtype=np.int32)
                tp = self._tok.ctypes.data
            B.pb_prefill_enqueue(self.ctx, tp, batch, seq)

    def sync(self):
        with torch.cuda.device(self.device):
            B.pb_sync(self.ctx)

    def abort(self):
        """f1: abandon the trial after a peer died (pb_ctx_abort); only close() remains."""
        with torch.cuda.device(self.device):
            B.pb_ctx_abort(self.ctx)

    def weights_bytes(self) -> np.ndarray:
        return self.weights.cpu().numpy()

    def close(self):
        if getattr(self, "ctx", None):
            B.pb_ctx_free(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pinned_host(nbytes: int) -> torch.Tensor:
    return torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
