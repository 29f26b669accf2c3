"""Multi-GPU partitioning of the Kascade path.

One process per GPU, ``torch.distributed`` for the plumbing.  The independent
units are (sequence, kv head) in decode and (kv head, tile) in prefill --
pooling and Top-k are per kv head and per tile (runner.py:199-206) -- so:

* **Batch sharding** (decode, first choice): every rank owns whole
  sequences with all heads and layers.  No data-path collective at all.
* **KV-head sharding** (decode when B < #GPUs, 70B-style TP, and prefill):
  rank r owns kv heads [g0, g1) and their G query heads.  The one real
  exchange step is the head remap: a reuse kv head g borrows the anchor list
  of head_map[g] (runner.py:220), which can live on another rank, so every
  anchor layer all-gathers its index lists (B*Hkv*k*4 B -- 3.4 MB at b8/128K)
  and reuse layers read the gathered lists locally.  Head-sharded outputs are
  all-gathered only when the caller wants them reassembled.

The collectives run on whatever backend the process group has (NCCL over
NVLink on the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

from typing import Optional, Tuple

import torch
import torch.distributed as dist

from .exceptions import InvalidArgumentError


def _world(group=None) -> Tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def even_split(n: int, world: int, rank: int) -> Tuple[int, int]:
    """[start, end) of rank's share of n units; shares differ by at most 1."""
    if world < 1 or not 0 <= rank < world:
        raise InvalidArgumentError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def batch_shard(batch: int, group=None) -> Tuple[int, int]:
    """Sequences owned by this rank under batch sharding."""
    world, rank = _world(group)
    return even_split(batch, world, rank)


def kv_head_shard(num_kv_heads: int, group=None) -> Tuple[int, int]:
    """kv heads [g0, g1) owned by this rank under kv-head sharding; requires
    Hkv divisible by the world size so every rank holds whole groups."""
    world, rank = _world(group)
    if num_kv_heads % world:
        raise InvalidArgumentError(f"{num_kv_heads} kv heads do not split over {world} ranks")
    per = num_kv_heads // world
    return rank * per, (rank + 1) * per


def _all_gather_dim0(x: torch.Tensor, world: int, group) -> torch.Tensor:
    """all_gather_into_tensor along dim 0; CUDA tensors on a gloo group are
    staged through host memory (gloo has no CUDA all-gather), which lets the
    multi-process tests share one GPU."""
    stage = x.is_cuda and dist.get_backend(group) == "gloo"
    src = x.cpu() if stage else x
    out = torch.empty((world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src.contiguous(), group=group)
    return out.to(x.device) if stage else out


def gather_index_lists(local_idx: torch.Tensor, local_cnt: torch.Tensor, group=None,
                       head_dim: int = 1) -> Tuple[torch.Tensor, torch.Tensor]:
    """All-gather per-kv-head index lists along ``head_dim`` so every rank
    holds the anchor sets of ALL kv heads (the head-remap exchange).

    decode: idx [B][Hloc][k_cap], cnt [B][Hloc]      (head_dim = 1)
    prefill: idx [Hloc][T][k_cap], cnt [Hloc][T]     (head_dim = 0)
    Ranks are concatenated in rank order, i.e. global kv head order."""
    world, _ = _world(group)
    if world == 1:
        return local_idx, local_cnt

    def cat(t: torch.Tensor) -> torch.Tensor:
        return _all_gather_dim0(t.movedim(head_dim, 0), world, group).movedim(0, head_dim).contiguous()

    return cat(local_idx), cat(local_cnt)


class PendingIndexGather:
    """An index-list all-gather in flight (NCCL: on the communicator's
    stream, ordered after the select that produced the lists).  ``wait()``
    makes the current stream wait for it and returns (idx, cnt) in global
    kv-head order, as gather_index_lists does."""

    def __init__(self, local_idx, local_cnt, group=None, head_dim: int = 1):
        self.head_dim = head_dim
        self.works, self.outs, self.srcs, self.done = [], [], [], None
        world, _ = _world(group)
        if world == 1 or not local_idx.is_cuda or dist.get_backend(group) == "gloo":
            self.done = gather_index_lists(local_idx, local_cnt, group, head_dim)   # staged / trivial: in place
            return
        for t in (local_idx, local_cnt):
            src = t.movedim(head_dim, 0).contiguous()
            out = torch.empty((world * src.shape[0],) + tuple(src.shape[1:]), dtype=src.dtype, device=src.device)
            self.works.append(dist.all_gather_into_tensor(out, src, group=group, async_op=True))
            self.outs.append(out)
            self.srcs.append(src)          # alive until wait(): the collective reads it asynchronously

    def wait(self) -> Tuple[torch.Tensor, torch.Tensor]:
        if self.done is None:
            for w in self.works:
                w.wait()
            self.done = tuple(o.movedim(0, self.head_dim).contiguous() for o in self.outs)
            self.srcs = []
        return self.done


def gather_head_outputs(local_out: torch.Tensor, group=None, head_dim: int = 1) -> torch.Tensor:
    """Reassemble head-sharded outputs (decode [B][Hq_loc][d], head_dim 1;
    prefill [Hq_loc][N][d], head_dim 0)."""
    world, _ = _world(group)
    if world == 1:
        return local_out
    return _all_gather_dim0(local_out.movedim(head_dim, 0), world, group).movedim(0, head_dim)


def local_head_map(head_map, g0: int, g1: int, device=None) -> torch.Tensor:
    """The head-remap entries of this rank's kv heads.  Values stay GLOBAL
    source heads: they index the gathered (all-heads) lists."""
    m = [int(x) for x in head_map]
    return torch.tensor(m[g0:g1], dtype=torch.int32, device=device)


class IndexExchange:
    """The head-remap exchange of one sharded executor with every buffer
    preallocated, so a decode step that contains it can be captured in a
    CUDA graph (NCCL collectives are graph-capturable once the communicator
    exists; the executors run one eager step before capturing).

    ``local_idx`` / ``local_cnt`` are the executor's per-kv-head lists with
    the kv-head axis at ``head_dim``; ``full_idx`` / ``full_cnt`` receive
    the lists of ALL kv heads (global head order = rank order).  With the
    kv-head axis leading (prefill, head_dim 0) the all-gather writes straight
    into ``full_*``; otherwise (decode, head_dim 1) one small copy on each
    side moves the axis."""

    def __init__(self, local_idx, local_cnt, full_idx, full_cnt, group=None, head_dim: int = 1):
        self.group, self.head_dim = group, head_dim
        self.world, _ = _world(group)
        self.local, self.full = (local_idx, local_cnt), (full_idx, full_cnt)
        self.staged = self.world > 1 and (not local_idx.is_cuda or dist.get_backend(group) == "gloo")
        self.works = []
        if self.world == 1 or self.staged:
            return
        if head_dim == 0:
            self.send = self.local
            self.recv = self.full
        else:
            self.send = tuple(torch.empty_like(t.movedim(head_dim, 0).contiguous()) for t in self.local)
            self.recv = tuple(torch.empty((self.world * s.shape[0],) + tuple(s.shape[1:]), dtype=s.dtype,
                                          device=s.device) for s in self.send)

    def start(self) -> None:
        """Enqueue the all-gather behind the select that wrote the local lists."""
        if self.world == 1:
            for f, t in zip(self.full, self.local):
                f.copy_(t)
            return
        if self.staged:                 # gloo (CPU tests): host-staged, synchronous
            idx, cnt = gather_index_lists(*self.local, self.group, self.head_dim)
            self.full[0].copy_(idx)
            self.full[1].copy_(cnt)
            return
        if self.head_dim != 0:
            for s, t in zip(self.send, self.local):
                s.copy_(t.movedim(self.head_dim, 0))
        self.works = [dist.all_gather_into_tensor(r, s, group=self.group, async_op=True)
                      for r, s in zip(self.recv, self.send)]

    def finish(self) -> None:
        """Make the current stream wait for the exchange; full_* then hold it."""
        for w in self.works:
            w.wait()
        self.works = []
        if self.world > 1 and not self.staged and self.head_dim != 0:
            for f, r in zip(self.full, self.recv):
                f.copy_(r.movedim(0, self.head_dim))


class ShardedKascadeDecoder:
    """KV-head-sharded decode executor (one rank's share).

    Anchor layers select on the local kv heads, then all-gather the index
    lists; reuse layers gather through the GLOBAL head map from the gathered
    lists.  q / caches passed to ``step`` are the rank's local head slices.
    Every buffer (including the exchange's) is preallocated, so ``capture``
    records the whole step -- kernels and NCCL all-gathers -- as one CUDA
    graph."""

    def __init__(self, plan, num_layers: int, batch: int, num_q_heads: int, num_kv_heads: int,
                 max_seq_len: int, group=None, device=None):
        from . import engine
        from .host_types import KIND_REUSE, MODE_ALL_HEADS_POOLED, k_budget, validate_plan
        validate_plan(plan, num_layers, num_kv_heads)
        if plan.mode == MODE_ALL_HEADS_POOLED:
            raise InvalidArgumentError("all-heads-pooled mode needs the pooled vectors of every kv head; "
                                       "use batch sharding (SURVEY.md 8(e) mode caveat)")
        self.group = group
        self.g0, self.g1 = kv_head_shard(num_kv_heads, group)
        self.G = num_q_heads // num_kv_heads
        self.Hkv, self.Hloc = num_kv_heads, self.g1 - self.g0
        self.local = engine.KascadeDecoder(plan, num_layers, batch, self.Hloc * self.G, self.Hloc, max_seq_len,
                                           device=device, validate=False)
        dev = self.local.device
        self.kinds = self.local.kinds
        self.maps = {l: local_head_map(plan.head_maps[l].map, self.g0, self.g1, dev)
                     for l, kind in enumerate(self.kinds) if kind == KIND_REUSE}
        # [L][Hloc] table of the reuse layers' maps (rows of other layers unused)
        zeros = torch.zeros(self.Hloc, dtype=torch.int32, device=dev)
        self.map_table = torch.stack([self.maps.get(l, zeros) for l in range(num_layers)]).contiguous()
        kc = k_budget(plan.k_policy, max_seq_len)
        self.full_idx = torch.empty(batch, num_kv_heads, kc, dtype=torch.int32, device=dev)
        self.full_cnt = torch.zeros(batch, num_kv_heads, dtype=torch.int32, device=dev)
        self.exchange = IndexExchange(self.local.indices, self.local.counts, self.full_idx, self.full_cnt,
                                      group, head_dim=1)
        self._graphs = {}

    def step(self, q, k_caches, v_caches, seq_len: int, seq_lens=None) -> torch.Tensor:
        """One decode step on this rank's heads; ``seq_lens`` (device int32
        [B]) runs a ragged batch as in KascadeDecoder.step."""
        from . import ops
        from .host_types import KIND_ANCHOR, KIND_REUSE
        loc = self.local
        loc.seq_lens = seq_lens
        ws = loc.ws
        l = 0
        while l < len(self.kinds):
            kind = self.kinds[l]
            ql, kl, vl = q[l], k_caches[l], v_caches[l]
            if kind == KIND_REUSE:
                # a run of consecutive reuse layers reads the gathered lists
                # through each layer's local -> global map: one multi-layer
                # launch (uniform batch, one cache layout), as in the local step
                end = loc.run_end[l]
                if end - l >= 2 and seq_lens is None and loc._fusable(k_caches, v_caches, l, end):
                    ops.decode_layers(q[l:end], k_caches[l:end], v_caches[l:end], seq_len, out=loc.out[l:end],
                                      workspace=loc.ws_layers, tables=loc._layer_tables(k_caches, v_caches, l, end),
                                      indices=self.full_idx, counts=self.full_cnt, head_maps=self.map_table[l:end])
                else:
                    for i in range(l, end):
                        ops.sparse_decode(q[i], k_caches[i], v_caches[i], seq_len, self.full_idx, self.full_cnt,
                                          self.maps[i], out=loc.out[i], workspace=ws)
                l = end
                continue
            ge = loc.group_end.get(l, l + 1) if kind == KIND_ANCHOR else l + 1
            if ge - l >= 2 and seq_lens is None and not loc.pre and loc._fusable(k_caches, v_caches, l, ge):
                # consecutive anchors as one group (as the local step): one
                # score launch, one select over their (sequence, kv head) rows
                # (layer l + i into list slot m - 1 - i), ONE all-gather of the
                # last anchor's lists (slot 0, what the reuse layers read),
                # overlapping the group's sparse launch over its own sets
                m, B, Hs = ge - l, loc.B, loc.indices.shape[1]
                tabs = loc._layer_tables(k_caches, v_caches, l, ge)
                sc_ls = loc.scores_g.stride(0) * B
                ops.decode_layers(q[l:ge], k_caches[l:ge], v_caches[l:ge], seq_len, workspace=loc.ws_layers,
                                  tables=tabs, scores=loc.scores_g[(m - 1) * B:m * B], scores_layer_stride=-sc_ls,
                                  lse=loc.lse_g[(m - 1) * B:m * B], lse_layer_stride=-B * loc.Hq)
                ops.select_decode(loc.scores_g[:m * B], loc.lse_g[:m * B], seq_len, loc.plan.k_policy, loc.Hkv,
                                  indices=loc.idx_g[:m].view(m * B, Hs, -1), counts=loc.cnt_g[:m].view(m * B, Hs),
                                  pooled=loc.pooled_g[:m * B * Hs])
                self.exchange.start()
                ops.decode_layers(q[l:ge], k_caches[l:ge], v_caches[l:ge], seq_len, out=loc.out[l:ge],
                                  workspace=loc.ws_layers, tables=tabs, indices=loc.idx_g[m - 1],
                                  counts=loc.cnt_g[m - 1], index_layer_stride=-loc.idx_g.stride(0),
                                  count_layer_stride=-loc.cnt_g.stride(0))
                self.exchange.finish()
                l = ge
                continue
            loc._anchor_select(l, kind, ql, kl, vl, seq_len, loc.out[l])
            # the exchange overlaps the anchor's own sparse pass, which only
            # needs this rank's lists
            self.exchange.start()
            if kind == KIND_ANCHOR:
                ops.sparse_decode(ql, kl, vl, seq_len, loc.indices, loc.counts, None, out=loc.out[l], workspace=ws)
            self.exchange.finish()
            l += 1
        return loc.out

    def capture(self, q, k_caches, v_caches, seq_len: int, dense: bool = False, seq_lens=None):
        """The whole sharded step (kernels + index-list all-gathers) as one
        CUDA graph; ``dense`` captures the local Top-k = 100% baseline."""
        if dense:
            return self.local.capture(q, k_caches, v_caches, seq_len, dense=True, seq_lens=seq_lens)
        self.step(q, k_caches, v_caches, seq_len, seq_lens)   # communicator + kernel attributes outside capture
        torch.cuda.synchronize()
        if self.exchange.staged:
            raise InvalidArgumentError("a gloo-staged exchange cannot be captured (NCCL only)")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(q, k_caches, v_caches, seq_len, seq_lens)
        self._graphs[(seq_len, dense)] = g
        return g

    def gather_outputs(self) -> torch.Tensor:
        """[L][B][Hq][d] reassembled from every rank's heads."""
        return gather_head_outputs(self.local.out, self.group, head_dim=2)


class ShardedKascadePrefill:
    """KV-head-sharded prefill executor (one rank's share; SURVEY.md 8(e)
    prefill partitioning).  Each anchor layer selects on the local kv heads
    and all-gathers its per-(kv head, tile) lists (<= 205 MiB per layer at
    128K over 8 heads) straight into the all-heads list buffer; reuse layers
    gather through the GLOBAL head map."""

    def __init__(self, plan, num_layers: int, num_q_heads: int, num_kv_heads: int, seq_len: int, group=None,
                 device=None):
        from . import engine
        from .host_types import KIND_REUSE, MODE_ALL_HEADS_POOLED, validate_plan
        validate_plan(plan, num_layers, num_kv_heads)
        if plan.mode == MODE_ALL_HEADS_POOLED:
            raise InvalidArgumentError("all-heads-pooled mode needs every kv head's pooled vectors; "
                                       "use q-tile or batch partitioning (SURVEY.md 8(e) mode caveat)")
        self.group = group
        self.g0, self.g1 = kv_head_shard(num_kv_heads, group)
        self.G = num_q_heads // num_kv_heads
        self.Hkv, self.Hloc = num_kv_heads, self.g1 - self.g0
        self.local = engine.KascadePrefill(plan, num_layers, self.Hloc * self.G, self.Hloc, seq_len, device=device,
                                           validate=False)
        dev = self.local.device
        self.kinds = self.local.kinds
        self.maps = {l: local_head_map(plan.head_maps[l].map, self.g0, self.g1, dev)
                     for l, kind in enumerate(self.kinds) if kind == KIND_REUSE}
        # [L][Hloc] table of the reuse layers' maps (rows of other layers unused)
        zeros = torch.zeros(self.Hloc, dtype=torch.int32, device=dev)
        self.map_table = torch.stack([self.maps.get(l, zeros) for l in range(num_layers)]).contiguous()
        T, kc = self.local.indices.shape[1], self.local.indices.shape[2]
        self.full_idx = torch.empty(num_kv_heads, T, kc, dtype=torch.int32, device=dev)
        self.full_cnt = torch.zeros(num_kv_heads, T, dtype=torch.int32, device=dev)
        self.exchange = IndexExchange(self.local.indices, self.local.counts, self.full_idx, self.full_cnt,
                                      group, head_dim=0)

    def forward(self, qs, ks, vs) -> torch.Tensor:
        """qs/ks/vs: this rank's head slices per layer ([Hq_loc][N][128] and
        [Hloc][N][128]).  Returns the local outputs [L][Hq_loc][N][128]."""
        from . import ops
        from .host_types import KIND_ANCHOR, KIND_REUSE
        loc = self.local
        for l, kind in enumerate(self.kinds):
            q, k, v = qs[l], ks[l], vs[l]
            if kind == KIND_REUSE:
                ops.sparse_prefill(q, k, v, self.full_idx, self.full_cnt, self.maps[l], out=loc.out[l])
                continue
            loc._anchor_select(kind, q, k, v, loc.out[l])
            self.exchange.start()
            if kind == KIND_ANCHOR:           # overlaps the exchange: own lists only
                ops.sparse_prefill(q, k, v, loc.indices, loc.counts, None, out=loc.out[l])
            self.exchange.finish()
        return loc.out

    def gather_outputs(self) -> torch.Tensor:
        """[L][Hq][N][d] reassembled from every rank's heads."""
        return gather_head_outputs(self.local.out, self.group, head_dim=1)
