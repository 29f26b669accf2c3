"""Layer-loop executors: the device-side counterpart of run_kascade's loop
(runner.py:228-297) without the reference's always-on dense pass.

``KascadeDecoder.step`` runs one decode step (one query token per sequence)
through every layer of a plan:

  layer 0      dense attention + scores -> pooled Top-k   (anchor0)
  anchor l     scores-only pass -> pooled Top-k -> sparse over its own sets
  reuse l      sparse over the latest anchor's sets routed by head_map[l]

and ``dense_step`` is the Top-k = 100% baseline over the same layers.  All
buffers are preallocated, so a step can be captured once in a CUDA graph
and replayed (``capture``), which removes the per-kernel launch gaps that
dominate the small reuse layers.

On uniform batches with post-softmax pooling, ``step`` issues the anchor
groups' score passes and selections on an internal side stream ahead of the
layer loop (the selections overlap the attention of other layers) and joins
that stream back into the caller's stream before it returns, so the step is
ordered on the caller's stream exactly like a single-stream call (and a
captured graph holds both branches).
"""

from __future__ import annotations

from typing import Dict, List, Optional, Sequence

import torch

from . import ops
from .exceptions import InvalidArgumentError
from .host_types import (KIND_ANCHOR, KIND_ANCHOR0, KIND_REUSE, MODE_ALL_HEADS_POOLED, MODE_REMAPPED,
                         POOL_PRE, k_budget, validate_plan)


def layer_kinds(plan, num_layers: int) -> List[str]:
    anchors = set(plan.core.anchors)
    return [KIND_ANCHOR0 if l == 0 else KIND_ANCHOR if l in anchors else KIND_REUSE
            for l in range(num_layers)]


class KascadeDecoder:
    # output-copy chunk boundaries of capture_host_step (layers; a class
    # attribute, so a caller can set its own).  Measured e2e on B200 (32
    # layers, 128K, b8, same box): 8,16,24 -> 569.7 us/token; 16,24,28,30 ->
    # 568.0; 24,31 -> 567.2 (one copy of the last layer left after the loop).
    D2H_SPLITS = (24, 31)

    def __init__(self, plan, num_layers: int, batch: int, num_q_heads: int, num_kv_heads: int,
                 max_seq_len: int, device=None, validate: bool = True):
        if validate:   # sharded executors validate against the GLOBAL head count themselves
            validate_plan(plan, num_layers, num_kv_heads)
        self.plan = plan
        self.pre = plan.pooling == POOL_PRE     # pre-softmax pooling (runner.py:155-161)
        self.L, self.B, self.Hq, self.Hkv = num_layers, batch, num_q_heads, num_kv_heads
        self.n_max = max_seq_len
        self.device = torch.device(device or "cuda")
        self.kinds = layer_kinds(plan, num_layers)
        self.all_heads = plan.mode == MODE_ALL_HEADS_POOLED
        Hsrc = 1 if self.all_heads else num_kv_heads
        dev = self.device
        self.head_maps: Dict[int, Optional[torch.Tensor]] = {}
        for l, kind in enumerate(self.kinds):
            if kind != KIND_REUSE:
                continue
            if self.all_heads:
                self.head_maps[l] = torch.zeros(num_kv_heads, dtype=torch.int32, device=dev)
            else:
                hm = plan.head_maps[l]
                self.head_maps[l] = torch.tensor(hm.map, dtype=torch.int32, device=dev)
        self.shared_map = torch.zeros(num_kv_heads, dtype=torch.int32, device=dev) if self.all_heads else None
        k_cap = k_budget(plan.k_policy, max_seq_len)
        n_pad = (max_seq_len + 3) // 4 * 4
        # groups of consecutive anchor layers (other than layer 0): they are
        # independent of each other, so a group runs its score passes, its
        # selections and its sparse passes as one launch each; every group
        # member has its own slot of scores / pooled / lists, the LAST anchor
        # in slot 0 (= self.indices, what the following reuse layers read)
        self.group_end: Dict[int, int] = {}
        l = 1
        while l < num_layers:
            e = l
            while e < num_layers and self.kinds[e] == KIND_ANCHOR:
                e += 1
            for i in range(l, e):
                self.group_end[i] = e
            l = max(e, l + 1)
        gmax = 1 if self.pre else max([e - l for l, e in self.group_end.items()] + [1])
        if self.pre:   # q_bar scores -> softmax -> Top-k: no score pass, no per-head score scratch
            self.scores_g = None
            self.pooled, self.pre_ws, _, _ = ops.select_pre_buffers(batch, num_kv_heads, max_seq_len, plan.k_policy,
                                                                    dev, prefill=False, all_heads=self.all_heads,
                                                                    num_q_heads=num_q_heads)
            self.scores = None
        else:
            self.scores_g = torch.empty(gmax * batch, num_q_heads, n_pad, dtype=torch.float32, device=dev)
            self.pooled_g = torch.empty(gmax * batch * Hsrc, n_pad, dtype=torch.float32, device=dev)
            self.scores = self.scores_g[:batch]
            self.pooled = self.pooled_g[:batch * Hsrc]
        self.lse_g = torch.empty(gmax * batch, num_q_heads, dtype=torch.float32, device=dev)
        self.idx_g = torch.empty(gmax, batch, Hsrc, k_cap, dtype=torch.int32, device=dev)
        self.cnt_g = torch.zeros(gmax, batch, Hsrc, dtype=torch.int32, device=dev)
        self.lse = self.lse_g[:batch]
        self.indices = self.idx_g[0]
        self.counts = self.cnt_g[0]
        self.zero_maps = torch.zeros(gmax, num_kv_heads, dtype=torch.int32, device=dev)
        self.out = torch.empty(num_layers, batch, num_q_heads, 128, dtype=torch.float32, device=dev)
        # the executor's own split-K workspace: its layers run stream-ordered,
        # so they share it; no other executor, stream or graph touches it
        self.ws = ops.new_decode_workspace(dev, batch, num_q_heads, num_kv_heads)
        # consecutive reuse layers run as ONE multi-layer launch (they only
        # share the anchor's lists); run_end[l] = end of l's reuse run
        self.run_end: Dict[int, int] = {}
        l = 0
        while l < num_layers:
            if self.kinds[l] != KIND_REUSE:
                l += 1
                continue
            e = l
            while e < num_layers and self.kinds[e] == KIND_REUSE:
                e += 1
            for i in range(l, e):
                self.run_end[i] = e
            l = e
        # (a sharded executor's local decoder holds GLOBAL maps and runs its own loop)
        zeros = torch.zeros(num_kv_heads, dtype=torch.int32, device=dev)
        self.map_table = torch.stack([self.head_maps[l] if self.kinds[l] == KIND_REUSE and
                                      self.head_maps[l].numel() == num_kv_heads else zeros
                                      for l in range(num_layers)]).contiguous()
        self.ws_layers = ops.new_decode_layers_workspace(dev, batch, num_q_heads, num_kv_heads, num_layers)
        # Overlapped selection (step() on uniform batches, post-softmax
        # pooling): every anchor group (consecutive anchors other than layer
        # 0) runs its score pass and its selection on a side stream, ahead of
        # the main stream's layer loop -- they depend only on the step's q and
        # caches -- so the latency-bound pooled Top-k of one anchor overlaps
        # the HBM-bound attention of other layers; the main stream waits for a
        # group's lists right before the sparse launch that reads them.  Each
        # group owns its scores / pooled / lists and the side stream its own
        # split-K workspaces; the LAST group's lists are self.indices (what a
        # step leaves behind, as in the per-layer path), layer 0's its own.
        self.groups: List[tuple] = []
        if not self.pre:
            l = 1
            while l < num_layers:
                if self.kinds[l] == KIND_ANCHOR:
                    self.groups.append((l, self.group_end[l]))
                    l = self.group_end[l]
                else:
                    l += 1
        self.group_bufs: Dict[int, dict] = {}
        for gi, (gl, ge) in enumerate(self.groups):
            m, last = ge - gl, gi == len(self.groups) - 1
            self.group_bufs[gl] = {
                "end": ge,
                "scores": torch.empty(m * batch, num_q_heads, n_pad, dtype=torch.float32, device=dev),
                "lse": torch.empty(m * batch, num_q_heads, dtype=torch.float32, device=dev),
                "pooled": torch.empty(m * batch * Hsrc, n_pad, dtype=torch.float32, device=dev),
                "idx": self.idx_g[:m] if last else torch.empty(m, batch, Hsrc, k_cap, dtype=torch.int32, device=dev),
                "cnt": self.cnt_g[:m] if last else torch.zeros(m, batch, Hsrc, dtype=torch.int32, device=dev),
                "event": torch.cuda.Event(),
            }
        if self.groups:
            self.idx0 = torch.empty(batch, Hsrc, k_cap, dtype=torch.int32, device=dev)
            self.cnt0 = torch.zeros(batch, Hsrc, dtype=torch.int32, device=dev)
            self.ws_side = ops.new_decode_workspace(dev, batch, num_q_heads, num_kv_heads)
            self.ws_layers_side = ops.new_decode_layers_workspace(dev, batch, num_q_heads, num_kv_heads, gmax)
        else:
            self.idx0, self.cnt0 = self.indices, self.counts
        self.side: Optional[torch.cuda.Stream] = None
        self._tables = {}
        self._graphs = {}
        self.seq_lens: Optional[torch.Tensor] = None     # ragged batch (step / dense_step)

    # -------------------------------------------------------------- eager
    def step(self, q: torch.Tensor, k_caches: Sequence[torch.Tensor], v_caches: Sequence[torch.Tensor],
             seq_len: int, seq_lens: Optional[torch.Tensor] = None) -> torch.Tensor:
        """q [L][B][Hq][128] bf16; k/v_caches: L tensors [B][Hkv][n_cap][128].
        ``seq_lens`` (device int32 [B], each <= seq_len) runs a ragged batch:
        sequence b attends its own first seq_lens[b] keys and selects with
        k_budget(seq_lens[b]); CUDA graphs read it at replay time, so a
        serving loop updates it in place.  Returns the preallocated fp32
        outputs [L][B][Hq][128]."""
        if seq_len > self.n_max:
            raise InvalidArgumentError(f"seq_len {seq_len} exceeds max_seq_len {self.n_max}")
        self.seq_lens = seq_lens
        overlap = self._can_overlap([(0, self.L)], k_caches, v_caches)
        if overlap:
            main = torch.cuda.current_stream()
            self._side_stream().wait_stream(main)      # the step's q and cache rows are in place
            self._issue_selects(q, k_caches, v_caches, seq_len)
        self._run_range(0, self.L, q, k_caches, v_caches, seq_len, overlap=overlap)
        if overlap:
            main.wait_stream(self.side)
        return self.out

    def _layer_tables(self, k_caches, v_caches, l0: int, l1: int):
        """Device pointer tables of layers [l0, l1)'s caches (cached: built
        on the eager warm-up before any graph capture)."""
        key = (l0, l1) + tuple(t.data_ptr() for t in k_caches[l0:l1]) + tuple(t.data_ptr() for t in v_caches[l0:l1])
        tab = self._tables.get(key)
        if tab is None:
            if self.device.type == "cuda" and torch.cuda.is_current_stream_capturing():
                raise InvalidArgumentError("new cache buffers inside a CUDA graph capture: run the step eagerly first")
            kp = torch.tensor([t.data_ptr() for t in k_caches[l0:l1]], dtype=torch.int64, device=self.device)
            vp = torch.tensor([t.data_ptr() for t in v_caches[l0:l1]], dtype=torch.int64, device=self.device)
            tab = self._tables[key] = (kp, vp)
        return tab

    def _run_range(self, l0: int, l1: int, q, k_caches, v_caches, seq_len: int, dense: bool = False,
                   overlap: bool = False) -> None:
        """Layers [l0, l1): every run of consecutive reuse layers (every
        layer in dense mode) is one multi-layer launch; an anchor (or a group
        of consecutive anchors) runs its score passes and its selection, then
        its own sparse passes AND the reuse run that follows it -- they all
        read the anchor's fresh lists -- as one more launch."""
        if overlap and not dense:
            self._run_range_overlapped(l0, l1, q, k_caches, v_caches, seq_len)
            return
        l = l0
        while l < l1:
            if not dense and self.kinds[l] == KIND_ANCHOR and not self.pre and self.seq_lens is None:
                e = min(self.group_end[l], l1)
                end = min(self.run_end[e], l1) if e < l1 and self.kinds[e] == KIND_REUSE else e
                if end - l >= 2 and self._fusable(k_caches, v_caches, l, end):
                    self._anchor_group(l, e, end, q, k_caches, v_caches, seq_len)
                    l = end
                    continue
            end = l1 if dense else (min(self.run_end[l], l1) if self.kinds[l] == KIND_REUSE else l + 1)
            # one launch needs one cache layout; dense layers of a ragged batch
            # run per layer (the multi-layer launch has no per-sequence lengths)
            fuse = end - l >= 2 and not (dense and self.seq_lens is not None) and \
                self._fusable(k_caches, v_caches, l, end)
            if fuse:
                ops.decode_layers(q[l:end], k_caches[l:end], v_caches[l:end], seq_len, out=self.out[l:end],
                                  workspace=self.ws_layers, tables=self._layer_tables(k_caches, v_caches, l, end),
                                  indices=None if dense else self.indices, counts=None if dense else self.counts,
                                  head_maps=None if dense else self.map_table[l:end])
            else:
                for i in range(l, end):
                    (self._dense_layer if dense else self._layer)(i, q, k_caches, v_caches, seq_len)
            l = end

    def _can_overlap(self, ranges, k_caches, v_caches) -> bool:
        """Whether a step split into the layer ``ranges`` runs the overlapped
        schedule (decided per step: its lists live in other buffers than the
        single-stream schedule's): post-softmax pooling, a uniform batch, at
        least one anchor group, one cache layout for every layer (multi-layer
        launches) and no group cut by a range boundary."""
        if not self.groups or self.pre or self.seq_lens is not None or \
                not self._fusable(k_caches, v_caches, 0, self.L):
            return False
        return not any(l0 < gl < l1 < ge or gl < l0 < ge for gl, ge in self.groups for l0, l1 in ranges)

    def _lists_before(self, l: int):
        """(indices, counts) of the latest anchor before layer l in the
        overlapped schedule: slot 0 of its group (its last anchor) or layer 0's."""
        src = None
        for gl, ge in self.groups:
            if gl < l:
                src = gl
        if src is None:
            return self.idx0, self.cnt0
        b = self.group_bufs[src]
        return b["idx"][0], b["cnt"][0]

    def _group_select(self, gl: int, q, k_caches, v_caches, seq_len: int) -> None:
        """Score pass(es) and the selection of the anchor group starting at
        gl into its own buffers (side stream, side workspaces); layer gl + i
        lands in list slot m - 1 - i."""
        b = self.group_bufs[gl]
        ge = b["end"]
        m, B, Hq = ge - gl, self.B, self.Hq
        Hs = self.indices.shape[1]
        if m == 1:
            ops.anchor_scores_decode(q[gl], k_caches[gl], seq_len, b["scores"], b["lse"], workspace=self.ws_side)
        else:
            sc_ls = b["scores"].stride(0) * B
            ops.decode_layers(q[gl:ge], k_caches[gl:ge], v_caches[gl:ge], seq_len, workspace=self.ws_layers_side,
                              tables=self._layer_tables(k_caches, v_caches, gl, ge),
                              scores=b["scores"][(m - 1) * B:m * B], scores_layer_stride=-sc_ls,
                              lse=b["lse"][(m - 1) * B:m * B], lse_layer_stride=-B * Hq)
        ops.select_decode(b["scores"], b["lse"], seq_len, self.plan.k_policy, self.Hkv,
                          indices=b["idx"].view(m * B, Hs, -1), counts=b["cnt"].view(m * B, Hs),
                          pooled=b["pooled"], all_heads=self.all_heads)

    def _run_range_overlapped(self, l0: int, l1: int, q, k_caches, v_caches, seq_len: int) -> None:
        """The main stream's share of layers [l0, l1) in the overlapped
        schedule (the anchor groups' score passes + selections were issued on
        the side stream by _issue_selects): layer 0's dense pass and
        selection, then per anchor group one sparse launch over its own sets
        and the reuse run behind it (after waiting for that group's lists),
        other reuse runs on the lists of the latest anchor before them.  Same
        kernels and launch shapes per layer as the single-stream step, so the
        outputs and lists are bit-identical to it."""
        main = torch.cuda.current_stream()
        pol = self.plan.k_policy
        l = l0
        while l < l1:
            kind = self.kinds[l]
            if kind == KIND_ANCHOR0:
                ops.dense_decode(q[0], k_caches[0], v_caches[0], seq_len, out=self.out[0], lse=self.lse,
                                 scores=self.scores, workspace=self.ws)
                ops.select_decode(self.scores, self.lse, seq_len, pol, self.Hkv, indices=self.idx0,
                                  counts=self.cnt0, pooled=self.pooled, all_heads=self.all_heads)
                l += 1
                continue
            if kind == KIND_ANCHOR:
                b = self.group_bufs[l]
                ge = b["end"]
                end = min(self.run_end[ge], l1) if ge < l1 and self.kinds[ge] == KIND_REUSE else ge
                main.wait_event(b["event"])
                if end - l >= 2:
                    ops.decode_layers(q[l:end], k_caches[l:end], v_caches[l:end], seq_len, out=self.out[l:end],
                                      workspace=self.ws_layers, tables=self._layer_tables(k_caches, v_caches, l, end),
                                      indices=b["idx"][0], counts=b["cnt"][0], head_maps=self._fused_maps(l, ge, end))
                else:                      # a lone last anchor: its own sets, one layer
                    ops.sparse_decode(q[l], k_caches[l], v_caches[l], seq_len, b["idx"][0], b["cnt"][0],
                                      self.shared_map, out=self.out[l], workspace=self.ws)
                l = end
                continue
            end = min(self.run_end[l], l1)
            idx, cnt = self._lists_before(l)
            if end - l >= 2:
                ops.decode_layers(q[l:end], k_caches[l:end], v_caches[l:end], seq_len, out=self.out[l:end],
                                  workspace=self.ws_layers, tables=self._layer_tables(k_caches, v_caches, l, end),
                                  indices=idx, counts=cnt, head_maps=self.map_table[l:end])
            else:
                ops.sparse_decode(q[l], k_caches[l], v_caches[l], seq_len, idx, cnt, self.head_maps[l],
                                  out=self.out[l], workspace=self.ws)
            l = end

    def _side_stream(self) -> torch.cuda.Stream:
        if self.side is None:
            self.side = torch.cuda.Stream(device=self.device)
        return self.side

    def _issue_selects(self, q, k_caches, v_caches, seq_len: int) -> None:
        """Every anchor group's score pass + selection, in layer order, on the
        side stream (the caller orders the side stream after the step's
        inputs and joins it back at the end of the step)."""
        with torch.cuda.stream(self._side_stream()):
            for gl, _ in self.groups:
                self._group_select(gl, q, k_caches, v_caches, seq_len)
                self.group_bufs[gl]["event"].record(self.side)

    @staticmethod
    def _fusable(k_caches, v_caches, l: int, end: int) -> bool:
        ref = k_caches[l]
        return all(t.shape == ref.shape and t.stride() == ref.stride() for t in list(k_caches[l:end]) +
                   list(v_caches[l:end]))

    def launches_per_step(self, dense: bool = False) -> int:
        """Kernel launches of one step() (post-softmax pooling, uniform batch):
        anchor 0 = dense + pool + Top-k; an anchor or a group of consecutive
        anchors = scores + pool + Top-k + one sparse launch that also runs the
        reuse run behind it; any other reuse run = one launch."""
        if dense:
            return 1
        n, l = 0, 0
        while l < self.L:
            kind = self.kinds[l]
            if kind == KIND_ANCHOR0:
                n, l = n + 3, l + 1
            elif kind == KIND_ANCHOR:
                e = self.group_end[l]
                n, l = n + 4, (self.run_end[e] if e < self.L and self.kinds[e] == KIND_REUSE else e)
            else:
                n, l = n + 1, self.run_end[l]
        return n

    def _fused_maps(self, l0: int, l1: int, end: int) -> torch.Tensor:
        """Head-map table of the sparse launch over [l0, end) that follows the
        selection of anchors [l0, l1): anchor l0 + i reads its own lists in
        slot m - 1 - i of idx_g / cnt_g -- a map entry may address any row of
        the [slots][B][Hsrc] list space, so slot s of source head h is row
        s * B * Hsrc + h -- and the reuse layers read slot 0 (the last
        anchor's lists) through their own maps.  Built on the eager warm-up,
        looked up inside graph captures."""
        key = ("maps", l0, l1, end)
        t = self._tables.get(key)
        if t is None:
            if self.device.type == "cuda" and torch.cuda.is_current_stream_capturing():
                raise InvalidArgumentError("new launch layout inside a CUDA graph capture: run the step eagerly first")
            m, Hs = l1 - l0, self.indices.shape[1]
            own = torch.zeros(self.Hkv, dtype=torch.int32, device=self.device) if self.all_heads else \
                torch.arange(self.Hkv, dtype=torch.int32, device=self.device)
            rows = [own + (m - 1 - i) * self.B * Hs for i in range(m)]
            rows += [self.map_table[l] for l in range(l1, end)]
            t = self._tables[key] = torch.stack(rows).contiguous()
        return t

    def _anchor_group(self, l0: int, l1: int, end: int, q, k_caches, v_caches, seq_len: int) -> None:
        """Consecutive anchor layers [l0, l1) as three launches: their score
        passes, one select over all their (sequence, kv head) rows, and their
        sparse passes over their own fresh sets (runner.py:263-266) together
        with the reuse layers [l1, end) over the last anchor's sets routed by
        their head maps (runner.py:267-275).  Layer l0 + i uses slot m - 1 - i,
        so the last anchor's lists land in slot 0 (self.indices)."""
        m = l1 - l0
        B, Hq = self.B, self.Hq
        Hs = self.indices.shape[1]
        if m == 1:
            ops.anchor_scores_decode(q[l0], k_caches[l0], seq_len, self.scores, self.lse, workspace=self.ws)
            ops.select_decode(self.scores, self.lse, seq_len, self.plan.k_policy, self.Hkv, indices=self.indices,
                              counts=self.counts, pooled=self.pooled, all_heads=self.all_heads)
        else:
            tabs = self._layer_tables(k_caches, v_caches, l0, l1)
            sc_ls = self.scores_g.stride(0) * B
            ops.decode_layers(q[l0:l1], k_caches[l0:l1], v_caches[l0:l1], seq_len, workspace=self.ws_layers,
                              tables=tabs, scores=self.scores_g[(m - 1) * B:m * B], scores_layer_stride=-sc_ls,
                              lse=self.lse_g[(m - 1) * B:m * B], lse_layer_stride=-B * Hq)
            ops.select_decode(self.scores_g[:m * B], self.lse_g[:m * B], seq_len, self.plan.k_policy, self.Hkv,
                              indices=self.idx_g[:m].view(m * B, Hs, -1), counts=self.cnt_g[:m].view(m * B, Hs),
                              pooled=self.pooled_g[:m * B * Hs], all_heads=self.all_heads)
        ops.decode_layers(q[l0:end], k_caches[l0:end], v_caches[l0:end], seq_len, out=self.out[l0:end],
                          workspace=self.ws_layers, tables=self._layer_tables(k_caches, v_caches, l0, end),
                          indices=self.indices, counts=self.counts, head_maps=self._fused_maps(l0, l1, end))

    def _layer(self, l: int, q, k_caches, v_caches, seq_len: int) -> None:
        """The kernels of layer l (runner.py:250-275 for one decode token)."""
        kind = self.kinds[l]
        ql, kl, vl = q[l], k_caches[l], v_caches[l]
        if kind == KIND_REUSE:
            ops.sparse_decode(ql, kl, vl, seq_len, self.indices, self.counts, self.head_maps[l], out=self.out[l],
                              workspace=self.ws)
            return
        self._anchor_select(l, kind, ql, kl, vl, seq_len, self.out[l])
        if kind == KIND_ANCHOR:
            ops.sparse_decode(ql, kl, vl, seq_len, self.indices, self.counts, self.shared_map, out=self.out[l],
                              workspace=self.ws)

    def _anchor_select(self, l: int, kind: str, ql, kl, vl, seq_len: int, out) -> None:
        """Layer 0's dense output (into ``out``) and the anchor selection of
        layer l into self.indices / self.counts (runner.py:250-266): post-
        softmax pooling from the dense or score pass, or pre-softmax pooling
        from q_bar with no attention pass."""
        pol, sl = self.plan.k_policy, self.seq_lens
        if self.pre:
            if kind == KIND_ANCHOR0:
                ops.dense_decode(ql, kl, vl, seq_len, out=out, lse=self.lse, seq_lens=sl, workspace=self.ws)
            ops.select_decode_pre(ql, kl, seq_len, pol, pooled=self.pooled, workspace=self.pre_ws,
                                  indices=self.indices, counts=self.counts, all_heads=self.all_heads, seq_lens=sl)
            return
        if kind == KIND_ANCHOR0:
            ops.dense_decode(ql, kl, vl, seq_len, out=out, lse=self.lse, scores=self.scores, seq_lens=sl,
                             workspace=self.ws)
        else:
            ops.anchor_scores_decode(ql, kl, seq_len, self.scores, self.lse, seq_lens=sl, workspace=self.ws)
        ops.select_decode(self.scores, self.lse, seq_len, pol, self.Hkv, indices=self.indices,
                          counts=self.counts, pooled=self.pooled, all_heads=self.all_heads, seq_lens=sl)

    def _dense_layer(self, l: int, q, k_caches, v_caches, seq_len: int) -> None:
        ops.dense_decode(q[l], k_caches[l], v_caches[l], seq_len, out=self.out[l], lse=self.lse,
                         seq_lens=self.seq_lens, workspace=self.ws)

    def dense_step(self, q, k_caches, v_caches, seq_len: int, seq_lens: Optional[torch.Tensor] = None
                   ) -> torch.Tensor:
        """Top-k = 100% baseline: dense attention on every layer (one launch
        for all layers, like the Kascade step's reuse runs; per layer with a
        ragged batch)."""
        self.seq_lens = seq_lens
        self._run_range(0, self.L, q, k_caches, v_caches, seq_len, dense=True)
        return self.out

    # -------------------------------------------------------------- graphs
    def capture(self, q, k_caches, v_caches, seq_len: int, dense: bool = False,
                seq_lens: Optional[torch.Tensor] = None) -> torch.cuda.CUDAGraph:  # noqa: D102
        """Capture one step (fixed buffers and seq_len) in a CUDA graph; replay
        with ``graph.replay()`` after writing new queries into ``q`` (and new
        lengths into ``seq_lens`` for a ragged batch)."""
        fn = self.dense_step if dense else self.step
        fn(q, k_caches, v_caches, seq_len, seq_lens)  # warm-up: one-time kernel attributes outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn(q, k_caches, v_caches, seq_len, seq_lens)
        self._graphs[(seq_len, dense)] = g
        return g

    def capture_host_step(self, q_host, kv_host, out_host, q, k_caches, v_caches, seq_len: int,
                          dense: bool = False, seq_lens: Optional[torch.Tensor] = None) -> torch.cuda.CUDAGraph:
        """A whole serving decode step from and to pinned host memory as ONE
        CUDA graph: H2D of the step's queries (``q_host`` [L][B][Hq][128]) and
        new K/V rows (``kv_host`` [L][2][B][Hkv][128]), one append launch that
        writes the rows at cache position ``seq_len - 1`` of every layer, the
        layer loop, and D2H of the outputs into ``out_host`` [L][B][Hq][128]
        fp32.  Replay, then synchronise the stream before reading out_host."""
        # ragged batch: sequence b appends at seq_lens[b] - 1 and attends its
        # own prefix; the graph reads seq_lens (device) at every replay
        self.seq_lens = seq_lens
        for t, name in ((q_host, "q_host"), (kv_host, "kv_host"), (out_host, "out_host")):
            if t.is_cuda or not t.is_pinned():
                raise InvalidArgumentError(f"{name} must be pinned host memory")
        kp, vp, sb, sh, n_cap = ops.cache_pointer_tables(k_caches, v_caches, self.device)
        # every append lands inside the caches: validated before anything is enqueued
        # (a ragged row outside [0, n_cap) is skipped by the kernel as well)
        if not 1 <= seq_len <= min(self.n_max, n_cap):
            raise InvalidArgumentError(f"seq_len {seq_len} outside [1, min(max_seq_len {self.n_max}, "
                                       f"cache capacity {n_cap})]")
        kv_dev = torch.empty(kv_host.shape, dtype=torch.bfloat16, device=self.device)
        tables0, tables_rest = (kp[:1], vp[:1], sb, sh, n_cap), (kp[1:], vp[1:], sb, sh, n_cap)
        # The copies are pipelined against the layer loop on two side streams
        # (graph branches): layer 0's new K/V rows and queries arrive first
        # and layer 0 starts behind their append; the other layers' rows and
        # queries stream in behind layer 0 and get one append launch.  The
        # outputs leave in chunks that shrink toward the end (boundaries
        # D2H_SPLITS), so the copy exposed after the last layer is small.
        # Few cross-stream edges keep consecutive reuse-layer kernels chained
        # by programmatic dependent launch (decode.cu).
        h2d, d2h = torch.cuda.Stream(device=self.device), torch.cuda.Stream(device=self.device)
        ev_first, ev_rest, ev_app = torch.cuda.Event(), torch.cuda.Event(), torch.cuda.Event()
        ends = sorted({e for e in self.D2H_SPLITS if 0 < e < self.L} | {self.L})
        ev_done = [torch.cuda.Event() for _ in ends]

        def body():
            main = torch.cuda.current_stream()
            h2d.wait_stream(main)
            d2h.wait_stream(main)
            with torch.cuda.stream(h2d):
                kv_dev[:1].copy_(kv_host[:1], non_blocking=True)
                q[0].copy_(q_host[0], non_blocking=True)
                ev_first.record(h2d)
                if self.L > 1:
                    kv_dev[1:].copy_(kv_host[1:], non_blocking=True)
                    q[1:].copy_(q_host[1:], non_blocking=True)
                ev_rest.record(h2d)
            main.wait_event(ev_first)
            ops.append_kv(kv_dev[:1], seq_len - 1, tables0, seq_lens)
            # segments: layer 0 alone (its rows and queries arrive first), then
            # the layers between the output-copy boundaries
            bounds = sorted({0, 1, self.L} | set(ends))
            overlap = not dense and self._can_overlap(list(zip(bounds[:-1], bounds[1:])), k_caches, v_caches)
            if overlap:
                # the other layers' rows are appended on the side stream as
                # soon as they arrive, then the anchor groups' score passes and
                # selections follow there, concurrent with layer 0 on main
                side = self._side_stream()
                side.wait_stream(main)
                side.wait_event(ev_rest)
                with torch.cuda.stream(side):
                    ops.append_kv(kv_dev[1:], seq_len - 1, tables_rest, seq_lens)
                    ev_app.record(side)
                self._issue_selects(q, k_caches, v_caches, seq_len)
            start = 0
            for a_, b_ in zip(bounds[:-1], bounds[1:]):
                if a_ == 1:
                    if overlap:
                        main.wait_event(ev_app)
                    else:
                        main.wait_event(ev_rest)
                        ops.append_kv(kv_dev[1:], seq_len - 1, tables_rest, seq_lens)
                self._run_range(a_, b_, q, k_caches, v_caches, seq_len, dense=dense, overlap=overlap)
                if b_ in ends:
                    c = ends.index(b_)
                    ev_done[c].record(main)
                    with torch.cuda.stream(d2h):
                        d2h.wait_event(ev_done[c])
                        out_host[start:b_].copy_(self.out[start:b_], non_blocking=True)
                    start = b_
            main.wait_stream(h2d)
            main.wait_stream(d2h)
            if overlap:
                main.wait_stream(self.side)

        body()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        self._graphs[("host", seq_len, dense)] = (g, kv_dev, kp, vp, h2d, d2h)   # keep the staging alive
        return g


class KascadePrefill:
    """Prefill executor over every layer of a plan (batch 1, tiles of 128
    query rows -- the reference's prefill phase, tiles.py:137-144):

      layer 0   dense attention (O, LSE) -> pass B pooled Top-k per tile
      anchor l  pass A (LSE) -> pass B pooled Top-k -> sparse over own sets
      reuse l   sparse over the latest anchor's sets routed by head_map[l]

    ``dense_forward`` is the Top-k = 100% baseline over the same layers."""

    def __init__(self, plan, num_layers: int, num_q_heads: int, num_kv_heads: int, seq_len: int, device=None,
                 validate: bool = True):
        if validate:   # sharded executors validate against the GLOBAL head count themselves
            validate_plan(plan, num_layers, num_kv_heads)
        if plan.tile_size != ops.TILE:
            raise InvalidArgumentError(f"prefill engine tiles are {ops.TILE} rows (plan has {plan.tile_size})")
        self.plan = plan
        self.L, self.Hq, self.Hkv, self.N = num_layers, num_q_heads, num_kv_heads, seq_len
        self.device = torch.device(device or "cuda")
        self.kinds = layer_kinds(plan, num_layers)
        self.all_heads = plan.mode == MODE_ALL_HEADS_POOLED
        dev = self.device
        T = (seq_len + ops.TILE - 1) // ops.TILE
        rows = 1 if self.all_heads else num_kv_heads
        kc = k_budget(plan.k_policy, seq_len)
        self.head_maps: Dict[int, Optional[torch.Tensor]] = {}
        for l, kind in enumerate(self.kinds):
            if kind == KIND_REUSE:
                m = [0] * num_kv_heads if self.all_heads else plan.head_maps[l].map
                self.head_maps[l] = torch.tensor(m, dtype=torch.int32, device=dev)
        self.shared_map = torch.zeros(num_kv_heads, dtype=torch.int32, device=dev) if self.all_heads else None
        self.lse = torch.empty(num_q_heads, seq_len, dtype=torch.float32, device=dev)
        self.pre = plan.pooling == POOL_PRE     # pre-softmax pooling (runner.py:155-161): no pass A / pass B
        if self.pre:
            self.pooled, self.pre_ws, _, _ = ops.select_pre_buffers(1, num_kv_heads, seq_len, plan.k_policy, dev,
                                                                    prefill=True, all_heads=self.all_heads,
                                                                    num_q_heads=num_q_heads)
        else:
            self.pooled = ops.select_prefill_scratch(num_q_heads, num_kv_heads, seq_len, dev, self.all_heads)
        self.indices = torch.empty(rows, T, kc, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(rows, T, dtype=torch.int32, device=dev)
        self.out = torch.empty(num_layers, num_q_heads, seq_len, 128, dtype=torch.bfloat16, device=dev)

    def forward(self, qs: Sequence[torch.Tensor], ks: Sequence[torch.Tensor], vs: Sequence[torch.Tensor],
                stop_after: Optional[int] = None) -> torch.Tensor:
        """qs/ks/vs: per-layer [Hq][N][128] / [Hkv][N][128] bf16.  Returns the
        bf16 outputs [L][Hq][N][128].  ``stop_after`` ends the loop after that
        layer (the index lists then hold that layer's latest anchor sets)."""
        for l, kind in enumerate(self.kinds):
            if stop_after is not None and l > stop_after:
                break
            q, k, v = qs[l], ks[l], vs[l]
            if kind == KIND_REUSE:
                ops.sparse_prefill(q, k, v, self.indices, self.counts, self.head_maps[l], out=self.out[l])
                continue
            self._anchor_select(kind, q, k, v, self.out[l])
            if kind == KIND_ANCHOR:
                ops.sparse_prefill(q, k, v, self.indices, self.counts, self.shared_map, out=self.out[l])
        return self.out

    def _anchor_select(self, kind: str, q, k, v, out) -> None:
        """Layer 0's dense output and the anchor's per-(kv head, tile) sets
        (runner.py:250-266): pass A (LSE) + pass B pooled Top-k, or the
        pre-softmax q_bar selection (no attention pass)."""
        pol = self.plan.k_policy
        if kind == KIND_ANCHOR0:
            ops.dense_prefill(q, k, v, out=out, lse=self.lse)
        if self.pre:
            ops.select_prefill_pre(q, k, pol, pooled=self.pooled, workspace=self.pre_ws, indices=self.indices,
                                   counts=self.counts, all_heads=self.all_heads)
            return
        if kind != KIND_ANCHOR0:
            ops.anchor_lse_prefill(q, k, lse=self.lse)
        ops.select_prefill(q, k, self.lse, pol, indices=self.indices, counts=self.counts, pooled=self.pooled,
                           all_heads=self.all_heads)

    def dense_forward(self, qs, ks, vs) -> torch.Tensor:
        for l in range(self.L):
            ops.dense_prefill(qs[l], ks[l], vs[l], out=self.out[l], lse=self.lse)
        return self.out
