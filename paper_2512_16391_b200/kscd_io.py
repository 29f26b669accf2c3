"""KSCD v1 traces and run reports (the reference's wire formats,
traceio.py:3-17,75-156,419-510), with a device loader for the engine.

``read_trace`` returns an ``AttentionTrace`` (numpy, validated with the
reference's FormatError offsets).  ``TraceFile`` memory-maps the payload and
streams one layer at a time to the GPU: an mmap slice is copied into a
pinned staging buffer, uploaded asynchronously and rounded to bf16 on the
device, so a multi-GB trace never has to fit in host RAM.
"""

from __future__ import annotations

import io
import json
import struct
from typing import Optional, Tuple

import numpy as np

from .exceptions import FormatError, InvalidArgumentError
from .host_types import AttentionTrace, LayerReport, RunReport

MAGIC = b"KSCD"
VERSION = 1
_HEAD = struct.Struct("<4sH5I2BH")      # magic, version, L Hq Hkv d N, dtype, flags, prompt length
FLAG_XY = 0x01


def _parse_header(blob: bytes):
    if len(blob) < _HEAD.size:
        raise FormatError(f"file truncated inside the {_HEAD.size}-byte header", offset=len(blob))
    magic, version, L, Hq, Hkv, d, N, dtype, flags, plen = _HEAD.unpack_from(blob, 0)
    if magic != MAGIC:
        raise FormatError(f"bad magic {magic!r}, expected {MAGIC!r}", offset=0)
    if version != VERSION:
        raise FormatError(f"unsupported version {version}", offset=4)
    if dtype != 0:
        raise FormatError(f"unsupported dtype code {dtype}", offset=26)
    if min(L, Hq, Hkv, d, N) < 1:
        raise FormatError("header dimensions must all be >= 1", offset=6)
    if Hq % Hkv:
        raise FormatError(f"query heads ({Hq}) not divisible by kv heads ({Hkv})", offset=10)
    return L, Hq, Hkv, d, N, flags, plen


class TraceFile:
    """Memory-mapped KSCD v1 trace: header, tensor offsets, per-layer access."""

    def __init__(self, path: str):
        with open(path, "rb") as f:
            head = f.read(_HEAD.size + 65536)
        self.L, self.Hq, self.Hkv, self.d, self.N, flags, plen = _parse_header(head)
        start = _HEAD.size
        if len(head) < start + plen:
            raise FormatError("file truncated inside prompt_id", offset=len(head))
        try:
            self.prompt_id = head[start:start + plen].decode("utf-8")
        except UnicodeDecodeError as e:
            raise FormatError(f"prompt_id is not valid UTF-8: {e}", offset=start) from None
        self.has_xy = bool(flags & FLAG_XY)
        self.path = path
        self._mm = np.memmap(path, dtype=np.uint8, mode="r")
        L, Hq, Hkv, d, N = self.L, self.Hq, self.Hkv, self.d, self.N
        off = start + plen
        self.off_q = off
        self.off_k = self.off_q + L * Hq * N * d * 4
        self.off_v = self.off_k + L * Hkv * N * d * 4
        self.off_end = self.off_v + L * Hkv * N * d * 4
        size = int(self._mm.size)
        for name, lo, hi in (("Q", self.off_q, self.off_k), ("K", self.off_k, self.off_v),
                             ("V", self.off_v, self.off_end)):
            if size < hi:
                raise FormatError(f"file truncated inside tensor {name}: need {hi - lo} bytes at offset {lo}, "
                                  f"have {max(size - lo, 0)}", offset=size)
        rest = self._mm.size - self.off_end
        if self.has_xy:
            if rest <= 0 or rest % 2 or (rest // 2) % (L * N * 4):
                raise FormatError(f"trailing {rest} bytes do not form two [L][N][model_dim] float32 tensors",
                                  offset=self.off_end)
            self.model_dim = (rest // 2) // (L * N * 4)
        elif rest:
            raise FormatError(f"{rest} unexpected trailing bytes", offset=self.off_end)

    def _view(self, off: int, shape) -> np.ndarray:
        n = int(np.prod(shape))
        return np.frombuffer(self._mm, dtype="<f4", count=n, offset=off).reshape(shape)

    def layer_numpy(self, layer: int) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Zero-copy fp32 views of one layer's Q [Hq][N][d], K, V [Hkv][N][d]."""
        if not 0 <= layer < self.L:
            raise InvalidArgumentError(f"layer {layer} out of range [0, {self.L})")
        L, Hq, Hkv, d, N = self.L, self.Hq, self.Hkv, self.d, self.N
        q = self._view(self.off_q + layer * Hq * N * d * 4, (Hq, N, d))
        k = self._view(self.off_k + layer * Hkv * N * d * 4, (Hkv, N, d))
        v = self._view(self.off_v + layer * Hkv * N * d * 4, (Hkv, N, d))
        return q, k, v

    # duck-typed AttentionTrace header, so the engine's executors and
    # validate_plan accept a TraceFile and stream it layer by layer
    num_layers = property(lambda self: self.L)
    num_query_heads = property(lambda self: self.Hq)
    num_kv_heads = property(lambda self: self.Hkv)
    head_dim = property(lambda self: self.d)
    seq_len = property(lambda self: self.N)

    @property
    def X(self):
        """Zero-copy [L][N][model_dim] fp32 view of the attention inputs (None without X/Y)."""
        return self._view(self.off_end, (self.L, self.N, self.model_dim)) if self.has_xy else None

    @property
    def Y(self):
        """Zero-copy [L][N][model_dim] fp32 view of the attention outputs (None without X/Y)."""
        if not self.has_xy:
            return None
        return self._view(self.off_end + self.L * self.N * self.model_dim * 4, (self.L, self.N, self.model_dim))

    def layer_device(self, layer: int, device="cuda"):
        """One layer as bf16 CUDA tensors (Q [Hq][N][d], K/V [Hkv][N][d]):
        mmap slice -> reused pinned staging buffer -> async H2D on the
        current stream -> on-device bf16 rounding and finiteness check (the
        reference rejects non-finite payloads at read time, trace.py:75)."""
        import torch
        need = (self.Hq + 2 * self.Hkv) * self.N * self.d
        if getattr(self, "_pinned", None) is None or self._pinned.numel() < need:
            self._pinned = torch.empty(need, dtype=torch.float32).pin_memory()
        stage, pos, out = self._pinned.numpy(), 0, []
        torch.cuda.current_stream().synchronize()    # staging buffer may still feed the previous upload
        for name, arr in zip("QKV", self.layer_numpy(layer)):
            n = arr.size
            stage[pos:pos + n] = arr.reshape(-1)
            dev = self._pinned[pos:pos + n].view(arr.shape).to(device, non_blocking=True)
            if not bool(torch.isfinite(dev).all()):
                raise FormatError(f"trace payload violates header invariants: {name} contains non-finite values")
            out.append(dev.to(torch.bfloat16))
            pos += n
        return tuple(out)

    def to_trace(self) -> AttentionTrace:
        L, Hq, Hkv, d, N = self.L, self.Hq, self.Hkv, self.d, self.N
        Q = self._view(self.off_q, (L, Hq, N, d)).copy()
        K = self._view(self.off_k, (L, Hkv, N, d)).copy()
        V = self._view(self.off_v, (L, Hkv, N, d)).copy()
        X = Y = None
        if self.has_xy:
            X = self._view(self.off_end, (L, N, self.model_dim)).copy()
            Y = self._view(self.off_end + L * N * self.model_dim * 4, (L, N, self.model_dim)).copy()
        for name, arr in (("Q", Q), ("K", K), ("V", V)):
            if not np.isfinite(arr).all():
                raise FormatError(f"trace payload violates header invariants: {name} contains non-finite values")
        try:
            return AttentionTrace(L, Hq, Hkv, d, N, Q, K, V, X, Y, prompt_id=self.prompt_id)
        except InvalidArgumentError as e:
            raise FormatError(f"trace payload violates header invariants: {e}") from None


def read_trace(path) -> AttentionTrace:
    return TraceFile(path).to_trace()


def write_trace(path, trace) -> None:
    """Serialise a trace in KSCD v1 (bit-exact round trip with read_trace)."""
    prompt = trace.prompt_id.encode("utf-8")
    if len(prompt) > 0xFFFF:
        raise InvalidArgumentError("prompt_id longer than 65535 bytes")
    xy = trace.X is not None and trace.Y is not None
    with open(path, "wb") as f:
        f.write(_HEAD.pack(MAGIC, VERSION, trace.num_layers, trace.num_query_heads, trace.num_kv_heads,
                           trace.head_dim, trace.seq_len, 0, FLAG_XY if xy else 0, len(prompt)))
        f.write(prompt)
        tensors = [trace.Q, trace.K, trace.V] + ([trace.X, trace.Y] if xy else [])
        for arr in tensors:
            f.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())


# ------------------------------------------------------------------ reports
def report_to_dict(report: RunReport) -> dict:
    """Run-report JSON, schema v1 (traceio.py:419-435)."""
    return {"schema_version": 1, "kind": "kascade-run-report",
            "per_layer": [{"layer": r.layer, "kind": r.kind, "output_rel_err_l2": r.output_rel_err_l2,
                           "mass_recovered_mean": r.mass_recovered_mean, "fallback_rows": r.fallback_rows}
                          for r in report.per_layer],
            "overall": report.overall, "config": report.config}


def write_report(path, report: RunReport) -> None:
    with open(path, "w", encoding="utf-8") as f:
        json.dump(report_to_dict(report), f, indent=2, sort_keys=True)
        f.write("\n")


def report_from_dict(data: dict) -> RunReport:
    """traceio.py:438-453."""
    rows = [LayerReport(e["layer"], e["kind"], e["output_rel_err_l2"], e["mass_recovered_mean"],
                        e.get("fallback_rows", 0)) for e in data.get("per_layer", [])]
    return RunReport(per_layer=rows, overall=data.get("overall", {}), config=data.get("config", {}))


def read_report(path) -> RunReport:
    with open(path, "r", encoding="utf-8") as f:
        try:
            data = json.load(f)
        except json.JSONDecodeError as e:
            raise FormatError(f"report file is not valid JSON: {e}") from None
    return report_from_dict(data)


def plans_equal(a, b) -> bool:
    """traceio.py:410-411: equal serialised forms."""
    from .host_types import plan_to_dict
    return plan_to_dict(a) == plan_to_dict(b)


def format_report(report: RunReport) -> str:
    """Text rendering with the reference's columns (traceio.py:471-485)."""
    buf = io.StringIO()
    buf.write(f"{'layer':>5}  {'kind':<8}  {'rel_err_l2':>12}  {'mass_recovered':>14}\n")
    for r in report.per_layer:
        mass = "-" if np.isnan(r.mass_recovered_mean) else f"{r.mass_recovered_mean:.6f}"
        buf.write(f"{r.layer:>5}  {r.kind:<8}  {r.output_rel_err_l2:>12.3e}  {mass:>14}\n")
    buf.write("overall:\n")
    for key in sorted(report.overall):
        buf.write(f"  {key} = {report.overall[key]:.6g}\n")
    for key, val in sorted(report.config.items()):
        buf.write(f"  # {key}: {val}\n")
    return buf.getvalue()


# ----------------------------------------------------- CSV text forms (analyze)
def similarity_csv(S) -> str:
    """traceio.py:488-494: upper triangle of a SimilarityMatrix."""
    lines = ["row,col,value"]
    for a in range(S.num_layers):
        for b in range(a, S.num_layers):
            lines.append(f"{a},{b},{S.S[a, b]:.8g}")
    return "\n".join(lines) + "\n"


def importance_csv(importance) -> str:
    """traceio.py:497-501."""
    lines = ["layer,weight"] + [f"{layer},{w:.8g}" for layer, w in enumerate(importance.w)]
    return "\n".join(lines) + "\n"


def coverage_csv(coverage_by_layer) -> str:
    """traceio.py:504-510: coverage_by_layer[l][h] = mean Top-k mass of (layer l, head h)."""
    lines = ["layer,head,coverage"]
    for layer, per_head in enumerate(coverage_by_layer):
        for head, cov in enumerate(np.atleast_1d(per_head)):
            lines.append(f"{layer},{head},{cov:.8g}")
    return "\n".join(lines) + "\n"
