"""Test helper: PROTOCOL.md frame codec in Python (the product's codec is
C++ in libsfg; this one builds requests and reads responses in tests).
Byte layout: [u32 LE header len][sorted-key compact JSON][tensor][mask]."""
from __future__ import annotations

import json
import struct

import numpy as np


def encode(kind: str, session_id: str = "", shape=(0,), dtype: str = "f16", pos=None, crop=None, keep=None,
           mask_shape=None, err=None, srv_ms=None, tensor: bytes = b"", mask: bytes = b"") -> bytes:
    j = {"kind": kind, "session_id": session_id, "shape": list(shape), "dtype": dtype}
    if pos:
        j["pos"] = [int(p) for p in pos]
    if crop is not None:
        j["crop"] = int(crop)
    if keep is not None:
        j["keep"] = [int(k) for k in keep]
    if mask_shape is not None:
        j["mask_shape"] = list(mask_shape)
    if err is not None:
        j["err"] = err
    if srv_ms is not None:
        j["srv_ms"] = srv_ms
    hdr = json.dumps(j, sort_keys=True, separators=(",", ":"), ensure_ascii=False).encode()
    return struct.pack("<I", len(hdr)) + hdr + tensor + mask


def decode(b: bytes):
    (n,) = struct.unpack("<I", b[:4])
    h = json.loads(b[4:4 + n])
    body = b[4 + n:]
    return h, body


def hidden_request(kind, sid, rows: np.ndarray, positions, dtype="f32", keep=None, crop=None, mask=None):
    rows = np.asarray(rows, dtype=np.float32)
    if dtype == "f32":
        t = rows.tobytes()
    else:
        t = rows.astype(np.float16).tobytes()  # only used with values exactly representable
    ms, mb = None, b""
    if mask is not None:
        m = np.asarray(mask, dtype=np.float32)
        ms = [1, 1, m.shape[0], m.shape[1]]
        mb = m.astype(np.float16).tobytes()
    return encode(kind, sid, rows.shape, dtype, pos=list(positions), keep=keep, crop=crop, mask_shape=ms,
                  tensor=t, mask=mb)


def response_rows(b: bytes, hidden: int):
    h, body = decode(b)
    if h["kind"] != "response":
        return h, None
    dt = np.float32 if h["dtype"] == "f32" else np.float16
    return h, np.frombuffer(body, dtype=dt).astype(np.float32).reshape(h["shape"])


def rows_of(h: dict, body: bytes) -> np.ndarray:
    """The hidden-row tensor of a decoded request/response frame as fp32
    (the mask, when present, follows the tensor and is ignored)."""
    rows, dim = h["shape"]
    dt = np.float32 if h["dtype"] == "f32" else np.float16
    n = rows * dim
    return np.frombuffer(body[:n * np.dtype(dt).itemsize], dtype=dt).astype(np.float32).reshape(rows, dim)


def strip_srv_ms(b: bytes) -> bytes:
    h, body = decode(b)
    h.pop("srv_ms", None)
    hdr = json.dumps(h, sort_keys=True, separators=(",", ":"), ensure_ascii=False).encode()
    return struct.pack("<I", len(hdr)) + hdr + body
