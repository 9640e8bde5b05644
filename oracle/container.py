"""VIET container restatement (TEST INFRASTRUCTURE ONLY -- the checker, never the product).

Follows /root/reference/proj/include/vie/container.hpp:15-159 byte for byte: "VIET", u32
version 1, u8 kind (0 dense, 1 tucker, 2 tucker_cp), u8 rule (0 sigma_max, 1 energy), u16 0,
f64 tol, u64 dims[3], u64 ranks[3], then (re, im) f64 pairs -- dense n1 n2 n3 axis-1 fastest
(container.hpp:95-100), tucker U1 U2 U3 column-major then the core (:102-111), tucker_cp W1
W2 W3 (:113-120).  Little-endian, as the reference writes on x86-64 (write_pod of the host
representation, :40-44).  Used by tests/test_container.py to pin the library's writer and
reader."""
import struct

import numpy as np

MAGIC = b"VIET"
VERSION = 1


def encode(kind, rule, tol, dims, ranks, blocks):
    head = MAGIC + struct.pack("<IBBHd3Q3Q", VERSION, kind, rule, 0, tol, *dims, *ranks)
    body = b"".join(np.asarray(b, np.complex128).reshape(-1, order="F").astype("<c16").tobytes() for b in blocks)
    return head + body


def decode(data):
    if len(data) < 4 or data[:4] != MAGIC:
        raise ValueError("container: bad magic")
    if len(data) < 68:
        raise ValueError("container: truncated file")
    version, kind, rule, _, tol, *rest = struct.unpack("<IBBHd3Q3Q", data[4:68])
    if version != VERSION:
        raise ValueError("container: unsupported version")
    dims, ranks = tuple(rest[:3]), tuple(rest[3:])
    payload = np.frombuffer(data[68:], "<c16")
    return kind, rule, tol, dims, ranks, payload
