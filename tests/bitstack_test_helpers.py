"""Small helpers shared by the test modules (no method arithmetic of their own:
stored blocks come from oracle/ or synthetic/, expected values from oracle/)."""
import numpy as np


def read_golden(path):
    rows = []
    with open(path) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(line.split())
    return rows


def stack_blocks(blocks, factor_dtype):
    """Oracle Block list -> (signs [n, nbytes] u8, u, v) arrays in the storage dtype
    the library is told about (bf16 as uint16 bit patterns)."""
    from oracle import bitstack_oracle as O
    signs = np.stack([b.signs for b in blocks]).astype(np.uint8)
    u = np.stack([b.u for b in blocks])
    v = np.stack([b.v for b in blocks])
    if factor_dtype == "bf16":
        return signs, O.bf16_bits(u), O.bf16_bits(v)
    if factor_dtype == "f16":
        return signs, u.astype(np.float16), v.astype(np.float16)
    return signs, u.astype(np.float32), v.astype(np.float32)


def blocks_from_arrays(signs, u, v):
    """Stored arrays (f32 values) -> oracle Block objects (values as the oracle sees them)."""
    from oracle import bitstack_oracle as O
    return [O.Block(signs=signs[i].copy(), u=np.asarray(u[i], np.float64), v=np.asarray(v[i], np.float64))
            for i in range(signs.shape[0])]
