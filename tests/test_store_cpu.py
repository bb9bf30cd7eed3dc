"""Block store (include/bitstack.h bitstack_store_*, csrc/store.cuh): residual blocks on disk as
"basic transmission units" (PAPER.md abstract P:8, Fig.2) readable by record range
(SPEC S:475 read_block_range).  Host code of the library: runs without a GPU.

Pins: byte-exact round trip of every field, deterministic bytes, range reads equal the slice of
a full read, the declared size equals Eq.9 via the oracle, and every corruption
(magic, version, truncation, payload bit flip, random prefixes) is a typed E_IO error.
"""
import os

import numpy as np
import pytest

from oracle import bitstack_oracle as O
from synthetic import make_random_blocks

pkg = pytest.importorskip("paper_2410_23918_b200")


@pytest.fixture(scope="module")
def lib():
    try:
        return pkg.load_library()
    except (FileNotFoundError, OSError) as e:
        pytest.skip(f"library not built: {e}")


def _stacks():
    """Two small stacks in a universal (interleaved) order: (stack, block, signs, u, v, s)."""
    out = []
    shapes = [(96, 160, 16, "bf16"), (64, 200, 8, "f16")]
    data = []
    for sid, (d_out, d_in, k, dt) in enumerate(shapes):
        signs, u, v, s = make_random_blocks(3, d_out, d_in, k, seed=40 + sid)
        if dt == "bf16":
            u, v = O.bf16_bits(u), O.bf16_bits(v)
        else:
            u, v = u.astype(np.float16), v.astype(np.float16)
        data.append((signs, u, v, s, dt))
    for i in range(3):                      # Average order: level by level
        for sid in range(2):
            signs, u, v, s, dt = data[sid]
            out.append((sid, i, signs[i], u[i], v[i], s if i == 0 else None, dt))
    return out


def _write(path, recs):
    with pkg.Store.create(str(path)) as st:
        for sid, i, signs, u, v, s, dt in recs:
            st.append(sid, i, signs, u, v, s, factor_dtype=dt)


def test_round_trip_and_ranges(lib, tmp_path):
    recs = _stacks()
    p = tmp_path / "m.bstk"
    _write(p, recs)
    with pkg.Store.open(str(p)) as st:
        assert len(st) == len(recs)
        full = st.read_range(0, len(recs))
        for (sid, i, signs, u, v, s, dt), (sid2, i2, signs2, u2, v2, s2) in zip(recs, full):
            assert (sid, i) == (sid2, i2)
            np.testing.assert_array_equal(signs, signs2)
            np.testing.assert_array_equal(np.asarray(u).view(np.uint16), u2.view(np.uint16))
            np.testing.assert_array_equal(np.asarray(v).view(np.uint16), v2.view(np.uint16))
            if s is None:
                assert s2 is None
            else:
                np.testing.assert_array_equal(s, s2)
        for a, b in [(0, 0), (2, 3), (5, 1), (1, 4)]:
            part = st.read_range(a, b)
            for x, y in zip(part, full[a:a + b]):
                assert x[:2] == y[:2] and all(np.array_equal(p_, q_) for p_, q_ in zip(x[2:5], y[2:5]))
        for r, (sid, i, signs, u, v, s, dt) in enumerate(recs):
            info = st.info(r)
            d_out, k = np.asarray(u).shape
            d_in = np.asarray(v).shape[0]
            # Eq.9 at 16-bit factors, the oracle's closed form (pinned against Table A.4)
            assert info["size_bits"] == O.block_size_bits(d_out, d_in, k)
            assert info["sign_bytes"] == (d_out * d_in + 7) // 8


def test_deterministic_bytes(lib, tmp_path):
    recs = _stacks()
    _write(tmp_path / "a.bstk", recs)
    _write(tmp_path / "b.bstk", recs)
    assert (tmp_path / "a.bstk").read_bytes() == (tmp_path / "b.bstk").read_bytes()


def test_empty_store(lib, tmp_path):
    p = tmp_path / "e.bstk"
    with pkg.Store.create(str(p)):
        pass
    assert os.path.getsize(p) == 32          # header only
    with pkg.Store.open(str(p)) as st:
        assert len(st) == 0
        assert st.read_range(0, 0) == []


def _err(fn):
    with pytest.raises(pkg.BitStackError) as e:
        fn()
    return e.value.name


def test_corruption_is_a_typed_error(lib, tmp_path):
    recs = _stacks()
    p = tmp_path / "c.bstk"
    _write(p, recs)
    raw = bytearray(p.read_bytes())
    bad = tmp_path / "bad.bstk"
    bad.write_bytes(b"XSTK" + raw[4:])
    assert _err(lambda: pkg.Store.open(str(bad))) == "E_IO"            # BadMagic
    bad.write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    assert _err(lambda: pkg.Store.open(str(bad))) == "E_IO"            # VersionMismatch
    bad.write_bytes(raw[: len(raw) - 5])
    assert _err(lambda: pkg.Store.open(str(bad))) == "E_IO"            # truncated index
    flipped = bytearray(raw)
    with pkg.Store.open(str(p)) as st:
        off = st.info(3)["offset"] + 64 + 10
    flipped[off] ^= 0x10
    bad.write_bytes(bytes(flipped))
    with pkg.Store.open(str(bad)) as st:
        st.read(2)                                                      # other records are fine
        assert _err(lambda: st.read(3)) == "E_IO"                      # CorruptRecord (CRC)
        assert _err(lambda: st.read(len(recs))) == "E_LEVEL_OUT_OF_RANGE"


def test_random_prefixes_never_crash(lib, tmp_path):
    recs = _stacks()
    p = tmp_path / "f.bstk"
    _write(p, recs)
    raw = p.read_bytes()
    rng = np.random.default_rng(3)
    bad = tmp_path / "pre.bstk"
    for cut in sorted(set(rng.integers(0, len(raw), 40).tolist()) | {0, 3, 31, 32, 33}):
        bad.write_bytes(raw[:cut])
        try:
            with pkg.Store.open(str(bad)) as st:
                for r in range(len(st)):
                    st.read(r)
        except pkg.BitStackError as e:
            assert e.name in ("E_IO", "E_LEVEL_OUT_OF_RANGE")


def test_append_validation(lib, tmp_path):
    signs, u, v, s = make_random_blocks(1, 9, 7, 4, seed=1)     # 63 bits: one pad bit
    u16, v16 = O.bf16_bits(u[0]), O.bf16_bits(v[0])
    with pkg.Store.create(str(tmp_path / "v.bstk")) as st:
        assert _err(lambda: st.append(0, 1, signs[0], u16, v16, s)) == "E_INVALID_ARG"   # s only with block 0
        assert _err(lambda: st.append(0, 0, signs[0], u16, v16, None)) == "E_INVALID_ARG"
        bad = signs[0].copy()
        bad[-1] |= 0x80
        assert _err(lambda: st.append(0, 0, bad, u16, v16, s)) == "E_MALFORMED_BUFFER"
        st.append(0, 0, signs[0], u16, v16, s)


@pytest.mark.parametrize("kind", ["average", "random"])
def test_budget_prefix_is_a_contiguous_record_range(lib, tmp_path, kind):
    """Records written in the universal stack's order (budget.py): the blocks a memory
    budget admits (prefix_levels) are exactly records [0, L) for L = the prefix length, and each
    record's size is the Eq.9 block size the budget counts (reading R20)."""
    from paper_2410_23918_b200 import budget as BG
    shapes = [(96, 160, 3), (64, 200, 4), (128, 64, 2)]
    blocks = {}
    for m, (do, di, nb) in enumerate(shapes):
        signs, u, v, s = make_random_blocks(nb, do, di, 8, seed=70 + m)
        blocks[m] = (signs, O.bf16_bits(u), O.bf16_bits(v), s)
    stack = BG.universal_stack([nb for _, _, nb in shapes], kind=kind, seed=5)
    p = tmp_path / "u.bstk"
    with pkg.Store.create(str(p)) as st:
        for m, i in stack:
            signs, u, v, s = blocks[m]
            st.append(m, i, signs[i], u[i], v[i], s if i == 0 else None, factor_dtype="bf16")
    sizes = [BG.block_bytes(do, di, 8) for do, di, _ in shapes]
    with pkg.Store.open(str(p)) as st:
        for r, (m, i) in enumerate(stack):
            info = st.info(r)
            assert (info["stack"], info["block"]) == (m, i)
            assert info["size_bits"] / 8 == sizes[m]
        for budget in [0, sizes[0], 2.5 * max(sizes), 0.5 * sum(sizes[m] for m, _ in stack), 1e12]:
            levels = BG.prefix_levels(stack, sizes, budget)
            L = sum(levels)
            got = {}
            for sid, blk, *_ in st.read_range(0, L):
                got[sid] = got.get(sid, 0) + 1
                assert blk == got[sid] - 1                     # each stack's blocks in order
            assert [got.get(m, 0) for m in range(len(shapes))] == levels
