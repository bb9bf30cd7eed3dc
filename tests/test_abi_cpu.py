"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports
every symbol include/bitstack.h declares; host-only entry points behave."""
import ctypes
import os
import re
import subprocess

import pytest

from bitstack_test_helpers import read_golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_23918_b200 import build as B
    B.build()
    from paper_2410_23918_b200 import bitstack as bsmod
    return bsmod.load_library()


def header_symbols():
    with open(os.path.join(ROOT, "include", "bitstack.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"BITSTACK_API\s+[\w\s\*]+?\b(bitstack_\w+)\s*\(", text)))


def test_header_declares_the_four_north_star_calls():
    syms = header_symbols()
    for name in ("bitstack_load_blocks", "bitstack_set_num_blocks", "bitstack_matmul", "bitstack_reconstruct"):
        assert name in syms


def test_library_exports_every_header_symbol(lib):
    from paper_2410_23918_b200 import bitstack as bsmod
    out = subprocess.run(["nm", "-D", "--defined-only", bsmod.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (bitstack_\w+)", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing
    assert set(bsmod.EXPORTED_SYMBOLS) == set(header_symbols())
    for s in header_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a_with_tcgen05(lib):
    """The fatbin holds sm_100a SASS with tcgen05 MMA (UTCHMMA), TMEM st/ld and bulk copies."""
    from paper_2410_23918_b200 import bitstack as bsmod
    sass = subprocess.run(["cuobjdump", "-sass", bsmod.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", bsmod.LIB_PATH], capture_output=True,
                                       text=True).stdout
    for mnemonic in ("UTCHMMA", "STTM", "LDTM", "UBLKCP"):
        assert mnemonic in sass, mnemonic


def test_block_size_bits_matches_table_a4(lib, golden_dir):
    """Eq.9 as computed by the library reproduces Table A.4."""
    from decimal import ROUND_HALF_UP, Decimal
    for _, _, m, n, printed in read_golden(os.path.join(golden_dir, "table_a4.txt")):
        bits = lib.bitstack_block_size_bits(int(m), int(n), 16, 16)
        mib = Decimal(bits) / Decimal(8 * 2 ** 20)
        assert mib.quantize(Decimal("0.01"), rounding=ROUND_HALF_UP) == Decimal(printed)
    assert lib.bitstack_block_size_bits(4096, 4096, 16, 32) == 4096 * 4096 + 32 * 16 * 8192


def test_create_rejects_bad_arguments_without_gpu(lib):
    """Argument validation happens before any device call; no GPU here -> clean error."""
    from paper_2410_23918_b200 import bitstack as bsmod
    h = ctypes.c_void_p()
    assert lib.bitstack_create(64, 64, 0, 4, 1, 0, 64, 0, ctypes.byref(h)) == -1       # k < 1
    assert lib.bitstack_create(64, 64, 33, 4, 1, 0, 64, 0, ctypes.byref(h)) == -1      # k > 32
    assert lib.bitstack_create(64, 64, 16, 4, 7, 0, 64, 0, ctypes.byref(h)) == -1      # dtype
    assert lib.bitstack_create(64, 64, 16, 4, 1, 10, 5, 0, ctypes.byref(h)) == -2      # rows
    assert lib.bitstack_create(64, 64, 16, 4, 1, 0, 65, 0, ctypes.byref(h)) == -2
    assert b"row range" in lib.bitstack_last_error()
    assert lib.bitstack_set_num_blocks(None, 0) == -1
    assert lib.bitstack_matmul(None, None, 0, None, 0, 1, None) == -1
    with pytest.raises(bsmod.BitStackError):
        bsmod.Layer(64, 64, k=0)


def test_grouped_load_and_compress_validate_without_gpu(lib):
    """Host-side validation of the later entry points (no device call needed)."""
    from paper_2410_23918_b200 import bitstack as bsmod
    VP = ctypes.c_void_p
    # grouped: count 0 is a no-op; NULL arrays with count > 0 are rejected
    assert lib.bitstack_matmul_grouped(None, 0, None, 1, None, 0, 1, None) == 0
    assert lib.bitstack_matmul_grouped(None, 2, None, 1, None, 0, 1, None) == -1
    # async load: NULL handle, like the synchronous one
    assert lib.bitstack_load_blocks_async(None, 0, 1, None, None, None, None, None) == -1
    assert lib.bitstack_load_blocks(None, 0, 1, None, None, None, None, None) == -1
    # compress: NULL inputs, bad k, bad sizes -- all before touching a device
    assert lib.bitstack_compress(None, None, 1, 8, 8, 1, 4, 1, 0, 0, 0, None, None, None, None, None, None, None) == -1
    dummy = VP(1)
    assert lib.bitstack_compress(dummy, dummy, 1, 8, 8, 1, 0, 1, 0, 0, 0, dummy, dummy, dummy, dummy, None, None,
                                 None) == -1                                     # k < 1
    assert lib.bitstack_compress(dummy, dummy, 1, 64, 64, 1, 33, 1, 0, 0, 0, dummy, dummy, dummy, dummy, None, None,
                                 None) == -1                                     # k > 32
    assert b"k=33" in lib.bitstack_last_error()
    assert lib.bitstack_compress(dummy, dummy, 0, 8, 8, 1, 4, 1, 0, 0, 0, dummy, dummy, dummy, dummy, None, None,
                                 None) == -1                                     # p < 1
    # Python-side argument checks of the grouped helpers
    with pytest.raises(ValueError):
        bsmod.Group([], [1], [])
    assert bsmod.matmul_grouped([], []) == []


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: pointing the binding at a missing library raises instead of computing."""
    import subprocess
    import sys
    code = ("import os, sys; sys.path.insert(0, %r); os.environ['BITSTACK_LIB'] = %r\n"
            "import paper_2410_23918_b200 as bs\n"
            "try:\n    bs.Layer(64, 64)\nexcept FileNotFoundError as e:\n    print('LOUD', e)\n") % (
        ROOT, str(tmp_path / "missing.so"))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert "LOUD" in out.stdout and "no CPU fallback" in out.stdout, out.stdout + out.stderr


def _build_c_demo(tmp_path):
    import shutil
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    exe = tmp_path / "abi_demo"
    lib_dir = os.path.join(ROOT, "paper_2410_23918_b200")
    subprocess.run(["gcc", "-O2", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "abi_demo.c"), "-L", lib_dir, "-lbitstack", "-lm",
                    f"-Wl,-rpath,{lib_dir}", "-o", str(exe)], check=True)
    return exe


def test_c_demo_compiles_links_and_fails_cleanly_without_gpu(lib, tmp_path):
    """The header is plain C99 and the library links from C; without a GPU the first call
    returns an ABI status (no crash, no exception across the boundary)."""
    exe = _build_c_demo(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    if out.returncode == 0:      # a GPU is present: the demo ran to completion
        assert "OK" in out.stdout
    else:
        assert out.returncode == 2 and "bitstack_create: status" in out.stdout, out.stdout + out.stderr
