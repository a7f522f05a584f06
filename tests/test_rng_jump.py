"""The threaded S^(0) draw: every host thread (and every device warp) positions
its own mt19937_64 at its slice of the reference's ONE sequential stream
(rng.hpp:22-49, smoothing.hpp:84-92) by jump-ahead, so the output must stay bit
for bit that of the serial loop. CPU checks of the jump polynomials, the
jumped generator, the threaded normal stream and its rejection fallback."""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2601_20174_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _words(seed, skip, count, jump):
    out = np.empty(count, dtype=np.uint64)
    lib = L.inputs_lib()
    if jump:
        assert lib.nlsp_mt19937_64_jump_fill(seed, skip, count, L.u64ptr(out)) == 0
    else:
        lib.nlsp_mt19937_64_fill(seed, skip, count, L.u64ptr(out))
    return out


def test_jump_table_is_what_the_generator_script_derives(tmp_path):
    """mt_jump_table.inc is generated: the script re-derives phi by
    Berlekamp-Massey, checks x^(2^j) mod phi against plain stepping and must
    reproduce the committed table byte for byte."""
    out = tmp_path / "table.inc"
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "make_mt_jump_table.py"), "--out", str(out)],
                   check=True, timeout=300)
    committed = open(os.path.join(ROOT, "paper_2601_20174_b200", "csrc", "mt_jump_table.inc")).read()
    assert out.read_text() == committed


def test_known_answer_of_mt19937_64():
    # the 10000th output of a default-seeded std::mt19937_64 (C++ standard, [rand.predef])
    assert int(_words(5489, 9999, 1, jump=False)[0]) == 9981545732273789042


@pytest.mark.parametrize("skip", [1 << 17, (1 << 17) + (1 << 19), 5 << 20, (1 << 24) + (1 << 17)])
def test_jumped_generator_equals_discard(skip):
    a = _words(20174, skip, 2000, jump=False)
    b = _words(20174, skip, 2000, jump=True)
    assert np.array_equal(a, b)


def test_jump_rejects_untabulated_distances():
    out = np.empty(4, dtype=np.uint64)
    assert L.inputs_lib().nlsp_mt19937_64_jump_fill(1, 12345, 4, L.u64ptr(out)) != 0


def _serial(seed, count, zero_below=0.0):
    out = np.empty(count)
    L.inputs_lib().nlsp_rng_normal_serial(seed, count, zero_below, L.dptr(out))
    return out


def _chunks(seed, count, chunk_pairs, zero_below=0.0, workers=0):
    out = np.full(count, np.nan)
    L.inputs_lib().nlsp_rng_normal_chunks(seed, count, chunk_pairs, zero_below, workers, L.dptr(out))
    return out


@pytest.mark.parametrize("count,chunk,workers", [
    ((1 << 22) + 3, 1 << 18, 0),   # odd count, several chunks, all threads
    (3 * (1 << 20), 1 << 19, 2),   # even count ending on a chunk boundary, two workers
    ((1 << 21) + 12346, 1 << 20, 4),
    (1001, 1 << 18, 0),            # shorter than a chunk: the serial path
    (1 << 20, 3 << 16, 0),         # a chunk that is no power of two: the serial path
])
def test_threaded_normal_stream_is_the_serial_loop(count, chunk, workers):
    assert np.array_equal(_chunks(991, count, chunk, 0.0, workers), _serial(991, count))


def test_threaded_stream_hands_over_at_a_rejected_uniform():
    """`while (u1 <= 0) u1 = uniform()` (rng.hpp:43) shifts the rest of the
    stream by a word, which only a sequential pass can follow: with the
    rejection widened to u1 <= 2e-6 it happens a few times in 2^22 pairs, and
    the threaded stream must still equal the serial loop from there on."""
    count, zb = (1 << 23) + 1, 2e-6
    ref = _serial(4242, count, zb)
    assert not np.array_equal(ref, _serial(4242, count))  # the rejection did fire
    assert np.array_equal(_chunks(4242, count, 1 << 18, zb), ref)


def test_default_fill_is_the_serial_loop():
    # nlsp_rng_normal_fill / nlsp_smoothed_s0 (bench.py, the goldens) at a size that takes the threaded path
    count = (1 << 23) + (1 << 20) + 1
    out = np.empty(count)
    L.inputs_lib().nlsp_rng_normal_fill(77, count, L.dptr(out))
    assert np.array_equal(out, _serial(77, count))
