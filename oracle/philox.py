"""ORACLE (test infrastructure only) -- restatement of the reference's random streams.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline leg may
import this module.  It is the checker, never the product.

The reference keys every draw by ``rng.stream(seed, *path)``
(``/root/reference/pkg/src/gridcast/rng.py:27-31``) which is
``Generator(Philox(SeedSequence(seed & 2**64-1, spawn_key=path & 0xFFFFFFFF)))``.
numpy is an un-vendored dependency of the reference (``pkg/pyproject.toml:10-14``);
the arithmetic below restates numpy 2.3's published algorithms:

* ``SeedSequence`` entropy assembly + hashmix pool (numpy ``bit_generator.pyx``,
  ``get_assembled_entropy`` / ``mix_entropy`` / ``generate_state``), see SURVEY.md App. A.4;
* ``Philox4x64-10`` (Salmon et al. 2011; numpy ``philox.h``): counter incremented
  before each 4-word block, so the first block uses ctr = (1, 0, 0, 0);
* ``random(dtype=float32)``: ``(u32 >> 8) * 2**-24`` drawing u32 halves low-then-high
  from each u64 word; ``random()`` (float64): ``(u64 >> 11) * 2**-53``.

``tests/test_oracle_golden.py`` pins every function here against numpy's own
generator (and the golden fixtures generated from the live reference).
"""

from __future__ import annotations

import numpy as np

M32 = 0xFFFFFFFF
M64 = (1 << 64) - 1

# SeedSequence constants (numpy bit_generator.pyx)
INIT_A = 0x43B0D7E5
MULT_A = 0x931E8875
INIT_B = 0x8B51F9DD
MULT_B = 0x58F38DED
MIX_MULT_L = 0xCA01F9DD
MIX_MULT_R = 0x4973F715
XSHIFT = 16
POOL = 4

# Philox4x64 constants
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def _words(x: int) -> list[int]:
    """Little-endian u32 words of a nonnegative int ([0] for 0)."""
    if x == 0:
        return [0]
    out = []
    while x:
        out.append(x & M32)
        x >>= 32
    return out


def seed_sequence_state(seed: int, path=(), n_words32: int = 4) -> list[int]:
    """``SeedSequence(seed & M64, spawn_key=path & M32).generate_state(n, uint32)``."""
    entropy = _words(int(seed) & M64)
    spawn = []
    for p in path:
        spawn += _words(int(p) & M32)
    if spawn and len(entropy) < POOL:
        entropy = entropy + [0] * (POOL - len(entropy))
    ent = entropy + spawn

    hc = INIT_A

    def hashmix(v):
        nonlocal hc
        v = (v ^ hc) & M32
        hc = (hc * MULT_A) & M32
        v = (v * hc) & M32
        v ^= v >> XSHIFT
        return v

    def mix(x, y):
        r = (MIX_MULT_L * x - MIX_MULT_R * y) & M32
        r ^= r >> XSHIFT
        return r

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(POOL)]
    for s in range(POOL):
        for d in range(POOL):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(POOL, len(ent)):
        for d in range(POOL):
            pool[d] = mix(pool[d], hashmix(ent[s]))

    out = []
    h = INIT_B
    for i in range(n_words32):
        v = pool[i % POOL] ^ h
        h = (h * MULT_B) & M32
        v = (v * h) & M32
        v ^= v >> XSHIFT
        out.append(v)
    return out


def philox_key(seed: int, path=()) -> tuple[int, int]:
    st = seed_sequence_state(seed, path, 4)
    return st[0] | (st[1] << 32), st[2] | (st[3] << 32)


def derive_seed(seed: int, *path) -> int:
    """Restates ``rng.derive_seed`` (``rng.py:34-39``)."""
    k0, k1 = philox_key(seed, path)
    return k0 ^ k1


# --- Philox4x64-10, vectorised over blocks with numpy uint64 ---------------------

_U32 = np.uint64(M32)
_S32 = np.uint64(32)


def _mul64(a: np.ndarray, b: int):
    """(hi, lo) of the 128-bit product a * b, a a uint64 array, b a python int."""
    a = a.astype(np.uint64)
    a_lo = a & _U32
    a_hi = a >> _S32
    b_lo = np.uint64(b & M32)
    b_hi = np.uint64(b >> 32)
    with np.errstate(over="ignore"):
        ll = a_lo * b_lo
        lh = a_lo * b_hi
        hl = a_hi * b_lo
        hh = a_hi * b_hi
        mid = (ll >> _S32) + (lh & _U32) + (hl & _U32)
        hi = hh + (lh >> _S32) + (hl >> _S32) + (mid >> _S32)
        lo = a * np.uint64(b)
    return hi, lo


def philox4x64_blocks(key: tuple[int, int], counters: np.ndarray) -> np.ndarray:
    """Philox4x64-10 output blocks for counters ``(c, 0, 0, 0)``: shape (len, 4) uint64."""
    c0 = np.asarray(counters, dtype=np.uint64)
    c1 = np.zeros_like(c0)
    c2 = np.zeros_like(c0)
    c3 = np.zeros_like(c0)
    k0, k1 = key
    with np.errstate(over="ignore"):
        for _ in range(10):
            hi0, lo0 = _mul64(c0, PHILOX_M0)
            hi1, lo1 = _mul64(c2, PHILOX_M1)
            c0, c1, c2, c3 = (
                hi1 ^ c1 ^ np.uint64(k0),
                lo1,
                hi0 ^ c3 ^ np.uint64(k1),
                lo0,
            )
            k0 = (k0 + PHILOX_W0) & M64
            k1 = (k1 + PHILOX_W1) & M64
    return np.stack([c0, c1, c2, c3], axis=1)


def stream_u64(seed: int, path, n_words: int, first_word: int = 0) -> np.ndarray:
    """Words ``first_word .. first_word+n_words-1`` of ``stream(seed, *path)``."""
    key = philox_key(seed, path)
    w = np.arange(first_word, first_word + n_words, dtype=np.int64)
    blocks = np.unique(w // 4)
    out = philox4x64_blocks(key, blocks.astype(np.uint64) + np.uint64(1))
    lut = {int(b): i for i, b in enumerate(blocks)}
    rows = np.array([lut[int(b)] for b in (w // 4)])
    return out[rows, w % 4]


def stream_random_f32(seed: int, path, n: int) -> np.ndarray:
    """``stream(seed, *path).random(n, dtype=np.float32)``."""
    words = stream_u64(seed, path, (n + 1) // 2)
    lo = (words & _U32).astype(np.uint32)
    hi = (words >> _S32).astype(np.uint32)
    u32 = np.empty(2 * len(words), dtype=np.uint32)
    u32[0::2] = lo
    u32[1::2] = hi
    u32 = u32[:n]
    return ((u32 >> np.uint32(8)).astype(np.float32) * np.float32(1.0 / 16777216.0)).astype(np.float32)


def stream_random_f64(seed: int, path, n: int) -> np.ndarray:
    """``stream(seed, *path).random(n)`` (float64)."""
    words = stream_u64(seed, path, n)
    return (words >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
