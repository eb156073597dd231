"""32-bit rANS coder, one lane (oracle; test infrastructure only).

P:98-101 — "We used the rANS variant for our coder."  P:103 — "In the GPU
implementation, we opted for 32-bit arithmetic".  The paper gives no
constants; reading R6: state x in [2^16, 2^32), 16-bit words,
precision k <= 16 (k = 16 for images), renormalise BEFORE encoding with at
most one word per symbol, initial state 2^16, final state flushed as two
words (high first); the decoder's final state returns to 2^16.

Python integers are unbounded, so every bound is asserted explicitly.
"""

from __future__ import annotations

import bisect

L = 1 << 16         # lower bound of the normalised interval
WORD_BITS = 16
WORD_MASK = 0xFFFF


def encode_symbol(x: int, f: int, c: int, k: int, emit) -> int:
    """Renormalise then x' = floor(x/f)*2^k + x mod f + c."""
    assert L <= x < (1 << 32) and 1 <= f <= (1 << k) and 0 <= c and c + f <= (1 << k)
    if x >= (f << (32 - k)):
        emit(x & WORD_MASK)
        x >>= WORD_BITS
        assert x < (f << (32 - k))
    x = ((x // f) << k) + (x % f) + c
    assert L <= x < (1 << 32)
    return x


def decode_symbol(x: int, freqs, cums, k: int, read):
    """slot = x mod 2^k; s: c_s <= slot < c_s + f_s; x' = f_s*(x>>k) + slot - c_s;
    then while x' < 2^16 read a word (at most one).  Returns (s, x')."""
    slot = x & ((1 << k) - 1)
    # s = max{i : c_i <= slot} (cums ascending; library binary search)
    s = bisect.bisect_right(cums, slot) - 1
    f, c = int(freqs[s]), int(cums[s])
    assert c <= slot < c + f
    x = f * (x >> k) + slot - c
    if x < L:
        x = (x << WORD_BITS) | read()
        assert x >= L
    return s, x


def encode_symbol_raw(x: int, f: int, c: int, k: int) -> int:
    """The state update alone, without renormalisation (SPEC S:63-65 examples
    use x below L to show the formula)."""
    return ((x // f) << k) + (x % f) + c


def decode_symbol_raw(x: int, freqs, cums, k: int):
    slot = x & ((1 << k) - 1)
    s = max(i for i in range(len(cums)) if cums[i] <= slot)
    return s, freqs[s] * (x >> k) + slot - cums[s]


def encode_sequence(symbols, tables, k: int = 16):
    """Encode in REVERSE (LIFO), flush hi then lo; returns list of 16-bit words
    in decoder read order.  tables[i] = (freqs, cums)."""
    x = L
    out = []
    for i in range(len(symbols) - 1, -1, -1):
        freqs, cums = tables[i]
        s = symbols[i]
        x = encode_symbol(x, freqs[s], cums[s], k, out.append)
    words = [x >> 16, x & WORD_MASK] + out[::-1]
    return words


class Underflow(Exception):
    """StreamUnderflow."""


def decode_sequence(words, tables, k: int = 16):
    """Inverse of encode_sequence; checks the final-state invariant."""
    if len(words) < 2:
        raise Underflow("no state")
    x = (words[0] << 16) | words[1]
    pos = [2]

    def read():
        if pos[0] >= len(words):
            raise Underflow("stream exhausted")
        w = words[pos[0]]
        pos[0] += 1
        return w

    out = []
    for freqs, cums in tables:
        s, x = decode_symbol(x, freqs, cums, k, read)
        out.append(s)
    return out, x, pos[0]


def words_to_bytes(words) -> bytes:
    """Little-endian 16-bit words."""
    b = bytearray()
    for w in words:
        b += int(w).to_bytes(2, "little")
    return bytes(b)


def bytes_to_words(b: bytes):
    assert len(b) % 2 == 0
    return [int.from_bytes(b[i:i + 2], "little") for i in range(0, len(b), 2)]
