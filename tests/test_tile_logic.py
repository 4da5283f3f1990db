"""Host emulation of the fused kernel's tile bookkeeping (bessel_kernels.cu).

These are the integer formulas of the padded, costliest-first sort order, written out
here exactly as the kernel evaluates them, and checked against their plain definitions:
  * the snake chunk order stepped on slot indices, p -> (p ^ 480) + ((p & 256) << 1)
    from p = tid, deals every chunk to exactly one warp (8 warps, 32-slot chunks);
  * the 4-bit per-thread counters widened to the warp scan's 8-bit fields by two byte
    permutes (__byte_perm selectors 0x5140 / 0x7362);
  * the padded key bases: tile totals rounded up to multiples of 32 and prefix-summed
    with SIMD-within-a-register arithmetic on four 16-bit fields per 64-bit word.
No GPU needed.
"""
import random

M64 = (1 << 64) - 1


def snake_chunks(warp, nchunk):
    """Chunks evaluated by `warp` (any lane) of a tile with `nchunk` 32-slot chunks."""
    out, p = [], warp * 32          # lane 0 of the warp: p = tid
    while p < nchunk * 32:
        out.append(p >> 5)
        p = (p ^ 480) + ((p & 256) << 1)
    return out


def test_snake_order_deals_every_chunk_once():
    for nchunk in range(1, 57):     # a padded order spans up to TILE + 8 * 31 slots: 56 chunks
        seen = []
        for w in range(8):
            ch = snake_chunks(w, nchunk)
            if w < nchunk:
                assert ch[0] == w
            seen += ch
        assert sorted(seen) == list(range(nchunk))


def test_snake_order_alternates_direction():
    # round r of eight chunks goes to warps 0..7 when r is even and 7..0 when r is odd
    for w in range(8):
        ch = snake_chunks(w, 56)
        for r, c in enumerate(ch):
            assert c == 8 * r + (w if r % 2 == 0 else 7 - w)


def test_snake_step_is_lane_independent():
    # the step maps every lane of a chunk to the same next chunk, lane kept
    for p in range(56 * 32):
        q = (p ^ 480) + ((p & 256) << 1)
        assert q & 31 == p & 31
        assert q >> 5 == ((p >> 5) ^ 15) + (16 if (p >> 5) & 8 else 0)


def byte_perm(a, b, sel):
    src = [(a >> (8 * i)) & 255 for i in range(4)] + [(b >> (8 * i)) & 255 for i in range(4)]
    return sum(src[(sel >> (4 * k)) & 7] << (8 * k) for k in range(4))


def test_four_bit_counters_widen_to_byte_fields():
    rng = random.Random(1)
    for _ in range(2000):
        counts = [rng.randint(0, 7) for _ in range(8)]   # ITEMS <= 7 per thread and key
        c4 = sum(c << (4 * k) for k, c in enumerate(counts))
        ev, od = c4 & 0x0F0F0F0F, (c4 >> 4) & 0x0F0F0F0F
        c8 = byte_perm(ev, od, 0x5140) | (byte_perm(ev, od, 0x7362) << 32)
        assert [(c8 >> (8 * k)) & 255 for k in range(8)] == counts


def test_padded_bases_by_swar_prefix():
    ONES = 0x0001000100010001
    F32 = 0xFFE0FFE0FFE0FFE0
    rng = random.Random(2)
    for _ in range(2000):
        tile = rng.choice([1536, 1792, rng.randint(1, 1536)])
        cuts = sorted(rng.randint(0, tile) for _ in range(7))
        counts = [b - a for a, b in zip([0] + cuts, cuts + [tile])]
        tlo = sum(counts[k] << (16 * k) for k in range(4))
        thi = sum(counts[4 + k] << (16 * k) for k in range(4))
        qlo, qhi = (tlo + 31 * ONES) & F32, (thi + 31 * ONES) & F32
        tp = (qlo * ONES) & M64
        blo = (tp - qlo) & M64
        bhi = (qhi * ONES - qhi + (tp >> 48) * ONES) & M64
        nchunk = (((bhi + qhi) & M64) >> 48) >> 5
        padded = [(c + 31) // 32 * 32 for c in counts]
        bases = [sum(padded[:k]) for k in range(8)]
        got = [(blo >> (16 * k)) & 0xFFFF for k in range(4)] + [(bhi >> (16 * k)) & 0xFFFF for k in range(4)]
        assert got == bases
        assert nchunk == sum(padded) // 32
        assert sum(padded) <= tile + 8 * 31
        if tile == 1536:                 # the f64 fused pass: slot words for TILE + 256 slots
            assert sum(padded) <= 1536 + 256
