"""Host emulation of the fused kernel's tile bookkeeping (bessel_kernels.cu).

These are the integer formulas of the padded, costliest-first sort order, written out
here exactly as the kernel evaluates them, and checked against their plain definitions:
  * the snake chunk order stepped on slot indices, p -> (p ^ 480) + ((p & 256) << 1)
    from p = tid, deals every chunk to exactly one warp (8 warps, 32-slot chunks);
  * the 4-bit per-thread counters widened to the warp scan's 8-bit fields by two byte
    permutes (__byte_perm selectors 0x5140 / 0x7362);
  * the padded key bases: tile totals rounded up to multiples of 32 and prefix-summed
    with SIMD-within-a-register arithmetic on four 16-bit fields per 64-bit word;
  * the fused pass's 11 elements per thread: warp sums on 16-bit fields (8-bit fields
    would carry past 255);
  * the blocked element map j = tid * ITEMS + i: conflict-free binning reads for odd
    ITEMS, and the strided map's ITEMS-way conflicts in a sorted chunk.
No GPU needed.
"""
import math
import os
import random
import re

M64 = (1 << 64) - 1


def snake_chunks(warp, nchunk):
    """Chunks evaluated by `warp` (any lane) of a tile with `nchunk` 32-slot chunks."""
    out, p = [], warp * 32          # lane 0 of the warp: p = tid
    while p < nchunk * 32:
        out.append(p >> 5)
        p = (p ^ 480) + ((p & 256) << 1)
    return out


def test_snake_order_deals_every_chunk_once():
    for nchunk in range(1, 98):     # a padded order spans up to TILE + 8 * 31 slots: 96 chunks at 2816
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
        tile = rng.choice([1536, 1792, 2816, rng.randint(1, 2816)])
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
        if tile == 2816:                 # the f64 fused pass: slot words for TILE + 256 slots
            assert sum(padded) <= 2816 + 256


def widen(c8):
    lo = byte_perm(c8 & 0xFFFFFFFF, 0, 0x4140) | (byte_perm(c8 & 0xFFFFFFFF, 0, 0x4342) << 32)
    hi = byte_perm(c8 >> 32, 0, 0x4140) | (byte_perm(c8 >> 32, 0, 0x4342) << 32)
    return lo, hi


def test_sixteen_bit_warp_sums_for_eleven_items():
    rng = random.Random(3)
    for _ in range(300):
        per_thread = []
        for _t in range(32):
            keys = [rng.choice([0, 1, 5, 7]) if rng.random() < 0.9 else rng.randint(0, 7) for _ in range(11)]
            per_thread.append([keys.count(k) for k in range(8)])
        words = [0, 0, 0, 0]                       # the four 32-bit REDUX sums
        for counts in per_thread:
            c4 = sum(c << (4 * k) for k, c in enumerate(counts))
            ev, od = c4 & 0x0F0F0F0F, (c4 >> 4) & 0x0F0F0F0F
            c8 = byte_perm(ev, od, 0x5140) | (byte_perm(ev, od, 0x7362) << 32)
            lo, hi = widen(c8)
            for w, val in enumerate((lo & 0xFFFFFFFF, lo >> 32, hi & 0xFFFFFFFF, hi >> 32)):
                words[w] = (words[w] + val) & 0xFFFFFFFF
        got = [(words[k // 2] >> (16 * (k % 2))) & 0xFFFF for k in range(8)]
        assert got == [sum(c[k] for c in per_thread) for k in range(8)]


def bank_pairs(elems):
    """Shared-memory wavefronts of one warp's 8-byte accesses: 32 banks of 4 bytes, so
    element j occupies banks 2j, 2j+1 (mod 32); distinct elements on the same banks serialise."""
    per_bank = {}
    for j in elems:
        per_bank.setdefault((2 * j) % 32, set()).add(j)
    return max(len(v) for v in per_bank.values())


def test_blocked_map_binning_reads_are_conflict_free_for_odd_items():
    for items in (7, 9, 11):
        for i in range(items):
            # a warp's 32 lanes read element tid * ITEMS + i: two per bank pair (the minimum
            # for 8-byte words, one 128-byte wavefront per 16 lanes)
            assert bank_pairs([t * items + i for t in range(32)]) == 2


def test_sorted_chunk_conflicts_strided_vs_blocked():
    # a mixed tile sorts a thread's elements of one key into consecutive slots: a chunk of
    # 32 slots holds runs of ITEMS elements of ~32 / ITEMS threads
    items, tpb = 11, 256
    run_threads = [0, 1, 2]
    strided = [t + i * tpb for t in run_threads for i in range(items)][:32]
    blocked = [t * items + i for t in run_threads for i in range(items)][:32]
    assert bank_pairs(strided) == items       # every element of a run on one bank pair
    assert bank_pairs(blocked) == 2           # consecutive words


def test_fused_tile_constant_matches_kernel_source():
    """tests/test_gpu_bessel.py builds its every-bin-every-tile case on FUSED_TILE."""
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2409_08729_b200", "csrc",
                            "bessel_kernels.cu")).read()
    macro = lambda name: int(re.search(r"#define %s (\d+)" % name, src).group(1))
    assert macro("B200_SB") == 1 and macro("B200_TPB") == 256
    from test_gpu_bessel import FUSED_TILE
    assert FUSED_TILE == macro("B200_TPB") * macro("B200_SB_ITEMS")


def _macro_hex(name):
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2409_08729_b200", "csrc", "tables.h")).read()
    return int(re.search(r"#define %s (0x[0-9A-Fa-f]+)u" % name, src).group(1), 16)


def test_slow_bin_order_test_folds_the_sign():
    """bin_of for log I and the fused pass tests the order with one unsigned compare of the
    raw high word, hvs > HI; it must equal the earlier three-part test
    hv > HI or hvs != hv (|v| above the range, NaN / inf, v < 0, -0.0), hv = hvs & 0x7FFFFFFF,
    for every double (f64 high words) and every float (f32 bit patterns)."""
    import struct
    rng = random.Random(5)
    specials = [0.0, -0.0, 1.0, -1.0, 1e140, 1.0000000001e140, -1e140, 9.99e139, float("inf"),
                float("-inf"), float("nan"), -float("nan"), 5e-324, -5e-324, 1e-300, 1e300, -1e300]
    for hi_name, fmt, width in (("B200_HW_HI", "<d", 64), ("B200_F32_HI32", "<f", 32)):
        HI = _macro_hex(hi_name)
        vals = specials + [rng.choice([-1, 1]) * 10 ** rng.uniform(-307, 307) for _ in range(5000)]
        for v in vals:
            try:
                bits = int.from_bytes(struct.pack(fmt, v), "little")
            except OverflowError:                       # beyond the float range: +-inf
                bits = int.from_bytes(struct.pack(fmt, math.copysign(float("inf"), v)), "little")
            hvs = bits >> 32 if width == 64 else bits
            hv = hvs & 0x7FFFFFFF
            assert (hvs > HI) == (hv > HI or hvs != hv), (v, hex(hvs))
        for hvs in [rng.getrandbits(32) for _ in range(20000)] + [HI, HI + 1, HI | 0x80000000, 0x80000000]:
            hv = hvs & 0x7FFFFFFF
            assert (hvs > HI) == (hv > HI or hvs != hv)
