// crs.cuh — device core of the coloured random-sequential (CRS) Monte Carlo schedule.
//
// One MCS = one round of four colour phases.  Per round a Philox draw picks the 2x2 tiling origin
// (oy, ox) and the colour order; in each phase every tile of that colour performs 4 sequential
// elementary steps (engine.hpp:108-141) with cell, direction and action drawn from counter-based
// Philox words.  Same-colour tiles have disjoint footprints, so a phase is an exact
// random-sequential update of its tiles in any order.  oracle/escg_oracle.c:orc_crs_run is the
// sequential definition these kernels reproduce bit-exactly (draw spec: DESIGN.md §RNG).
#pragma once
#include <cstdint>

namespace escgd {

constexpr uint32_t kDomStep = 0, kDomRefine = 1, kDomRound = 2, kDomInit = 3;
constexpr uint32_t kKey0 = 0xA4093822u, kKey1 = 0x299F31D0u;

// Philox4x32-10 (Salmon et al. SC'11) with the fixed key: every round key is an immediate, so a
// round is 2 IMAD.WIDE.U32 + 2 LOP3.
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
#ifdef ESCG_DIAG_CHEAP_RNG  // diagnostic builds only (tools/ablate.py): not a valid generator
    const uint32_t h = (c0 * 0x9E3779B9u) ^ (c1 * 0x85EBCA6Bu) ^ c2 ^ c3;
    return make_uint4(h, h * 0xC2B2AE35u, h ^ 0x27D4EB2Fu, h * 0x165667B1u);
#endif
    uint32_t k0 = kKey0, k1 = kKey1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        uint64_t p0, p1;
        asm("mul.wide.u32 %0, %1, %2;" : "=l"(p0) : "r"(c0), "r"(0xD2511F53u));
        asm("mul.wide.u32 %0, %1, %2;" : "=l"(p1) : "r"(c2), "r"(0xCD9E8D57u));
        const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
        const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
        c1 = static_cast<uint32_t>(p1);
        c3 = static_cast<uint32_t>(p0);
        c0 = n0;
        c2 = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return make_uint4(c0, c1, c2, c3);
}

__host__ __device__ __forceinline__ uint32_t murmur_finalize(uint32_t x) {
    x ^= x >> 16;
    x *= 0x85ebca6bu;
    x ^= x >> 13;
    x *= 0xc2b2ae35u;
    x ^= x >> 16;
    return x;
}

// c3 of every draw: the seed folded to 32 bits (identity for seeds < 2^32).
__host__ __device__ __forceinline__ uint32_t seed32(uint64_t seed) {
    return static_cast<uint32_t>(seed) ^ murmur_finalize(static_cast<uint32_t>(seed >> 32));
}

// c2 of every draw: mcs bits 32..47 | domain << 16 | phase << 20 | attempt << 24.
__host__ __device__ __forceinline__ uint32_t ctr2(uint64_t mcs, uint32_t dom, uint32_t phase, uint32_t attempt) {
    return (static_cast<uint32_t>(mcs >> 32) & 0xFFFFu) | (dom << 16) | (phase << 20) | (attempt << 24);
}

// Round parameters (orc_crs_round): origin (oy, ox) and the four colours in phase order.
struct Round {
    int oy, ox;
    uint32_t order;  // colour of phase p in bits 2p..2p+1
    __device__ __forceinline__ int colour(int p) const { return static_cast<int>((order >> (2 * p)) & 3u); }
};

__device__ __forceinline__ Round round_params(uint32_t s32, uint64_t mcs) {
    // Lexicographic permutations of {0,1,2,3}, packed 2 bits per colour (phase 0 in bits 0-1), one
    // byte per permutation in three 64-bit immediates (no local-memory table):
    // E4 B4 D8 78 9C 6C E1 B1 | C9 39 8D 2D D2 72 C6 36 | 4E 1E 93 63 87 27 4B 1B.
    const uint4 w = philox(0u, static_cast<uint32_t>(mcs), ctr2(mcs, kDomRound, 0u, 0u), s32);
    Round r;
    r.oy = static_cast<int>(w.x & 1u);
    r.ox = static_cast<int>((w.x >> 1) & 1u);
    const uint32_t pi = static_cast<uint32_t>((static_cast<uint64_t>(w.y) * 24u) >> 32);
    const uint64_t K = pi < 8u ? 0xB1E16C9C78D8B4E4ull : (pi < 16u ? 0x36C672D22D8D39C9ull : 0x1B4B278763931E4Eull);
    r.order = static_cast<uint32_t>((K >> (8u * (pi & 7u))) & 0xFFu);
    return r;
}

// Phase order for ncy x ncx colours (escg_oracle.c orc_crs_round_g): colour id of
// phase p in nibble p.  Four colours use round_params' table; 6 or 9 a Fisher-Yates shuffle driven by
// the 16-bit halves of a second ROUND draw (attempt field 1).
struct RoundG {
    int oy, ox;
    uint64_t order;
    __device__ __forceinline__ int colour(int p) const { return static_cast<int>((order >> (4 * p)) & 15u); }
};

__device__ __forceinline__ RoundG round_params_g(uint32_t s32, uint64_t mcs, int ncy, int ncx) {
    const Round r4 = round_params(s32, mcs);
    RoundG r;
    r.oy = r4.oy;
    r.ox = r4.ox;
    const int np = ncy * ncx;
    if (np == 4) {
        r.order = 0;
        for (int p = 0; p < 4; ++p) r.order |= static_cast<uint64_t>(r4.colour(p)) << (4 * p);
        return r;
    }
    const uint4 w = philox(0u, static_cast<uint32_t>(mcs), ctr2(mcs, kDomRound, 0u, 1u), s32);
    const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
    uint64_t ord = 0x876543210ull;
    for (int i = np - 1, k = 0; i >= 1; --i, ++k) {
        const uint32_t half = (ws[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
        const int j = static_cast<int>((half * static_cast<uint32_t>(i + 1)) >> 16);
        const uint64_t vi = (ord >> (4 * i)) & 15u, vj = (ord >> (4 * j)) & 15u;
        ord &= ~((15ull << (4 * i)) | (15ull << (4 * j)));
        ord |= (vi << (4 * j)) | (vj << (4 * i));
    }
    r.order = ord;
    return r;
}

// Periodic axis of length n >= 4: tiles T, colours (2 or 3), seam tile (-1 if none).
struct SeamAxis {
    int T, nc, seam;
    __host__ __device__ SeamAxis(int n) {
        T = (n % 4 == 0) ? n / 2 : (n + 1) / 2;
        nc = (n % 4 == 0) ? 2 : 3;
        seam = (n % 4 == 0) ? -1 : ((n % 4 == 3) ? T - 2 : T - 1);
    }
    // tiles of colour c: c < 2 → t = c + 2i (i < count), c == 2 → the seam tile
    __device__ __forceinline__ int count(int c) const {
        if (c == 2) return 1;
        return ((T - c + 1) >> 1) - ((seam >= 0 && (seam & 1) == c) ? 1 : 0);
    }
    __device__ __forceinline__ int tile(int c, int i) const { return c == 2 ? seam : c + 2 * i; }
};

// (drow, dcol) of direction d (params.hpp:81: up, down, left, right, ul, ur, dl, dr).
__host__ __device__ __forceinline__ void dir_rc(uint32_t d, int& dr, int& dc) {
    dr = (d < 4u) ? ((d < 2u) ? ((d & 1u) ? 1 : -1) : 0) : ((d & 2u) ? 1 : -1);
    dc = (d < 4u) ? ((d < 2u) ? 0 : ((d & 1u) ? 1 : -1)) : ((d & 1u) ? 1 : -1);
}

template <int ARITY>
struct Bits {
    static constexpr int DB = ARITY == 8 ? 3 : 2;  // direction bits
    static constexpr int LB = DB + 2;              // direction + cell bits of an attempt
    static constexpr int NT = 1 << LB;             // offset-table entries
    static constexpr int CBN = 16 - LB;            // coarse action bits of a NARROW attempt
};

// ---- 32-bit shared-memory access (volatile: keeps the sequential attempts in program order) ----
__device__ __forceinline__ uint32_t lds8(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts8(uint32_t a, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "r"(v)); }
__device__ __forceinline__ uint2 lds64(uint32_t a) {
    uint2 v;
    asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Per-CTA state of the attempt paths in static shared memory (immediate addresses, no registers):
//   sOffTbl  entry (dir | dy << DB | dx << DB+1) = (cell offset, neighbour offset) from the tile's
//            (0,0) cell in a row-major window of pitch P;
//   sSlow    what only the exact (slow) paths and the WIDE rule read: X_mig, X_int, the smem
//            address of the (S+1)^2 interaction thresholds, S+1.
struct SlowParams {
    uint32_t xm, xi, sT;  // sT: smem address of the coarse pair table (see fill_pair_thresholds)
    int S1;
    const uint32_t* gT;   // exact (S+1)^2 thresholds in global memory (rare exact path)
};
__shared__ int2 sOffTbl[32];
__shared__ SlowParams sSlow;

template <int ARITY>
__device__ __forceinline__ void build_offset_table(int P) {
    for (int e = threadIdx.x; e < Bits<ARITY>::NT; e += blockDim.x) {
        const uint32_t d = static_cast<uint32_t>(e) & (ARITY - 1);
        const int dy = (e >> Bits<ARITY>::DB) & 1, dx = (e >> (Bits<ARITY>::DB + 1)) & 1;
        int dr, dc;
        dir_rc(d, dr, dc);
        const int so = dy * P + dx;
        sOffTbl[e] = make_int2(so, so + dr * P + dc);
    }
}

// Offsets of attempt bits `bits` (low LB bits select the table entry).
template <int ARITY>
__device__ __forceinline__ uint2 offsets(uint32_t bits) {
    const int2 o = sOffTbl[bits & (Bits<ARITY>::NT - 1)];
    return make_uint2(static_cast<uint32_t>(o.x), static_cast<uint32_t>(o.y));
}

// Per-phase constants of the attempt loop (registers).  c2 is the STEP counter word of the phase;
// the REFINE word differs only in the domain field.
struct PhaseCtx {
    uint32_t fast;       // attempt bits below this are certain migrations (NARROW fast path)
    uint32_t xm, xi;     // X_mig, X_int (WIDE rule)
    uint32_t bf;         // WIDE rule form: 1 branch-free (mixed actions), 0 branchy (migration-dominated)
    uint32_t c1, c2, c3;  // draw counter words
};
constexpr uint32_t kStepToRefine = (0u ^ 1u) << 16;  // kDomStep ^ kDomRefine in the domain field

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

// REFINE-domain word of attempt a of `tile` (exact action completion; rare).
static __device__ __noinline__ uint32_t refine_word(uint32_t tile, int a, uint32_t c1, uint32_t c2, uint32_t c3) {
    return philox(tile, c1, (c2 ^ kStepToRefine) | (static_cast<uint32_t>(a) << 24), c3).x;
}

// The rule (engine.hpp:111-140) on (s, n) with the exact 32-bit action word x:
// migration iff x < X_mig, interaction iff X_mig <= x < X_int, else reproduction; interaction
// outcome u < D[a][b] (engine.hpp:125-131) ⇔ x < T[a][b].  Returns ns | nn << 8.
__device__ __forceinline__ uint32_t rule_exact(uint32_t s, uint32_t n, uint32_t x, uint32_t xm, uint32_t xi,
                                               const uint32_t* T, int S1) {
    uint32_t ns = s, nn = n;
    if (x < xm) {
        ns = n;
        nn = s;
    } else if (x >= xi) {
        if (n == 0u)
            nn = s;
        else if (s == 0u)
            ns = n;
    } else if ((s != 0u) & (n != 0u) & (s != n)) {
        if (x < T[s * S1 + n])
            nn = 0u;
        else if (x < T[n * S1 + s])
            ns = 0u;
    }
    return ns | (nn << 8);
}

// Same rule reading the thresholds from shared memory (32-bit address).
__device__ __forceinline__ uint32_t rule_exact_s(uint32_t s, uint32_t n, uint32_t x, uint32_t xm, uint32_t xi,
                                                 uint32_t sT, int S1) {
    uint32_t ns = s, nn = n;
    if (x < xm) {
        ns = n;
        nn = s;
    } else if (x >= xi) {
        if (n == 0u)
            nn = s;
        else if (s == 0u)
            ns = n;
    } else if ((s != 0u) & (n != 0u) & (s != n)) {
        if (x < lds32(sT + 4u * (s * S1 + n)))
            nn = 0u;
        else if (x < lds32(sT + 4u * (n * S1 + s)))
            ns = 0u;
    }
    return ns | (nn << 8);
}

// WIDE exact path: the low LB bits come from REFINE (taken only when a consulted threshold
// shares the coarse value of the word).
template <int ARITY>
__device__ __noinline__ uint32_t slow_wide(uint32_t s, uint32_t n, uint32_t word, uint32_t tile, int a, uint32_t c1,
                                           uint32_t c2, uint32_t c3) {
    constexpr int LB = Bits<ARITY>::LB;
    const uint32_t x = ((word >> LB) << LB) | (refine_word(tile, a, c1, c2, c3) & ((1u << LB) - 1u));
    return rule_exact(s, n, x, sSlow.xm, sSlow.xi, sSlow.gT, sSlow.S1);
}

// NARROW slow path: x = coarse(16-LB bits) << (16+LB) | low (16+LB) bits of the REFINE word.
template <int ARITY>
__device__ __noinline__ uint32_t slow_narrow(uint32_t s, uint32_t n, uint32_t half, uint32_t tile, int a,
                                             uint32_t c1, uint32_t c2, uint32_t c3) {
    constexpr int LB = Bits<ARITY>::LB, SH = 16 + LB;
    const uint32_t x = ((half >> LB) << SH) | (refine_word(tile, a, c1, c2, c3) & ((1u << SH) - 1u));
    return rule_exact(s, n, x, sSlow.xm, sSlow.xi, sSlow.gT, sSlow.S1);
}

// 64-bit shared load under a predicate (no branch); zeros when the predicate is false.
__device__ __forceinline__ uint2 lds64_if(bool p, uint32_t a) {
    uint2 v = make_uint2(0u, 0u);
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\t@q ld.shared.v2.u32 {%0, %1}, [%2];\n\t}"
        : "+r"(v.x), "+r"(v.y)
        : "r"(a), "r"(static_cast<uint32_t>(p)));
    return v;
}

// Coarse pair table of the WIDE rule: entry (s, n) = (T[s][n] & HI, T[n][s] & HI), HI the coarse-bit
// mask of the attempt word.  A coarse word x (low LB bits zero) decides x_exact < T exactly as
// x < (T & HI) unless x == T & HI, which is the exact path (exact T from global memory).
template <int ARITY>
__device__ __forceinline__ void fill_pair_thresholds(uint2* sTp, const uint32_t* T, int S1) {
    constexpr uint32_t HI = ~((1u << Bits<ARITY>::LB) - 1u);
    for (int i = threadIdx.x; i < S1 * S1; i += blockDim.x) {
        const int s = i / S1, n = i - s * S1;
        sTp[i] = make_uint2(T[s * S1 + n] & HI, T[n * S1 + s] & HI);
    }
}

// 32-bit shared load under a predicate (no branch); `dflt` when the predicate is false.
__device__ __forceinline__ uint32_t lds32_if(bool p, uint32_t a, uint32_t dflt) {
    uint32_t v = dflt;
    asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "r"(a), "r"(static_cast<uint32_t>(p)));
    return v;
}

// WIDE rule on the coarse word (low LB bits zero).  A comparison against threshold T is decided by
// the coarse bits unless coarse == T >> LB; those (rare) words take the exact path.  Branch-free:
// the migration / reproduction / interaction outcomes are selects and the interaction thresholds
// predicated loads, so lanes with different actions do not serialise (mixed buckets are the norm
// when P(migration) is 0.8-0.99); only the exact path branches.
template <int ARITY>
__device__ __forceinline__ uint32_t rule_wide(uint32_t s, uint32_t n, uint32_t word, uint32_t tile, int a,
                                              const PhaseCtx& C) {
    constexpr uint32_t HI = ~((1u << Bits<ARITY>::LB) - 1u);
    const uint32_t x = word & HI;
    if (!C.bf) {
        // branchy form: when migrations dominate (P >= 0.97) whole warps take the first branch and
        // never issue the interaction loads
        bool exact = (x == (C.xm & HI)) | (x == (C.xi & HI));
        uint32_t ns = s, nn = n;
        if (!exact) {
            if (x < C.xm) {
                ns = n;
                nn = s;
            } else if (x >= C.xi) {
                if (n == 0u)
                    nn = s;
                else if (s == 0u)
                    ns = n;
            } else if ((s != 0u) & (n != 0u) & (s != n)) {
                // coarse pair (T[s][n] & HI, T[n][s] & HI): x < T ⇔ x < (T & HI) unless they are equal
                const uint2 t = lds64(sSlow.sT + 8u * (s * static_cast<uint32_t>(sSlow.S1) + n));
                exact = (x == t.x) | (x == t.y);
                if (x < t.x)
                    nn = 0u;
                else if (x < t.y)
                    ns = 0u;
            }
        }
        if (exact) return slow_wide<ARITY>(s, n, word, tile, a, C.c1, C.c2, C.c3);
        return ns | (nn << 8);
    }
    const bool mig = x < C.xm, rep = x >= C.xi;
    const bool inter = !mig & !rep & (s != 0u) & (n != 0u) & (s != n);
    const uint2 t = lds64_if(inter, sSlow.sT + 8u * (s * static_cast<uint32_t>(sSlow.S1) + n));
    const uint32_t t1 = t.x, t2 = t.y;  // coarse (masked) thresholds: see fill_pair_thresholds
    const bool exact = (x == (C.xm & HI)) | (x == (C.xi & HI)) | (inter & ((x == t1) | (x == t2)));
    const bool k1 = inter & (x < t1);               // u < D[s][n]: the neighbour dies
    const bool k2 = inter & !(x < t1) & (x < t2);   // else u < D[n][s]: the cell dies
    const bool r1 = rep & (n == 0u), r2 = rep & (n != 0u) & (s == 0u);
    const uint32_t ns = mig ? n : (k2 ? 0u : (r2 ? n : s));
    const uint32_t nn = mig ? s : (k1 ? 0u : (r1 ? s : n));
    if (exact) return slow_wide<ARITY>(s, n, word, tile, a, C.c1, C.c2, C.c3);
    return ns | (nn << 8);
}

// One attempt: `bits` is the 32-bit word (WIDE) or the zero-extended 16-bit half (NARROW).
template <int ARITY, bool NARROW>
__device__ __forceinline__ void attempt(uint32_t bits, uint32_t base, uint32_t tile, int a, const PhaseCtx& C) {
    const uint2 t = offsets<ARITY>(bits);
    const uint32_t sa = base + t.x, na = base + t.y;
    const uint32_t s = lds8(sa), n = lds8(na);
    if (NARROW) {
        if (bits < C.fast) {  // certain migration: exchange (engine.hpp:118-122); s == n is a no-op
            if (s != n) {
                sts8(sa, n);
                sts8(na, s);
            }
            return;
        }
        const uint32_t r = slow_narrow<ARITY>(s, n, bits, tile, a, C.c1, C.c2, C.c3);
        sts8(sa, r & 0xFFu);
        sts8(na, r >> 8);
    } else {
        const uint32_t r = rule_wide<ARITY>(s, n, bits, tile, a, C);
        if (s != n) {  // engine.hpp:113: equal pairs never change
            sts8(sa, r & 0xFFu);
            sts8(na, r >> 8);
        }
    }
}

// Four attempts of a WIDE tile from its own STEP draw.
template <int ARITY>
__device__ __forceinline__ void tile_wide(const uint4 w, uint32_t base, uint32_t tile, const PhaseCtx& C) {
    attempt<ARITY, false>(w.x, base, tile, 0, C);
    attempt<ARITY, false>(w.y, base, tile, 1, C);
    attempt<ARITY, false>(w.z, base, tile, 2, C);
    attempt<ARITY, false>(w.w, base, tile, 3, C);
}

// Four attempts of half h of a NARROW pair draw (words 2h, 2h+1; low half first).
template <int ARITY>
__device__ __forceinline__ void tile_narrow(uint32_t wa, uint32_t wb, uint32_t base, uint32_t tile,
                                            const PhaseCtx& C) {
    attempt<ARITY, true>(wa & 0xFFFFu, base, tile, 0, C);
    attempt<ARITY, true>(wa >> 16, base, tile, 1, C);
    attempt<ARITY, true>(wb & 0xFFFFu, base, tile, 2, C);
    attempt<ARITY, true>(wb >> 16, base, tile, 3, C);
}

// Exchange the pair (a <- vb, b <- va) unless the values are equal (predicated, no branch).
__device__ __forceinline__ void swap_store(uint32_t a, uint32_t b, uint32_t va, uint32_t vb) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, %3;\n\t@p st.shared.u8 [%0], %3;\n\t@p st.shared.u8 [%1], %2;\n\t}" ::"r"(a),
        "r"(b), "r"(va), "r"(vb));
}

// Store a rule result r = ns | nn << 8 unless the pair was equal (engine.hpp:113: no change).
__device__ __forceinline__ void result_store(uint32_t a, uint32_t b, uint32_t s, uint32_t n, uint32_t r) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b32 t0, t1;\n\tsetp.ne.u32 p, %2, %3;\n\tand.b32 t0, %4, 255;\n\tshr.u32 t1, %4, 8;\n\t"
        "@p st.shared.u8 [%0], t0;\n\t@p st.shared.u8 [%1], t1;\n\t}" ::"r"(a),
        "r"(b), "r"(s), "r"(n), "r"(r));
}

// Two disjoint tiles A and B of the same phase, their 4 attempts interleaved (A0 B0 A1 B1 ...):
// each tile's attempts stay in order, the two chains overlap their shared-memory latencies.
// NARROW: bits are 16-bit halves; WIDE: 32-bit words.
template <int ARITY, bool NARROW>
__device__ __forceinline__ void tile_dual_ordered(const uint32_t (&bA)[4], uint32_t baseA, uint32_t tA,
                                                  const uint32_t (&bB)[4], uint32_t baseB, uint32_t tB,
                                                  const PhaseCtx& C) {
#ifdef ESCG_DIAG_NO_ATTEMPTS  // diagnostic: keep the draws live, skip the attempts
    if ((bA[0] ^ bA[1] ^ bA[2] ^ bA[3] ^ bB[0] ^ bB[1] ^ bB[2] ^ bB[3]) == 0x12345u) sts8(baseA, tA);
    return;
#endif
    uint2 oA = offsets<ARITY>(bA[0]), oB = offsets<ARITY>(bB[0]);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t saA = baseA + oA.x, naA = baseA + oA.y, saB = baseB + oB.x, naB = baseB + oB.y;
        const uint32_t sA = lds8(saA), nA = lds8(naA), sB = lds8(saB), nB = lds8(naB);
        if (a < 3) {  // next attempt's offsets do not depend on the lattice
            oA = offsets<ARITY>(bA[a + 1]);
            oB = offsets<ARITY>(bB[a + 1]);
        }
        if (NARROW) {
            const bool fA = bA[a] < C.fast, fB = bB[a] < C.fast;
            if (fA & fB) {  // both certain migrations (engine.hpp:118-122)
                swap_store(saA, naA, sA, nA);
                swap_store(saB, naB, sB, nB);
            } else {
                const uint32_t rA =
                    fA ? (nA | (sA << 8))
                       : slow_narrow<ARITY>(sA, nA, bA[a], tA, a, C.c1, C.c2, C.c3);
                const uint32_t rB =
                    fB ? (nB | (sB << 8))
                       : slow_narrow<ARITY>(sB, nB, bB[a], tB, a, C.c1, C.c2, C.c3);
                result_store(saA, naA, sA, nA, rA);
                result_store(saB, naB, sB, nB, rB);
            }
        } else {
            const uint32_t rA = rule_wide<ARITY>(sA, nA, bA[a], tA, a, C);
            const uint32_t rB = rule_wide<ARITY>(sB, nB, bB[a], tB, a, C);
            result_store(saA, naA, sA, nA, rA);
            result_store(saB, naB, sB, nB, rB);
        }
    }
}

// The upper half-warp runs B's chain first: with a window pitch ≡ 0 (mod 128 bytes) the two
// half-warps then touch the even and the odd banks (DESIGN.md §Shared-memory layout).
template <int ARITY, bool NARROW>
__device__ __forceinline__ void tile_dual(const uint32_t (&bA)[4], uint32_t baseA, uint32_t tA, const uint32_t (&bB)[4],
                                          uint32_t baseB, uint32_t tB, const PhaseCtx& C) {
    const bool sw = (threadIdx.x & 16) != 0;  // data swap (selects), not divergent control flow
    const uint32_t b1[4] = {sw ? bB[0] : bA[0], sw ? bB[1] : bA[1], sw ? bB[2] : bA[2], sw ? bB[3] : bA[3]};
    const uint32_t b2[4] = {sw ? bA[0] : bB[0], sw ? bA[1] : bB[1], sw ? bA[2] : bB[2], sw ? bA[3] : bB[3]};
    tile_dual_ordered<ARITY, NARROW>(b1, sw ? baseB : baseA, sw ? tB : tA, b2, sw ? baseA : baseB, sw ? tA : tB, C);
}

// NARROW pair draw → both tiles, interleaved.
template <int ARITY>
__device__ __forceinline__ void pair_narrow(const uint4 w, uint32_t baseA, uint32_t tA, uint32_t baseB, uint32_t tB,
                                            const PhaseCtx& C) {
    const uint32_t bA[4] = {w.x & 0xFFFFu, w.x >> 16, w.y & 0xFFFFu, w.y >> 16};
    const uint32_t bB[4] = {w.z & 0xFFFFu, w.z >> 16, w.w & 0xFFFFu, w.w >> 16};
    tile_dual<ARITY, true>(bA, baseA, tA, bB, baseB, tB, C);
}

// Two WIDE tiles with their own draws, interleaved.
template <int ARITY>
__device__ __forceinline__ void pair_wide(const uint4 wA, uint32_t baseA, uint32_t tA, const uint4 wB, uint32_t baseB,
                                          uint32_t tB, const PhaseCtx& C) {
    const uint32_t bA[4] = {wA.x, wA.y, wA.z, wA.w};
    const uint32_t bB[4] = {wB.x, wB.y, wB.z, wB.w};
    tile_dual<ARITY, false>(bA, baseA, tA, bB, baseB, tB, C);
}

// Seam variant (periodic axes of any length >= 4, WIDE format): the missing half of an odd axis'
// last tile (part_y / part_x) takes no attempt; everything else is the periodic attempt.
template <int ARITY>
__device__ __forceinline__ void tile_seam(const uint4 w, uint32_t base, uint32_t tile, bool part_y, bool part_x,
                                          const PhaseCtx& C) {
    constexpr int DB = Bits<ARITY>::DB;
    const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t word = words[a];
        if ((part_y && ((word >> DB) & 1u)) || (part_x && ((word >> (DB + 1)) & 1u))) continue;
        attempt<ARITY, false>(word, base, tile, a, C);
    }
}

// Mirror-reflect variant (flux=false, lattice.hpp:42-47; WIDE format only): tile cells outside the
// lattice are skipped (partial edge tiles), neighbours reflect one step inward.  (y0, x0) are the
// global coordinates of the tile's (0,0) cell; the window maps (y, x) to lat0 + (y+R0)*P + x + C0.
template <int ARITY>
__device__ __forceinline__ void tile_reflect(const uint4 w, uint32_t lat0, int y0, int x0, int R0, int C0, int P,
                                             int H, int L, uint32_t tile, const PhaseCtx& C) {
    constexpr int DB = Bits<ARITY>::DB;
    const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t word = words[a];
        const int y = y0 + static_cast<int>((word >> DB) & 1u);
        const int x = x0 + static_cast<int>((word >> (DB + 1)) & 1u);
        if (y < 0 || y >= H || x < 0 || x >= L) continue;
        int dr, dc;
        dir_rc(word & (ARITY - 1), dr, dc);
        int ny = y + dr, nx = x + dc;
        if (ny < 0) ny = -ny;
        if (ny >= H) ny = 2 * (H - 1) - ny;
        if (nx < 0) nx = -nx;
        if (nx >= L) nx = 2 * (L - 1) - nx;
        const uint32_t sa = lat0 + static_cast<uint32_t>((y + R0) * P + x + C0);
        const uint32_t na = lat0 + static_cast<uint32_t>((ny + R0) * P + nx + C0);
        const uint32_t s = lds8(sa), n = lds8(na);
        const uint32_t r = rule_wide<ARITY>(s, n, word, tile, a, C);
        sts8(sa, r & 0xFFu);
        sts8(na, r >> 8);
    }
}

}  // namespace escgd
