// slice_common.cuh — pieces shared by the bit-sliced kernels (slice.cu: overlapped-tile windows;
// ring.cu: persistent row bands with per-phase neighbour exchange).  DESIGN.md §2.3, §3.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

#include "crs.cuh"

// Checked builds (ESCG_CHECKED; tools/sanitize_cases.py — compute-sanitizer is closed on this pool):
// device asserts on shared-memory window rows and columns, queue and mailbox slots, snapshot rows.
#ifdef ESCG_CHECKED
#undef NDEBUG
#include <cassert>
#define ESCG_CHECK(c) assert(c)
#else
#define ESCG_CHECK(c) ((void)0)
#endif

namespace escgd {
namespace {

#ifdef ESCG_DIAG_SLICE
// diagnostic builds only (tools/slice_diag.py): clock64 stamps of CTA 0..3, warps 0..15, phases 0..7
__device__ long long g_sdiag[4][16][8][8];
#define SDIAG(ph, ev)                                                                                  \
    do {                                                                                              \
        const int cta_ = blockIdx.x + gridDim.x * blockIdx.y;                                         \
        if (cta_ < 4 && (threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < 16 && (ph) < 8)                \
            g_sdiag[cta_][threadIdx.x >> 5][ph][ev] = clock64();                                      \
    } while (0)
#else
#define SDIAG(ph, ev)
#endif
constexpr uint32_t kDomSlice = 4, kDomSliceRef = 5;
constexpr int kMaxSliceSpecies = 7;  // NPL <= 3 bit planes
constexpr unsigned kSliceQueue = 512;  // deferred tiles per phase replayed CTA-wide
constexpr uint32_t kFull = 0xffffffffu;

__device__ __forceinline__ uint4 lds128(const uint32_t* p) { return *reinterpret_cast<const uint4*>(p); }
// ordered shared load (the replay's next attempt reads what the previous one's red.xor wrote)
__device__ __forceinline__ uint32_t lds32o(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts128(uint32_t* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

// Shared-memory words per window row: NPL planes x Gw groups x 4 quads, padded to 4 (mod 8) words
// so that the two tile rows of a quarter-warp (Gw = 4) hit disjoint bank quads.
__host__ __device__ __forceinline__ int row_words(int npl, int gw) {
    const int base = npl * gw * 4;
    return (base & 7) == 0 ? base + 4 : base;
}

// Exact replay of one tile whose attempts left the bit-parallel pass (engine.hpp:108-141), on the
// tile's 12 footprint cells held as 3-bit fields of one register: the cells are read once, the four
// attempts run branch-free in registers, and the changed bits are written back with shared-memory
// XOR reductions (neighbouring lanes share the boundary words).  sw0 = shared address of the
// window; code: 4 choice bits per attempt (cell row, cell column, direction) in nibble a,
// undecided flag of attempt a in bit 16 + a.  Footprint positions: 0 (0,1) 1 (0,2) 2 (1,0) 3 (1,1)
// 4 (1,2) 5 (1,3) 6 (2,0) 7 (2,1) 8 (2,2) 9 (2,3) 10 (3,1) 11 (3,2) as (row - w + 1, col - acol + 1).
template <int NPL>
__device__ __forceinline__ void slice_replay(uint32_t sw0, int RP, int Gw, int w, int acol, uint32_t code,
                                             uint32_t item, int l, uint32_t c1, uint32_t c2r, uint32_t s32, uint32_t xm,
                                             uint32_t xi, uint32_t TK, uint32_t sT, int S1, int qd = 8, int Wc = 0) {
    constexpr int kRow[12] = {0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3};
    constexpr int kCol[12] = {1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 1, 2};
    constexpr uint32_t kCellPos = 0x8473u;               // position of cell (Y, X): nibble Y | X << 1
    constexpr uint64_t kNbrPos = 0x95847362b8a74130ull;  // neighbour position: nibble Y | X << 1 | dir << 2
    if (Wc == 0 && (acol < 1 || acol + 2 >= 128 * Gw)) return;  // window edge: margin cells, never stored
#ifdef ESCG_DIAG_REPLAY_NOPHILOX
    const uint4 rf = make_uint4(item ^ c1, c2r + l, s32, item);
#else
    const uint4 rf = philox(item, c1, c2r | (static_cast<uint32_t>(l) << 24), s32);
#endif
    const uint32_t PS = static_cast<uint32_t>(Gw) * 16u;  // plane stride (bytes)
    uint32_t addr[12], bit[12];
    uint64_t cells = 0;
#pragma unroll
    for (int k = 0; k < 12; ++k) {
        const int row = w - 1 + kRow[k];
        int col = acol - 1 + kCol[k];
        if (Wc) col = col < 0 ? col + Wc : (col >= Wc ? col - Wc : col);  // full-width rows wrap
        ESCG_CHECK(row >= 0 && col >= 0 && col < 128 * Gw);
        addr[k] = sw0 + 4u * static_cast<uint32_t>(row * RP + (col >> 7) * 4 + (col & 3));
        bit[k] = (static_cast<uint32_t>(col) >> 2) & 31u;
        uint32_t v = 0;
#pragma unroll
        for (int p = 0; p < NPL; ++p) v |= ((lds32o(addr[k] + p * PS) >> bit[k]) & 1u) << p;
        cells |= static_cast<uint64_t>(v) << (3 * k);
    }
#ifdef ESCG_DIAG_SLICE
    if ((cells + rf.x) != 1u) SDIAG(qd, 6);
#endif
    const uint64_t cells0 = cells;
    const uint32_t rw[4] = {rf.x, rf.y, rf.z, rf.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t cb = (code >> (4 * a)) & 15u;
        const uint32_t ps = (kCellPos >> (4 * (cb & 3u))) & 15u, pn = static_cast<uint32_t>(kNbrPos >> (4 * cb)) & 15u;
        const uint32_t s = static_cast<uint32_t>(cells >> (3 * ps)) & 7u, n = static_cast<uint32_t>(cells >> (3 * pn)) & 7u;
        // the rule (engine.hpp:111-140) with selects; a decided attempt is a certain migration
        const bool und = (code >> (16 + a)) & 1u;
        const uint32_t x = TK | (rw[a] & ~TK);
        const bool mig = !und || x < xm, rep = und && x >= xi;
        const bool inter = !mig && !rep && s != 0u && n != 0u && s != n;
        const uint32_t t1 = lds32_if(inter, sT + 4u * (s * S1 + n), 0u);
        const uint32_t t2 = lds32_if(inter, sT + 4u * (n * S1 + s), 0u);
        const bool kn = inter && x < t1, ks = inter && !(x < t1) && x < t2;
        const bool r1 = rep && n == 0u, r2 = rep && n != 0u && s == 0u;
        const uint32_t ns = mig ? n : (ks ? 0u : (r2 ? n : s));
        const uint32_t nn = mig ? s : (kn ? 0u : (r1 ? s : n));
        cells = (cells & ~((7ull << (3 * ps)) | (7ull << (3 * pn)))) | (static_cast<uint64_t>(ns) << (3 * ps)) |
                (static_cast<uint64_t>(nn) << (3 * pn));
    }
    const uint64_t delta = cells ^ cells0;
#ifdef ESCG_DIAG_SLICE
    if (delta != 1u) SDIAG(qd, 5);
#endif
#ifndef ESCG_DIAG_REPLAY_NOATOM
#pragma unroll
    for (int k = 0; k < 12; ++k)
#pragma unroll
        for (int p = 0; p < NPL; ++p)
            if ((delta >> (3 * k + p)) & 1u)
                asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(addr[k] + p * PS), "r"(1u << bit[k]) : "memory");
#else
    if (delta == 0x123456789ull) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(addr[0]), "r"(1u) : "memory");
#endif
}

// Group replay: the 8 lanes of group (lane >> 3) replay one tile together.  Lane j reads and writes
// footprint positions j and j + 8 (the 24 shared-memory reads and up to 24 XOR reductions of a
// tile are spread over the group); the packed cells are OR-combined with shuffles, and every lane
// of the group runs the four attempts on the same register copy (the exact rule, branch-free).
template <int NPL>
__device__ __forceinline__ void slice_replay_group(uint32_t sw0, int RP, int Gw, int w, int acol, uint32_t code,
                                                   uint32_t item, int l, uint32_t c1, uint32_t c2r, uint32_t s32,
                                                   uint32_t xm, uint32_t xi, uint32_t TK, uint32_t sT, int S1,
                                                   bool active, int Wc = 0) {
    constexpr int CB = NPL == 2 ? 2 : 3;  // bits per packed cell
    using Pack = typename std::conditional<NPL == 2, uint32_t, uint64_t>::type;
    constexpr uint32_t kCellPos = 0x8473u;
    constexpr uint64_t kNbrPos = 0x95847362b8a74130ull;
    constexpr uint32_t kRow = 0xFAA550u;  // 2-bit row offset + 1 of position k: 0 0 1 1 1 1 2 2 2 2 3 3
    constexpr uint32_t kCol = 0x9E4E49u;  // 2-bit column offset + 1 of position k: 1 2 0 1 2 3 0 1 2 3 1 2
    const int j = threadIdx.x & 7;
    // window edge: margin cells, skipped (Wc > 0: full-width rows of Wc columns that wrap)
    const bool ok = active && (Wc != 0 || (acol >= 1 && acol + 2 < 128 * Gw));
    const uint4 rf = philox(item, c1, c2r | (static_cast<uint32_t>(l) << 24), s32);  // overlaps the reads
    const uint32_t PS = static_cast<uint32_t>(Gw) * 16u;
    uint32_t addr[2] = {0u, 0u}, bit[2] = {0u, 0u};
    Pack part = 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int k = j + 8 * t;
        if (ok && k < 12) {
            const int rr = static_cast<int>((kRow >> (2 * k)) & 3u);
            const int cc = static_cast<int>((kCol >> (2 * k)) & 3u);
            const int row = w - 1 + rr;
            int col = acol - 1 + cc;
            if (Wc) col = col < 0 ? col + Wc : (col >= Wc ? col - Wc : col);
            ESCG_CHECK(row >= 0 && col >= 0 && col < 128 * Gw);
            addr[t] = sw0 + 4u * static_cast<uint32_t>(row * RP + (col >> 7) * 4 + (col & 3));
            bit[t] = (static_cast<uint32_t>(col) >> 2) & 31u;
            uint32_t v = 0;
#pragma unroll
            for (int p = 0; p < NPL; ++p) v |= ((lds32(addr[t] + p * PS) >> bit[t]) & 1u) << p;
            part |= static_cast<Pack>(v) << (CB * k);
        }
    }
    Pack cells = part;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        if constexpr (NPL == 2) {
            cells |= __shfl_xor_sync(kFull, cells, o);
        } else {
            const uint32_t lo = __shfl_xor_sync(kFull, static_cast<uint32_t>(cells), o);
            const uint32_t hi = __shfl_xor_sync(kFull, static_cast<uint32_t>(cells >> 32), o);
            cells |= (static_cast<uint64_t>(hi) << 32) | lo;
        }
    }
    if (!ok) return;
    const Pack cells0 = cells;
    const uint32_t rw[4] = {rf.x, rf.y, rf.z, rf.w};
    constexpr Pack M = (static_cast<Pack>(1) << CB) - 1;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t cb = (code >> (4 * a)) & 15u;
        const uint32_t ps = (kCellPos >> (4 * (cb & 3u))) & 15u, pn = static_cast<uint32_t>(kNbrPos >> (4 * cb)) & 15u;
        const uint32_t s = static_cast<uint32_t>(cells >> (CB * ps)) & M, n = static_cast<uint32_t>(cells >> (CB * pn)) & M;
        const bool und = (code >> (16 + a)) & 1u;
        const uint32_t x = TK | (rw[a] & ~TK);
        const bool mig = !und || x < xm, rep = und && x >= xi;
        const bool inter = !mig && !rep && s != 0u && n != 0u && s != n;
        const uint32_t t1 = lds32_if(inter, sT + 4u * (s * S1 + n), 0u);
        const uint32_t t2 = lds32_if(inter, sT + 4u * (n * S1 + s), 0u);
        const bool kn = inter && x < t1, ks = inter && !(x < t1) && x < t2;
        const bool r1 = rep && n == 0u, r2 = rep && n != 0u && s == 0u;
        const uint32_t ns = mig ? n : (ks ? 0u : (r2 ? n : s));
        const uint32_t nn = mig ? s : (kn ? 0u : (r1 ? s : n));
        cells = (cells & ~((M << (CB * ps)) | (M << (CB * pn)))) | (static_cast<Pack>(ns) << (CB * ps)) |
                (static_cast<Pack>(nn) << (CB * pn));
    }
    const Pack delta = cells ^ cells0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int k = j + 8 * t;
        if (k < 12) {
#pragma unroll
            for (int p = 0; p < NPL; ++p)
                if ((delta >> (CB * k + p)) & 1u)
                    asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(addr[t] + p * PS), "r"(1u << bit[t]) : "memory");
        }
    }
}

}  // namespace
}  // namespace escgd

namespace escgd {
namespace {

// SLICED3 draws (oracle/escg_oracle.c slice3_mask is the definition): the undecided
// mask U_a of an item's attempt a — bit l set iff tile l's action word has its K top bits all one,
// i.i.d. with probability 2^-K — drawn by inversion from one word instead of as the AND of K words.
// sT (shared, 64 words): T[1..32] then S[0..31]; gT (global): the whole orc_slice3_table, whose
// conditional-run rows C[m][g] serve only masks with two or more undecided tiles.
__device__ __forceinline__ uint32_t word_of(const uint4 w, int a) { return a == 0 ? w.x : (a == 1 ? w.y : (a == 2 ? w.z : w.w)); }

// ---- TMA bulk copies of plane rows (cp.async.bulk + mbarrier) ----------------------------------
__device__ __forceinline__ void tma_mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}
__device__ __forceinline__ void tma_expect_tx(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_wait(uint32_t mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "TWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra TWAIT_%=;\n\t}" ::"r"(mbar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

// A mask with at least two undecided tiles, the first at G (probability ~ 5e-4 per attempt at K = 10).
__device__ __noinline__ uint32_t slice3_multi(int G, int a, uint32_t item, uint32_t c1, uint32_t c2s, uint32_t s32,
                                              const uint32_t* sT, const uint32_t* gT) {
    uint32_t U = 1u << G;
    const int m = 31 - G;
    const uint32_t* Cm = gT + 64 + 32 * (m - 1) + 1;
    const uint32_t u = word_of(philox(item, c1, c2s | (5u << 24), s32), a);
    int g = 0;
    while (g < m - 1 && u < Cm[g]) ++g;
    int pos = G + 1 + g;
    U |= 1u << pos;
    ++pos;
    for (uint32_t k = 6; pos < 32; ++k) {
        const uint32_t w = word_of(philox(item, c1, c2s | (k << 24), s32), a);
        const int r = 32 - pos;
        int h = 0;
        while (h < r && w < sT[h]) ++h;
        if (h == r) break;
        pos += h;
        U |= 1u << pos;
        ++pos;
    }
    return U;
}

// The four attempts' undecided masks of an item: SLICE draw 4 gives u_0..u_3.  u < T[32] (32 decided
// tiles) costs one comparison; otherwise the first undecided tile is the run G found by binary search
// and u < S[G] makes it the only one — one converged pass per undecided attempt of the lane.
__device__ __forceinline__ void slice3_masks(uint32_t item, uint32_t c1, uint32_t c2s, uint32_t s32, const uint32_t* sT,
                                             const uint32_t* gT, uint32_t (&U)[4]) {
    const uint4 v = philox(item, c1, c2s | (4u << 24), s32);
    const uint32_t u[4] = {v.x, v.y, v.z, v.w};
    const uint32_t t32 = sT[31];
    uint32_t need = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        U[a] = 0u;
        need |= (u[a] >= t32 ? 1u : 0u) << a;
    }
    while (need) {
        const int a = __ffs(need) - 1;
        need &= need - 1u;
        const uint32_t w = a == 0 ? u[0] : (a == 1 ? u[1] : (a == 2 ? u[2] : u[3]));
        int lo = 0, hi = 31;  // G = #{g in 1..32 : w < T[g]} (<= 31 here)
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (w < sT[mid - 1])
                lo = mid;
            else
                hi = mid - 1;
        }
        const uint32_t m = w < sT[32 + lo] ? 1u << lo : slice3_multi(lo, a, item, c1, c2s, s32, sT, gT);
#pragma unroll
        for (int b = 0; b < 4; ++b) U[b] = a == b ? m : U[b];
    }
}

}  // namespace
}  // namespace escgd
