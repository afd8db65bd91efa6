// slice.cu — bit-sliced block kernel (draw format SLICED).
//
// The block kernel's overlapped-tile schedule with the lattice held as NPL bit planes: word q of
// group g of a row holds the species-code bit of columns 128g + 4b + q in bit b.  In a colour phase
// the same-colour tiles of one tile row sit 4 columns apart, so the 32 tiles whose anchor (top-left)
// cell lies in one 128-column group occupy bit b = tile of every word of that group: one thread
// ("item") updates all 32 of them with 32-bit logic.
//
//   footprint  rows w-1 .. w+2 (w = anchor row) x columns anchor-1 .. anchor+2 without corners:
//              12 words per plane, each one of the group's 4 quad words or a one-bit funnel shift
//              of it with the neighbouring group's word (lanes of a tile row hold consecutive groups:
//              warp shuffles, no shared-memory traffic).
//   attempt    the 16 (cell, direction) choices of a tile select one of 12 exchanges inside the
//              footprint; each tile selects at most one, so the 12 masked XOR deltas are computed
//              from the same words and applied together (engine.hpp:118-122, migration).
//   actions    K bit planes hold the top K bits of every action word.  With K <= the number of
//              leading one bits of X_mig, a word with any zero among them is a certain migration;
//              a tile with an undecided attempt (all K bits one: every non-migration is among them)
//              leaves the bit-parallel pass and its lane replays its four attempts afterwards with
//              the exact rule (crs.cuh rule_exact) on shared memory, atomically (neighbouring lanes
//              share the boundary words).  Tiles are disjoint, so the order is immaterial.
//
// oracle/escg_oracle.c orc_crs_run (fmt = 2 | K << 8) is the sequential definition; the kernel is
// bit-exact against it.  Windows are 128-column-group aligned with 64-column side margins (block
// boundaries sit at 64 mod 128); rows carry the usual 12k-row margins.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "crs.cuh"
#include "launch.h"
#include "record.cuh"
#include "slice_common.cuh"

namespace escgd {
namespace {

// Footprint word at column offset DX (-1..2) of a row from the group's quad words: column
// anchor + DX = 4b + t with t = XR + DX, i.e. quad t & 3 at bit b + (t >> 2).  The neighbouring
// groups' copies sit D lanes away (D = lanes per item).
template <int XR, int DX, int D>
__device__ __forceinline__ uint32_t fetch(const uint32_t (&q4)[4]) {
    constexpr int t = XR + DX, q = t & 3, s = t < 0 ? -1 : (t >> 2);
    if constexpr (s == 0) {
        return q4[q];
    } else if constexpr (s < 0) {  // bit b-1: this group's quad 3 shifted up, bit 0 from the left group
        const uint32_t l = __shfl_up_sync(kFull, q4[3], D);
        return __funnelshift_l(l, q4[3], 1);
    } else {  // bit b+1: shifted down, bit 31 from the right group
        const uint32_t r = __shfl_down_sync(kFull, q4[q], D);
        return __funnelshift_r(q4[q], r, 1);
    }
}

// Inverse of fetch: write the footprint word back into the group's quad word (the bit that belongs
// to the neighbouring group is taken over by that group's lane from its own copy).
template <int XR, int DX, int D>
__device__ __forceinline__ void put(uint32_t (&q4)[4], uint32_t f) {
    constexpr int t = XR + DX, q = t & 3, s = t < 0 ? -1 : (t >> 2);
    if constexpr (s == 0) {
        q4[q] = f;
    } else if constexpr (s < 0) {
        const uint32_t r = __shfl_down_sync(kFull, f, D);
        q4[3] = __funnelshift_r(f, r, 1);
    } else {
        const uint32_t l = __shfl_up_sync(kFull, f, D);
        q4[q] = __funnelshift_l(l, f, 1);
    }
}

struct SliceCtx {
    uint32_t* sw;      // window planes [Wh][RP] (row: [plane][group][quad])
    uint32_t sw0;      // its shared-memory address
    int RP, Gw, RW;    // row pitch (words), groups per window row, tile rows per warp (32 / Gw)
    int tr, gw;        // this lane's tile row within the warp and group within the window row
    int gs0, GL, Hg;   // first window group (global), groups per lattice row, lattice rows
    int wy0;           // global row of window row 0
    bool bigy;         // window taller than the lattice (true modulo)
    uint32_t s32;
    uint32_t xm, xi, TK;  // X_mig, X_int, the undecided action prefix (K leading ones)
    uint32_t sT;          // exact interaction thresholds (shared-memory address, (S+1)^2 words)
    int S1;
    uint4* q;             // deferred-tile queue of the phase: (w | acol << 16, code, item)
    unsigned* qn;         // its fill count
    unsigned qcap;        // its capacity (<= kSliceQueue; smaller in tests of the overflow path)
    const uint32_t* T3;   // SLICED3 thresholds T, S in shared memory, null: SLICED (K action words)
    const uint32_t* T3g;  // the whole SLICED3 table (global)
    int Wh;               // window rows (checked builds)
};

// Out-of-line copy for the in-place overflow path inside the (per-residue) phase bodies.
template <int NPL>
__device__ __noinline__ void slice_replay_ool(uint32_t sw0, int RP, int Gw, int w, int acol, uint32_t code,
                                              uint32_t item, int l, uint32_t c1, uint32_t c2r, uint32_t s32,
                                              uint32_t xm, uint32_t xi, uint32_t TK, uint32_t sT, int S1) {
    slice_replay<NPL>(sw0, RP, Gw, w, acol, code, item, l, c1, c2r, s32, xm, xi, TK, sT, S1);
}

// One colour phase: tile rows i_lo .. i_lo + nrows - 1 (anchor window row 4i + yr), every window
// group, anchor column residue XR.  LPI lanes per item: with 2 (NPL = 2) the pair splits the draws
// (attempts {0,1} / {2,3}: two choice draws and K/2 action draws each, exchanged by shuffles) and the
// planes (lane h updates plane h), so a phase has twice the warps with half the latency each.
template <int NPL, int K, int XR, int LPI>
__device__ __forceinline__ void slice_phase(const SliceCtx& C, int oy, int yr, int i_lo, int nrows, uint32_t c1,
                                            uint32_t c2s, uint32_t c2r, int qd) {
    static_assert(LPI == 1 || (LPI == 2 && NPL == 2 && K % 2 == 0), "lane split: two planes, even K");
    constexpr int NP = NPL / LPI;  // planes per lane
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5, lane = threadIdx.x & 31;
    const int h = LPI == 2 ? (lane & 1) : 0, pbase = lane & ~(LPI - 1);
    const int Hh = C.Hg >> 1;
#pragma unroll 1
    for (int base = warp * C.RW; base < nrows; base += nwarps * C.RW) {  // uniform per warp
        const int ir = base + C.tr;
        const bool valid = C.tr < C.RW && ir < nrows;
        const int w = 4 * (i_lo + ir) + yr;
        int gy = C.wy0 + w;
        gy = C.bigy ? gy % C.Hg : (gy >= C.Hg ? gy - C.Hg : gy);
        int j = (gy + oy) >> 1;
        j = j >= Hh ? j - Hh : j;
        int g = C.gs0 + C.gw;
        g = g >= C.GL ? g - C.GL : g;
        const uint32_t item = static_cast<uint32_t>(j) * static_cast<uint32_t>(C.GL) + static_cast<uint32_t>(g);

        // action planes (draws 4 .. 4+K-1, attempt a = word / K): undecided = all K leading bits one
        // choice planes (draws 0..3): cell row, cell column, direction bits
        uint32_t U[4], Y[4], X[4], D0[4], D1[4];
        if constexpr (LPI == 1) {
            if (C.T3 != nullptr) {
                slice3_masks(item, c1, c2s, C.s32, C.T3, C.T3g, U);
            } else {
#pragma unroll
                for (int a = 0; a < 4; ++a) U[a] = ~0u;
#pragma unroll
                for (int jj = 0; jj < K; ++jj) {
                    const uint4 v = philox(item, c1, c2s | (static_cast<uint32_t>(4 + jj) << 24), C.s32);
                    const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) U[(4 * jj + c) / K] &= vw[c];
                }
            }
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const uint4 v = philox(item, c1, c2s | (static_cast<uint32_t>(a) << 24), C.s32);
                Y[a] = v.x;
                X[a] = v.y;
                D0[a] = v.z;
                D1[a] = v.w;
            }
        } else {
            // lane h: attempts 2h, 2h+1 (action words [2hK, 2hK + 2K) = draws 4 + hK/2 .. 4 + hK/2 + K/2 - 1)
            uint32_t Ul[2] = {~0u, ~0u};
            uint32_t U3[4];
            if (C.T3 != nullptr) {
                slice3_masks(item, c1, c2s, C.s32, C.T3, C.T3g, U3);  // both lanes of the pair (same masks)
            } else {
#pragma unroll
                for (int t = 0; t < K / 2; ++t) {
                    const uint32_t jj = 4u + static_cast<uint32_t>(h * (K / 2) + t);
                    const uint4 v = philox(item, c1, c2s | (jj << 24), C.s32);
                    const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int c = 0; c < 4; ++c) Ul[(4 * t + c) / K] &= vw[c];
                }
            }
            const uint4 v0 = philox(item, c1, c2s | (static_cast<uint32_t>(2 * h) << 24), C.s32);
            const uint4 v1 = philox(item, c1, c2s | (static_cast<uint32_t>(2 * h + 1) << 24), C.s32);
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                const int src = pbase + (a >> 1);
                const uint4 v = (a & 1) ? v1 : v0;
                U[a] = C.T3 != nullptr ? U3[a] : __shfl_sync(kFull, Ul[a & 1], src);
                Y[a] = __shfl_sync(kFull, v.x, src);
                X[a] = __shfl_sync(kFull, v.y, src);
                D0[a] = __shfl_sync(kFull, v.z, src);
                D1[a] = __shfl_sync(kFull, v.w, src);
            }
        }
        const uint32_t Dm = valid ? (U[0] | U[1] | U[2] | U[3]) : 0u;
        const uint32_t act = ~Dm;
        if (base == warp * C.RW) SDIAG(qd, 1);

        // footprint rows w-1 .. w+2 of this group (this lane's planes)
        uint32_t Q[4][NP][4];
        ESCG_CHECK(!valid || (w >= 1 && w + 2 < C.Wh && C.gw < C.Gw));
        uint32_t* rowp = C.sw + (valid ? w - 1 : 0) * C.RP + C.gw * 4 + h * NP * C.Gw * 4;
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                uint4 t = make_uint4(0u, 0u, 0u, 0u);
                if (valid) t = lds128(rowp + rr * C.RP + p * C.Gw * 4);
                Q[rr][p][0] = t.x;
                Q[rr][p][1] = t.y;
                Q[rr][p][2] = t.z;
                Q[rr][p][3] = t.w;
            }
        }
        uint32_t F[4][4][NP];  // [row][column offset + 1][plane]; corners unused
#define ESCG_FET(rr, c)                                                         \
    _Pragma("unroll") for (int p = 0; p < NP; ++p) F[rr][c][p] = fetch<XR, (c)-1, LPI>(Q[rr][p]);
        ESCG_FET(0, 1) ESCG_FET(0, 2)
        ESCG_FET(1, 0) ESCG_FET(1, 1) ESCG_FET(1, 2) ESCG_FET(1, 3)
        ESCG_FET(2, 0) ESCG_FET(2, 1) ESCG_FET(2, 2) ESCG_FET(2, 3)
        ESCG_FET(3, 1) ESCG_FET(3, 2)
#undef ESCG_FET

#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const uint32_t y = Y[a], x = X[a], d0 = D0[a], d1 = D1[a];
            // direction 0 up, 1 down, 2 left, 3 right (params.hpp:81)
            const uint32_t up = act & ~(d1 | d0), dn = act & ~d1 & d0, lf = act & d1 & ~d0, rt = act & d1 & d0;
            const uint32_t ny = ~y, nx = ~x;
            const uint32_t vm = (ny & dn) | (y & up);  // exchange rows w, w+1
            const uint32_t hm = (nx & rt) | (x & lf);  // exchange columns +0, +1
            const uint32_t mV0[2] = {ny & nx & up, ny & x & up};
            const uint32_t mV1[2] = {nx & vm, x & vm};
            const uint32_t mV2[2] = {y & nx & dn, y & x & dn};
            const uint32_t mH[2][3] = {{ny & nx & lf, ny & hm, ny & x & rt}, {y & nx & lf, y & hm, y & x & rt}};
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                uint32_t dV0[2], dV1[2], dV2[2], dH[2][3];
#pragma unroll
                for (int xx = 0; xx < 2; ++xx) {
                    dV0[xx] = (F[0][1 + xx][p] ^ F[1][1 + xx][p]) & mV0[xx];
                    dV1[xx] = (F[1][1 + xx][p] ^ F[2][1 + xx][p]) & mV1[xx];
                    dV2[xx] = (F[2][1 + xx][p] ^ F[3][1 + xx][p]) & mV2[xx];
                }
#pragma unroll
                for (int yy = 0; yy < 2; ++yy)
#pragma unroll
                    for (int e = 0; e < 3; ++e) dH[yy][e] = (F[1 + yy][e][p] ^ F[1 + yy][e + 1][p]) & mH[yy][e];
#pragma unroll
                for (int xx = 0; xx < 2; ++xx) {
                    F[0][1 + xx][p] ^= dV0[xx];
                    F[1][1 + xx][p] ^= dV0[xx] ^ dV1[xx] ^ dH[0][xx] ^ dH[0][xx + 1];
                    F[2][1 + xx][p] ^= dV1[xx] ^ dV2[xx] ^ dH[1][xx] ^ dH[1][xx + 1];
                    F[3][1 + xx][p] ^= dV2[xx];
                }
                F[1][0][p] ^= dH[0][0];
                F[1][3][p] ^= dH[0][2];
                F[2][0][p] ^= dH[1][0];
                F[2][3][p] ^= dH[1][2];
            }
        }

#define ESCG_PUT(rr, c) \
    _Pragma("unroll") for (int p = 0; p < NP; ++p) put<XR, (c)-1, LPI>(Q[rr][p], F[rr][c][p]);
        ESCG_PUT(0, 1) ESCG_PUT(0, 2)
        ESCG_PUT(1, 0) ESCG_PUT(1, 1) ESCG_PUT(1, 2) ESCG_PUT(1, 3)
        ESCG_PUT(2, 0) ESCG_PUT(2, 1) ESCG_PUT(2, 2) ESCG_PUT(2, 3)
        ESCG_PUT(3, 1) ESCG_PUT(3, 2)
#undef ESCG_PUT
        if (base == warp * C.RW) SDIAG(qd, 2);
        if (valid) {
#pragma unroll
            for (int rr = 0; rr < 4; ++rr)
#pragma unroll
                for (int p = 0; p < NP; ++p)
                    sts128(rowp + rr * C.RP + p * C.Gw * 4, make_uint4(Q[rr][p][0], Q[rr][p][1], Q[rr][p][2], Q[rr][p][3]));
        }
        __syncwarp();
        // deferred tiles (rare: ~4 per 1024 tiles at P(migration) 0.999): queued for the phase's
        // replay pass, which spreads them over the CTA (one thread each) after the bulk barrier
        for (uint32_t dm = h == 0 ? Dm : 0u; dm != 0u; dm &= dm - 1u) {
            const int l = __ffs(dm) - 1;
            uint32_t code = 0;
#pragma unroll
            for (int a = 0; a < 4; ++a) {
                code |= (((Y[a] >> l) & 1u) | (((X[a] >> l) & 1u) << 1) | (((D0[a] >> l) & 1u) << 2) |
                         (((D1[a] >> l) & 1u) << 3))
                        << (4 * a);
                code |= ((U[a] >> l) & 1u) << (16 + a);
            }
            const int acol = 128 * C.gw + 4 * l + XR;
            const unsigned slot = atomicAdd(C.qn, 1u);
            if (slot < C.qcap) {
                ESCG_CHECK(slot < kSliceQueue);
                C.q[slot] = make_uint4(static_cast<uint32_t>(w) | (static_cast<uint32_t>(acol) << 16), code, item, 0u);
            } else {  // queue full: replay in place (the tile's footprint is disjoint from every other)
                slice_replay_ool<NPL>(C.sw0, C.RP, C.Gw, w, acol, code, item, l, c1, c2r, C.s32, C.xm, C.xi, C.TK, C.sT,
                                  C.S1);
            }
        }
    }
}

// The phase's replay pass: queued deferred tiles, one per 8-lane group (after the bulk barrier),
// dealt round-robin over the warps.
template <int NPL>
__device__ __forceinline__ void slice_replay_queue(const SliceCtx& C, unsigned n, uint32_t c1, uint32_t c2r,
                                                   int qd = 0) {
    n = n < C.qcap ? n : C.qcap;
    const unsigned nw = blockDim.x >> 5, ng = blockDim.x >> 3;
    const unsigned g0 = ((threadIdx.x & 31) >> 3) * nw + (threadIdx.x >> 5);  // group index, warps first
    for (unsigned base = 0; base < n; base += ng) {  // uniform
        const unsigned i = base + g0;
        const bool act = i < n;
        uint4 e = make_uint4(0u, 0u, 0u, 0u);
        if (act) e = C.q[i];
        const int w = static_cast<int>(e.x & 0xFFFFu), acol = static_cast<int>(e.x >> 16);
        slice_replay_group<NPL>(C.sw0, C.RP, C.Gw, w, acol, e.y, e.z, (acol >> 2) & 31, c1, c2r, C.s32, C.xm, C.xi,
                                C.TK, C.sT, C.S1, act);
        if (i < nw) SDIAG(qd, 7);
    }
}

template <int NPL, int K, int LPI>
__global__ void __launch_bounds__(slice_threads(LPI), slice_min_blocks(LPI)) slice_kernel(BlockArgs a) {
    extern __shared__ __align__(16) uint32_t sw[];
    __shared__ uint32_t sTh[(kMaxSliceSpecies + 1) * (kMaxSliceSpecies + 1)];
    __shared__ uint4 sQ[kSliceQueue];
    __shared__ unsigned sQn[3];
    __shared__ uint32_t sT3[64];
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int r = blockIdx.z, tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    // local rows (the buffer; band engines: halo + band + halo, never wrapped) vs global rows (draws)
    const int Hg = a.H, GL = a.L >> 7, S1 = a.S + 1;
    const int My = margin_rows(a.nmcs);
    const int ry0 = a.row_split[blockIdx.y], ry1 = a.row_split[blockIdx.y + 1];
    const int gs0 = a.col_split[blockIdx.x], gs1 = a.col_split[blockIdx.x + 1];
    const int Gw = gs1 - gs0 + 1, bh = ry1 - ry0, Wh = bh + 2 * My;
    const int RP = row_words(NPL, Gw), per_row = NPL * Gw;
    const int wy0 = a.wrap_rows ? ((ry0 - My) % Hg + Hg) % Hg : ry0 - My;  // bands: halo rows, no wrap
    const bool bigy = Wh > Hg;
    const size_t NW = static_cast<size_t>(Hg) * NPL * GL * 4;
    const uint32_t* src = a.psrc + r * NW;
    uint32_t* dst = a.pdst + r * NW;
    __shared__ uint32_t sCnt[1 << NPL];
    __shared__ int sLast;
    __shared__ __align__(8) unsigned long long sMbar;
    if (tid < (1 << NPL)) sCnt[tid] = 0u;
    if (tid < 3) sQn[tid] = 0u;
    for (int i = tid; i < S1 * S1; i += nt) sTh[i] = a.rule.T[i];
    if (a.T3 != nullptr && tid < 64) sT3[tid] = a.T3[tid];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (a.run.status[r] != kStatusRunning) return;  // uniform per CTA

#ifndef ESCG_SLICE_NO_TMA
    // the window by TMA: one bulk copy per (row, plane) run of Gw groups (two when the run wraps
    // around the row), completion counted in bytes on one mbarrier
    const uint32_t mbar = smem_addr(&sMbar);
    if (tid == 0) {
        tma_mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        tma_expect_tx(mbar, static_cast<uint32_t>(Wh) * NPL * Gw * 16u);
    }
    __syncthreads();
    {
        const int n1 = gs0 + Gw <= GL ? Gw : GL - gs0;  // groups before the row wraps
        const uint32_t sw0 = smem_addr(sw);
        for (int idx = tid; idx < Wh * NPL; idx += nt) {
            const int y = idx / NPL, p = idx - y * NPL;
            int gy = wy0 + y;
            gy = bigy ? gy % Hg : (gy >= Hg ? gy - Hg : gy);
            const uint32_t* srow = src + static_cast<size_t>(gy * NPL + p) * GL * 4;
            const uint32_t d = sw0 + static_cast<uint32_t>((y * RP + p * Gw * 4) * 4);
            tma_g2s(d, srow + gs0 * 4, static_cast<uint32_t>(n1) * 16u, mbar);
            if (n1 < Gw) tma_g2s(d + n1 * 16u, srow, static_cast<uint32_t>(Gw - n1) * 16u, mbar);
        }
    }
    tma_wait(mbar, 0);
#else
    for (int idx = tid; idx < Wh * per_row; idx += nt) {
        const int y = idx / per_row, rem = idx - y * per_row;
        const int p = rem / Gw, gw = rem - p * Gw;
        int gy = wy0 + y;
        gy = bigy ? gy % Hg : (gy >= Hg ? gy - Hg : gy);
        int g = gs0 + gw;
        g = g >= GL ? g - GL : g;
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(src + (static_cast<size_t>(gy * NPL + p) * GL + g) * 4));
        sts128(sw + y * RP + rem * 4, v);
    }
    __syncthreads();
#endif

    if (a.step) {
        SliceCtx C;
        C.sw = sw;
        C.sw0 = smem_addr(sw);
        C.RP = RP;
        C.Gw = Gw;
        C.RW = (32 / LPI) / Gw;
        C.tr = (lane / LPI) / Gw;
        C.gw = lane / LPI - C.tr * Gw;
        C.gs0 = gs0;
        C.GL = GL;
        C.Hg = a.Hg;                   // draws use global rows: local row r is global (row0 + r) mod Hg
        C.wy0 = (a.row0 + wy0) % a.Hg;
        C.bigy = Wh > a.Hg;
        C.s32 = seed32(a.seeds[r]);
        C.xm = a.rule.xm;
        C.xi = a.rule.xi;
        C.TK = ~0u << (32 - K);
        C.sT = smem_addr(sTh);
        C.q = sQ;
        C.qcap = a.qcap > 0 && a.qcap < static_cast<int>(kSliceQueue) ? static_cast<unsigned>(a.qcap) : kSliceQueue;
        C.T3 = a.T3 != nullptr ? sT3 : nullptr;
        C.T3g = a.T3;
        C.Wh = Wh;
        C.S1 = S1;
#pragma unroll 1
        for (int t = 0; t < a.nmcs; ++t) {
            const uint64_t mcs = static_cast<uint64_t>(a.mcs + t);
            const Round rp = round_params(C.s32, mcs);
#pragma unroll 1
            for (int p = 0; p < 4; ++p) {
                const int q = 4 * t + p;  // validity shrinks 3 rows per phase
                const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
                const int yr = (2 * cy - rp.oy) & 3, xr = (2 * cx - rp.ox) & 3;
                // anchor rows w = 4i + yr with footprint rows [w-1, w+2] inside [3q, Wh - 3q)
                const int v = 3 * q + 1 - yr;
                const int i_lo = v <= 0 ? 0 : (v + 3) >> 2;
                const int top = Wh - 3 * q - 3 - yr;
                const int nrows = top < 0 ? 0 : (top >> 2) - i_lo + 1;
                const uint32_t c1 = static_cast<uint32_t>(mcs);
                const uint32_t c2s = ctr2(mcs, kDomSlice, static_cast<uint32_t>(p), 0u);
                const uint32_t c2r = ctr2(mcs, kDomSliceRef, static_cast<uint32_t>(p), 0u);
                // queue counters rotate over three phases: the next phase's counter was last read
                // before this phase's predecessor's barrier, so it can be zeroed now
                C.qn = &sQn[q % 3];
                if (tid == 0) sQn[(q + 1) % 3] = 0u;
                SDIAG(q, 0);
                switch (xr) {
                    case 0: slice_phase<NPL, K, 0, LPI>(C, rp.oy, yr, i_lo, nrows, c1, c2s, c2r, q); break;
                    case 1: slice_phase<NPL, K, 1, LPI>(C, rp.oy, yr, i_lo, nrows, c1, c2s, c2r, q); break;
                    case 2: slice_phase<NPL, K, 2, LPI>(C, rp.oy, yr, i_lo, nrows, c1, c2s, c2r, q); break;
                    default: slice_phase<NPL, K, 3, LPI>(C, rp.oy, yr, i_lo, nrows, c1, c2s, c2r, q); break;
                }
                SDIAG(q, 3);
                __syncthreads();
                SDIAG(q, 4);
                const unsigned nq = sQn[q % 3];
#ifdef ESCG_DIAG_SLICE_NOREPLAY  // diagnostic builds only: skips the replay pass (wrong results)
                if (nq == 0x7fffffffu) {
#else
                if (nq != 0u) {  // uniform
#endif
                    slice_replay_queue<NPL>(C, nq, c1, c2r, q);
                    __syncthreads();
                }
            }
        }
        // block region: rows [My, My + bh), columns [64, 128 Gw - 64): the edge groups own one half
        for (int idx = tid; idx < bh * per_row; idx += nt) {
            const int y = idx / per_row, rem = idx - y * per_row;
            const int p = rem / Gw, gw = rem - p * Gw;
            int g = gs0 + gw;
            g = g >= GL ? g - GL : g;
            const uint4 v = lds128(sw + (My + y) * RP + rem * 4);
            uint32_t* d = dst + (static_cast<size_t>((ry0 + y) * NPL + p) * GL + g) * 4;
            unsigned short* d16 = reinterpret_cast<unsigned short*>(d);
            if (gw == 0) {
                d16[1] = static_cast<unsigned short>(v.x >> 16);
                d16[3] = static_cast<unsigned short>(v.y >> 16);
                d16[5] = static_cast<unsigned short>(v.z >> 16);
                d16[7] = static_cast<unsigned short>(v.w >> 16);
            } else if (gw == Gw - 1) {
                d16[0] = static_cast<unsigned short>(v.x);
                d16[2] = static_cast<unsigned short>(v.y);
                d16[4] = static_cast<unsigned short>(v.z);
                d16[6] = static_cast<unsigned short>(v.w);
            } else {
                __stcg(reinterpret_cast<uint4*>(d), v);
            }
        }
    }

    if (a.count) {
        // species histogram of the block region from the planes (codes 1 .. 2^NPL - 1 by popc)
        uint32_t cnt[1 << NPL];
#pragma unroll
        for (int v = 0; v < (1 << NPL); ++v) cnt[v] = 0u;
        for (int idx = tid; idx < bh * Gw * 4; idx += nt) {
            const int y = idx / (Gw * 4), rem = idx - y * (Gw * 4);
            const int gw = rem >> 2, qd = rem & 3;
            const uint32_t m = gw == 0 ? 0xFFFF0000u : (gw == Gw - 1 ? 0x0000FFFFu : ~0u);
            uint32_t pl[NPL];
#pragma unroll
            for (int p = 0; p < NPL; ++p) pl[p] = sw[(My + y) * RP + (p * Gw + gw) * 4 + qd];
#pragma unroll
            for (int v = 1; v < (1 << NPL); ++v) {
                uint32_t c = m;
#pragma unroll
                for (int p = 0; p < NPL; ++p) c &= ((v >> p) & 1) ? pl[p] : ~pl[p];
                cnt[v] += __popc(c);
            }
        }
#pragma unroll
        for (int v = 1; v < (1 << NPL); ++v) {
            const uint32_t tsum = __reduce_add_sync(kFull, cnt[v]);
            if (lane == 0 && tsum) atomicAdd(&sCnt[v], tsum);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t nz = 0;
            for (int v = 1; v < (1 << NPL); ++v) nz += sCnt[v];
            sCnt[0] = static_cast<uint32_t>(bh) * 128u * static_cast<uint32_t>(Gw - 1) - nz;
            for (int v = 0; v < S1; ++v)
                if (sCnt[v]) atomicAdd(&a.acc[r * S1 + v], static_cast<unsigned long long>(sCnt[v]));
            __threadfence();
            const unsigned int tk = atomicAdd(&a.ticket[r], 1u);
            sLast = tk == static_cast<unsigned int>(a.nby * a.nbx - 1);
        }
        __syncthreads();
        if (sLast && tid == 0) {
            __threadfence();
            uint64_t c64[kMaxSpecies + 1];
            for (int v = 0; v < S1; ++v) c64[v] = atomicExch(&a.acc[r * S1 + v], 0ull);
            a.ticket[r] = 0u;
            // plane buffer holding the recorded lattice, offset by 2 (0/1 name the byte buffers)
            if (a.run.cur) a.run.cur[r] = 2 + (a.step ? a.dst_index : 1 - a.dst_index);
            record_decide(c64, S1, a.mcs + (a.step ? a.nmcs : 0), r, a.run);
        }
    }
}

// u8 lattice → bit planes: one warp per (replica, row, group); lane b holds columns 4b .. 4b+3.
__global__ void to_planes_kernel(const uint8_t* lat, uint32_t* pl, int H, int L, int npl, int nrep) {
    const int GL = L >> 7;
    const int64_t units = static_cast<int64_t>(nrep) * H * GL;
    const int lane = threadIdx.x & 31;
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < units;
         u += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const int64_t rr = u / GL;
        const int g = static_cast<int>(u - rr * GL);
        const uint32_t v = __ldg(reinterpret_cast<const uint32_t*>(lat + rr * L + 128 * g) + lane);
        uint32_t mine = 0u;
        for (int p = 0; p < npl; ++p)
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t wd = __ballot_sync(kFull, (v >> (8 * q + p)) & 1u);
                if (lane == p * 4 + q) mine = wd;
            }
        // rr = replica * H + row: planes [rr][p][g][q]
        if (lane < 4 * npl) pl[(rr * npl + (lane >> 2)) * GL * 4 + g * 4 + (lane & 3)] = mine;
    }
}

// bit planes → u8 lattice (replica r from plane buffer cur[r] - 2, or `buf` when cur is null).
__global__ void from_planes_kernel(const uint32_t* pl0, const uint32_t* pl1, const int32_t* cur, int buf, uint8_t* lat,
                                   int H, int L, int npl, int nrep) {
    const int GL = L >> 7;
    const int64_t units = static_cast<int64_t>(nrep) * H * GL;
    const int lane = threadIdx.x & 31;
    for (int64_t u = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; u < units;
         u += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const int64_t rr = u / GL;
        const int g = static_cast<int>(u - rr * GL);
        const int rep = static_cast<int>(rr / H);
        int b = buf;
        if (cur) {
            if (cur[rep] < 2) continue;  // uniform per warp: the record preceded every step
            b = cur[rep] - 2;
        }
        const uint32_t* pl = b ? pl1 : pl0;
        uint32_t out = 0u;
        for (int p = 0; p < npl; ++p) {
            const uint4 wq = __ldg(reinterpret_cast<const uint4*>(pl + (rr * npl + p) * GL * 4 + g * 4));
            out |= ((wq.x >> lane) & 1u) << p;
            out |= ((wq.y >> lane) & 1u) << (8 + p);
            out |= ((wq.z >> lane) & 1u) << (16 + p);
            out |= ((wq.w >> lane) & 1u) << (24 + p);
        }
        reinterpret_cast<uint32_t*>(lat + rr * L + 128 * g)[lane] = out;
    }
}

int conv_grid(int64_t units) {
    int64_t g = (units * 32 + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : static_cast<int>(g);
}

template <int NPL, int K, int LPI>
cudaError_t slice_launch_t(const BlockArgs& a, int nrep, cudaStream_t s) {
    auto k = slice_kernel<NPL, K, LPI>;
    static std::atomic<int> configured[kMaxDevices];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices || configured[dev].load() < a.smem_bytes) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < kMaxDevices) {
            int c = configured[dev].load();
            while (c < a.smem_bytes && !configured[dev].compare_exchange_weak(c, a.smem_bytes)) {
            }
        }
    }
    static const bool pdl = !(std::getenv("ESCG_PDL") && std::getenv("ESCG_PDL")[0] == '0');
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(a.nbx), static_cast<unsigned>(a.nby), static_cast<unsigned>(nrep));
    cfg.blockDim = dim3(static_cast<unsigned>(slice_threads(LPI)));
    cfg.dynamicSmemBytes = static_cast<size_t>(a.smem_bytes);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, a);
}

template <int NPL, int LPI>
cudaError_t slice_launch_npl(const BlockArgs& a, int nrep, cudaStream_t s) {
    switch (a.K) {
        case 6: return slice_launch_t<NPL, 6, LPI>(a, nrep, s);
        case 8: return slice_launch_t<NPL, 8, LPI>(a, nrep, s);
        case 10: return slice_launch_t<NPL, 10, LPI>(a, nrep, s);
        case 12: return slice_launch_t<NPL, 12, LPI>(a, nrep, s);
        case 14: return slice_launch_t<NPL, 14, LPI>(a, nrep, s);
        case 16: return slice_launch_t<NPL, 16, LPI>(a, nrep, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

int slice_row_words(int npl, int gw) { return row_words(npl, gw); }

// Diagnostic: copy the bit-sliced kernel's clock64 stamps (ESCG_DIAG_SLICE builds; else returns -1).
extern "C" __attribute__((visibility("default"))) int escg_diag_slice(long long* out, int reset) {
#ifdef ESCG_DIAG_SLICE
    if (reset) {
        static long long z[4 * 16 * 8 * 8];
        return cudaMemcpyToSymbol(g_sdiag, z, sizeof(z)) == cudaSuccess ? 0 : -1;
    }
    return cudaMemcpyFromSymbol(out, g_sdiag, sizeof(long long) * 4 * 16 * 8 * 8) == cudaSuccess ? 0 : -1;
#else
    (void)out;
    (void)reset;
    return -1;
#endif
}

cudaError_t launch_slice(const BlockArgs& a, int nrep, cudaStream_t s) {
    if (a.npl == 2 && a.lpi == 2) return slice_launch_npl<2, 2>(a, nrep, s);
    if (a.npl == 2) return slice_launch_npl<2, 1>(a, nrep, s);
    if (a.npl == 3) return slice_launch_npl<3, 1>(a, nrep, s);
    return cudaErrorInvalidValue;
}

int slice_kernel_registers(int npl, int lpi) {
    cudaFuncAttributes fa{};
    const void* f = npl == 3   ? reinterpret_cast<const void*>(slice_kernel<3, 10, 1>)
                    : lpi == 2 ? reinterpret_cast<const void*>(slice_kernel<2, 10, 2>)
                               : reinterpret_cast<const void*>(slice_kernel<2, 10, 1>);
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return 255;
    return fa.numRegs;
}

cudaError_t launch_to_planes(const uint8_t* lat, uint32_t* pl, int H, int L, int npl, int nrep, cudaStream_t s) {
    to_planes_kernel<<<conv_grid(static_cast<int64_t>(nrep) * H * (L >> 7)), 256, 0, s>>>(lat, pl, H, L, npl, nrep);
    return cudaGetLastError();
}

cudaError_t launch_from_planes(const uint32_t* pl0, const uint32_t* pl1, const int32_t* cur, int buf, uint8_t* lat,
                               int H, int L, int npl, int nrep, cudaStream_t s) {
    from_planes_kernel<<<conv_grid(static_cast<int64_t>(nrep) * H * (L >> 7)), 256, 0, s>>>(pl0, pl1, cur, buf, lat,
                                                                                              H, L, npl, nrep);
    return cudaGetLastError();
}

}  // namespace escgd
