// kernels.cu — sm_100a kernels of the ESCG engine.
//
//   tile_kernel   whole lattice resident in one CTA's shared memory (ghost frame for the periodic
//                 wrap), persistent over many MCS, fused density records + on-device stop
//                 predicates; one CTA per replica (ensembles, L <= ~460).
//   block_kernel  one MCS per launch over an L2/HBM-resident lattice: each CTA loads its block
//                 plus a 12-cell margin, runs the 4 colour phases on shrinking valid regions
//                 (overlapped tiling — counter-based draws make the redundant margin work
//                 bit-identical across CTAs), and writes its block to the other buffer.
//   init/count/replay/convert helpers.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "crs.cuh"
#include "launch.h"
#include "record.cuh"

namespace escgd {

#ifdef ESCG_DIAG_TIMING
// diagnostic builds only: per-CTA %globaltimer stamps of the block kernel's sections, and per-warp
// stamps at the end of each phase's work (before the phase barrier) of CTA 0..7
__device__ unsigned long long g_diag_t[4096 * 16];
__device__ unsigned long long g_diag_w[8 * 32 * 16];
// per launch slot (launch index % 256): first CTA start, first CTA past griddepcontrol.wait, last CTA end
__device__ unsigned long long g_diag_span[256 * 3];
#endif

namespace {

#ifdef ESCG_DIAG_TIMING
__device__ __forceinline__ void diag_stamp(int slot) {
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
        if (cta < 4096) g_diag_t[cta * 16 + slot] = t;
    }
}
#define DIAG_STAMP(s) diag_stamp(s)
#else
#define DIAG_STAMP(s)
#endif

// n / d for 0 <= n < 2^22, 1 <= d < 2^22 via the float reciprocal (exact after one fix-up).
__device__ __forceinline__ int udiv_small(int n, int d) {
    int q = __float2int_rz(__int2float_rn(n) * __frcp_rn(__int2float_rn(d)));
    int r = n - q * d;
    if (r < 0) {
        --q;
    } else if (r >= d) {
        ++q;
    }
    return q;
}

// Sum of the four bytes of a (each byte <= 255).
__device__ __forceinline__ uint32_t byte_sum(uint32_t a) {
    const uint32_t h = (a & 0x00FF00FFu) + ((a >> 8) & 0x00FF00FFu);
    return (h & 0xFFFFu) + (h >> 16);
}

// Species histogram of a rows x cols region of a byte array (generic pointer, any space) with the
// given pitch, added into sCnt[0, S1) (shared; the caller zeroes sCnt[0, kCntSlots) and syncs
// before, and syncs after).  S1 <= 8: every thread walks 4-byte words of the flattened region and
// accumulates, per byte lane, the bit-subset indicators b0, b1, b2, b0b1, b0b2, b1b2, b0b1b2 of the
// cell codes (plain adds, flushed every 255 words); the exact per-code counts follow by inclusion-
// exclusion.  Otherwise one shared atomic per cell.
__device__ void block_count(const uint8_t* base, int rows, int cols, int pitch, int S1, uint32_t* sCnt) {
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31;
    if (S1 <= 8 && (cols & 3) == 0 && (pitch & 3) == 0 && ((reinterpret_cast<uintptr_t>(base) & 3) == 0)) {
        const int wpr = cols >> 2, n = rows * wpr;
        const int nb = S1 <= 2 ? 1 : (S1 <= 4 ? 2 : 3);  // code bits
        uint32_t s[7] = {0, 0, 0, 0, 0, 0, 0};           // s0 s1 s2 s01 s02 s12 s012
        uint32_t a[7] = {0, 0, 0, 0, 0, 0, 0};
        int y = udiv_small(tid, wpr), x = tid - y * wpr;
        const int dy = udiv_small(nt, wpr), dx = nt - dy * wpr;
        int pend = 0;
        for (int k = tid; k < n; k += nt) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(base + static_cast<size_t>(y) * pitch + 4 * x);
            const uint32_t b0 = w & 0x01010101u, b1 = (w >> 1) & 0x01010101u, b2 = (w >> 2) & 0x01010101u;
            a[0] += b0;
            if (nb >= 2) {
                a[1] += b1;
                a[3] += b0 & b1;
            }
            if (nb >= 3) {
                a[2] += b2;
                a[4] += b0 & b2;
                a[5] += b1 & b2;
                a[6] += b0 & b1 & b2;
            }
            if (++pend == 255) {
#pragma unroll
                for (int i = 0; i < 7; ++i) {
                    s[i] += byte_sum(a[i]);
                    a[i] = 0;
                }
                pend = 0;
            }
            x += dx;
            y += dy;
            if (x >= wpr) {
                x -= wpr;
                ++y;
            }
        }
#pragma unroll
        for (int i = 0; i < 7; ++i) {
            const uint32_t t = __reduce_add_sync(0xffffffffu, s[i] + byte_sum(a[i]));
            if (lane == 0 && t) atomicAdd(&sCnt[kMaxSpecies + 1 - 7 + i], t);
        }
        __syncthreads();
        if (tid == 0) {
            uint32_t* z = sCnt + kMaxSpecies + 1 - 7;
            const uint32_t N = static_cast<uint32_t>(rows) * static_cast<uint32_t>(cols);
            const uint32_t s0 = z[0], s1 = z[1], s2 = z[2], s01 = z[3], s02 = z[4], s12 = z[5], s012 = z[6];
            const uint32_t c[8] = {N - s0 - s1 - s2 + s01 + s02 + s12 - s012, s0 - s01 - s02 + s012,
                                   s1 - s01 - s12 + s012, s01 - s012, s2 - s02 - s12 + s012, s02 - s012,
                                   s12 - s012, s012};
            for (int v = 0; v < S1; ++v) sCnt[v] += c[v];
            for (int i = 0; i < 7; ++i) z[i] = 0;
        }
    } else {
        for (int y = tid >> 5; y < rows; y += nt >> 5)
            for (int x = lane; x < cols; x += 32) atomicAdd(&sCnt[base[static_cast<size_t>(y) * pitch + x]], 1u);
    }
}

// ---------------------------------------------------------------------------------------------
// Tile kernel (whole lattice in shared memory)
// ---------------------------------------------------------------------------------------------

struct TileSmem {
    int lat_bytes, T_off, snap_off, cnt_off, flag_off, total;
};

__host__ __device__ inline TileSmem tile_layout(int H, int L, int S, int P) {
    TileSmem t;
    const int S1 = S + 1;
    t.lat_bytes = align16((H + 3) * P);
    t.T_off = t.lat_bytes;
    t.snap_off = t.T_off + align16(S1 * S1 * 8);  // coarse pair table (crs.cuh fill_pair_thresholds)
    t.cnt_off = t.snap_off + align16(3 * (L + 3) + 3 * H);
    t.flag_off = t.cnt_off + align16((kMaxSpecies + 1) * 4);
    t.total = t.flag_off + 16;
    return t;
}

__device__ __forceinline__ int wrap(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// Ghost frame of the periodic tile kernel: rows {-2,-1,H} x cols [-2,L] and cols {-2,-1,L} x
// rows [0,H).  Band b (0..5) enumerates them; snap holds the value each ghost had after refresh.
// After a phase, a ghost that changed carries the phase's write of its physical cell (at most one
// representation of a physical cell lies in an active footprint per phase).
template <bool FOLD>
__device__ void ghost_pass(uint8_t* lat, uint8_t* snap, int H, int L, int P) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int b = warp; b < 6; b += nw) {
        const bool rowband = b < 3;
        const int len = rowband ? L + 3 : H;
        const int fixed = (b % 3) == 0 ? -2 : ((b % 3) == 1 ? -1 : (rowband ? H : L));
        uint8_t* sn = snap + (rowband ? b * (L + 3) : 3 * (L + 3) + (b - 3) * H);
        for (int k = lane; k < len; k += 32) {
            const int gy = rowband ? fixed : k;
            const int gx = rowband ? k - 2 : fixed;
            const int ga = (gy + kTileR0) * P + gx + kTileC0;
            const int pa = (wrap(gy, H) + kTileR0) * P + wrap(gx, L) + kTileC0;
            if (FOLD) {
                const uint8_t g = lat[ga];
                if (g != sn[k]) lat[pa] = g;
            } else {
                const uint8_t v = lat[pa];
                lat[ga] = v;
                sn[k] = v;
            }
        }
    }
}

template <int ARITY, bool BF = false>
__device__ __forceinline__ PhaseCtx phase_ctx(const RuleArgs& rule, int narrow, uint64_t mcs, int p, uint32_t s32) {
    constexpr int LB = Bits<ARITY>::LB;
    PhaseCtx C;
    (void)LB;
    C.fast = narrow ? rule.fast : 0u;
    C.xm = rule.xm;
    C.xi = rule.xi;
    C.bf = BF ? 1u : 0u;  // compile-time: the other rule_wide form folds away
    C.c1 = static_cast<uint32_t>(mcs);
    C.c2 = ctr2(mcs, kDomStep, static_cast<uint32_t>(p), 0u);
    C.c3 = s32;
    return C;
}

// Fill the per-CTA static shared state of the attempt paths (before the first phase barrier).
template <int ARITY>
__device__ __forceinline__ void attempt_setup(const RuleArgs& rule, uint32_t sT, int S1, int P) {
    build_offset_table<ARITY>(P);
    if (threadIdx.x == 0) {
        sSlow.xm = rule.xm;
        sSlow.xi = rule.xi;
        sSlow.sT = sT;
        sSlow.S1 = S1;
        sSlow.gT = rule.T;
    }
}

// Tile-kernel lattice modes: periodic with H, L ≡ 0 (mod 4); reflecting; periodic with seams.
constexpr int kModePeriodic = 0, kModeReflect = 1, kModeSeam = 2;

// One MCS of the seam mode: 4, 6 or 9 phases of single WIDE tiles.
template <int ARITY, bool BF>
__device__ void tile_round_seam(uint32_t lat0, uint8_t* lat, uint8_t* snap,
                                const RuleArgs& rule, int H, int L, int P, int S1, uint32_t s32, uint64_t mcs) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const SeamAxis ay(H), ax(L);
    const RoundG rg = round_params_g(s32, mcs, ay.nc, ax.nc);
    const int np = ay.nc * ax.nc;
#pragma unroll 1
    for (int p = 0; p < np; ++p) {
        const int v = rg.colour(p), cy = v / ax.nc, cx = v - cy * ax.nc;
        const PhaseCtx C = phase_ctx<ARITY, BF>(rule, 0, mcs, p, s32);
        const uint32_t c2 = C.c2;
        const int nty = ay.count(cy), ntx = ax.count(cx), cnt = nty * ntx;
        for (int k = tid; k < cnt; k += nt) {
            const int i = k / ntx, j = k - i * ntx;
            const int ty = ay.tile(cy, i), tx = ax.tile(cx, j);
            const uint32_t tile = static_cast<uint32_t>(ty) * static_cast<uint32_t>(ax.T) + static_cast<uint32_t>(tx);
            const uint32_t base =
                lat0 + static_cast<uint32_t>((2 * ty - rg.oy + kTileR0) * P + kTileC0 + 2 * tx - rg.ox);
            tile_seam<ARITY>(philox(tile, C.c1, c2, s32), base, tile, 2 * ty + 1 >= H, 2 * tx + 1 >= L, C);
        }
        __syncthreads();
        ghost_pass<true>(lat, snap, H, L, P);
        __syncthreads();
        ghost_pass<false>(lat, snap, H, L, P);
        __syncthreads();
    }
}

// One MCS of the tile kernel (whole lattice in shared memory at lat0, ghost frame when periodic).
template <int ARITY, int MODE, bool BF>
__device__ void tile_round(uint32_t lat0, uint8_t* lat, uint8_t* snap,
                           const RuleArgs& rule, int narrow, int H, int L, int P, int S1, uint32_t s32,
                           uint64_t mcs) {
    if (MODE == kModeSeam) {
        tile_round_seam<ARITY, BF>(lat0, lat, snap, rule, H, L, P, S1, s32, mcs);
        return;
    }
    constexpr bool REFLECT = MODE == kModeReflect;
    const int tid = threadIdx.x, nt = blockDim.x;
    const Round rp = round_params(s32, mcs);
    const int Ty = REFLECT ? (H + rp.oy + 1) >> 1 : H >> 1;
    const int Tx = REFLECT ? (L + rp.ox + 1) >> 1 : L >> 1;
#pragma unroll 1
    for (int p = 0; p < 4; ++p) {
        const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
        const PhaseCtx C = phase_ctx<ARITY, BF>(rule, narrow, mcs, p, s32);
        const uint32_t c2 = C.c2;
        const int nty = (Ty - cy + 1) >> 1;
        const int ntx = (Tx - cx + 1) >> 1;  // tiles of this colour per tile row
        // items: pairs of same-colour tiles (tx, tx+2) of a row (one NARROW draw, or two WIDE
        // draws, per pair; the last item of a row may hold one tile), single tiles when reflecting
        const int nxi = REFLECT ? ntx : ((ntx + 1) >> 1);
        const int cnt = nty * nxi;
        if (tid < cnt) {
            int i = udiv_small(tid, nxi), j = tid - udiv_small(tid, nxi) * nxi;
            const int di = udiv_small(nt, nxi), dj = nt - udiv_small(nt, nxi) * nxi;
            for (int k = tid; k < cnt; k += nt) {
                const int ty = cy + 2 * i;
                if (REFLECT) {
                    const int tx = cx + 2 * j;
                    const uint32_t tile = static_cast<uint32_t>(ty) * static_cast<uint32_t>(Tx) + static_cast<uint32_t>(tx);
                    const uint4 w = philox(tile, C.c1, c2, s32);
                    tile_reflect<ARITY>(w, lat0, 2 * ty - rp.oy, 2 * tx - rp.ox, kTileR0, kTileC0, P, H, L, tile, C);
                } else {
                    const int tx0 = cx + 4 * j;
                    const uint32_t row = lat0 + static_cast<uint32_t>((2 * ty - rp.oy + kTileR0) * P + kTileC0 - rp.ox);
                    const uint32_t t0 = static_cast<uint32_t>(ty) * static_cast<uint32_t>(Tx) + tx0;
                    const uint32_t b0 = row + 2 * tx0;
                    const bool two = 2 * j + 1 < ntx;
                    if (narrow) {  // L % 8 == 0: every pair is complete
                        const uint4 w = philox(static_cast<uint32_t>(ty) * static_cast<uint32_t>(Tx >> 2) + j, C.c1, c2, s32);
                        pair_narrow<ARITY>(w, b0, t0, b0 + 4, t0 + 2, C);
                    } else if (two) {
                        const uint4 wA = philox(t0, C.c1, c2, s32), wB = philox(t0 + 2, C.c1, c2, s32);
                        pair_wide<ARITY>(wA, b0, t0, wB, b0 + 4, t0 + 2, C);
                    } else {
                        tile_wide<ARITY>(philox(t0, C.c1, c2, s32), b0, t0, C);
                    }
                }
                j += dj;
                i += di;
                if (j >= nxi) {
                    j -= nxi;
                    ++i;
                }
            }
        }
        __syncthreads();
        if (!REFLECT) {
            ghost_pass<true>(lat, snap, H, L, P);
            __syncthreads();
            ghost_pass<false>(lat, snap, H, L, P);
            __syncthreads();
        }
    }
}

// Copy an H x L byte lattice between global (row pitch L) and shared (pitch P, origin R0/C0).
template <bool TO_SMEM>
__device__ void tile_copy(uint8_t* lat, uint8_t* glat, int H, int L, int P) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if ((L & 3) == 0) {
        const int wpr = L >> 2;
        for (int y = warp; y < H; y += nw) {
            uint32_t* g = reinterpret_cast<uint32_t*>(glat + static_cast<size_t>(y) * L);
            uint32_t* sm = reinterpret_cast<uint32_t*>(lat + (y + kTileR0) * P + kTileC0);
            for (int c = lane; c < wpr; c += 32) {
                if (TO_SMEM)
                    sm[c] = g[c];
                else
                    g[c] = sm[c];
            }
        }
    } else {
        for (int y = warp; y < H; y += nw) {
            uint8_t* g = glat + static_cast<size_t>(y) * L;
            uint8_t* sm = lat + (y + kTileR0) * P + kTileC0;
            for (int c = lane; c < L; c += 32) {
                if (TO_SMEM)
                    sm[c] = g[c];
                else
                    g[c] = sm[c];
            }
        }
    }
}

// Launch shapes of the tile kernel (measured on B200 ensembles): lattices whose shared memory allows
// two CTAs per SM use <= 384 threads at <= 80 registers (L=200 x 296 replicas +3%, L=100 +2% over
// 512 x 64); larger ones, one CTA per SM anyway, use <= 512 threads at up to 128 registers (L=400 +5%).
template <int ARITY, int MODE, bool BF, bool ONE_PER_SM>
__global__ void __launch_bounds__(ONE_PER_SM ? kTileThreadsOne : kTileThreadsTwo, ONE_PER_SM ? 1 : 2)
    tile_kernel(TileArgs a) {
    constexpr bool REFLECT = MODE == kModeReflect;
    extern __shared__ __align__(128) uint8_t smem[];
    const int H = a.H, L = a.L, P = a.P, S1 = a.S + 1;
    const TileSmem lay = tile_layout(H, L, a.S, P);
    uint8_t* lat = smem;
    uint32_t* sT = reinterpret_cast<uint32_t*>(smem + lay.T_off);
    uint8_t* snap = smem + lay.snap_off;
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(smem + lay.cnt_off);
    int* sFlag = reinterpret_cast<int*>(smem + lay.flag_off);
    const int tid = threadIdx.x, nt = blockDim.x;
    const int r = blockIdx.x;
    uint8_t* glat = a.lat + static_cast<size_t>(r) * H * L;
    const uint32_t s32 = seed32(a.seeds[r]);

    fill_pair_thresholds<ARITY>(reinterpret_cast<uint2*>(sT), a.rule.T, S1);
    attempt_setup<ARITY>(a.rule, smem_addr(sT), S1, P);
    tile_copy<true>(lat, glat, H, L, P);
    __syncthreads();
    if (!REFLECT) {
        ghost_pass<false>(lat, snap, H, L, P);
        __syncthreads();
    }
    const uint32_t lat0 = smem_addr(lat);
    int64_t mcs = a.run.mcs[r];
    int status = a.run.status[r];
    for (;;) {
        int64_t adv;
        if (a.record) {
            for (int v = tid; v <= kMaxSpecies; v += nt) sCnt[v] = 0;
            __syncthreads();
            block_count(lat + kTileR0 * P + kTileC0, H, L, P, S1, sCnt);
            __syncthreads();
            if (tid == 0) {
                uint64_t c64[kMaxSpecies + 1];
                for (int v = 0; v < S1; ++v) c64[v] = sCnt[v];
                *sFlag = record_decide(c64, S1, mcs, r, a.run);
            }
            __syncthreads();
            status = *sFlag;
            if (status != kStatusRunning) break;
            adv = a.run.interval < a.run.mcs_limit - mcs ? a.run.interval : a.run.mcs_limit - mcs;
        } else {
            if (mcs >= a.run.mcs_limit) break;
            adv = a.run.mcs_limit - mcs;
        }
        for (int64_t k = 0; k < adv; ++k, ++mcs)
            tile_round<ARITY, MODE, BF>(lat0, lat, snap, a.rule, a.narrow, H, L, P, S1, s32,
                                       static_cast<uint64_t>(mcs));
    }
    tile_copy<false>(lat, glat, H, L, P);
    if (tid == 0 && !a.record) a.run.mcs[r] = mcs;
}

// ---------------------------------------------------------------------------------------------
// Block kernel (overlapped tiling, one MCS per launch, periodic lattices with H, L ≡ 0 mod 4)
// ---------------------------------------------------------------------------------------------

// v mod n for v >= 0: one conditional subtract when the window is at most twice the lattice.
__device__ __forceinline__ int wrap_down(int v, int n, bool big) {
    if (big) return v % n;
    return v >= n ? v - n : v;
}

// Per-launch constants of the phase loop (by value: keeps the kernel-parameter block out of local
// memory).
struct BlockGeom {
    int P, H, L, nmcs;
    int Hg, row0;      // global rows / global row of local row 0 (draws use global tile ids)
    int64_t mcs;
    uint32_t scratch;  // smem address of a dummy 4-row box (edge items with one invalid tile)
};

// Per-(MCS, phase) geometry of one block-kernel launch, identical for every thread of a CTA: built
// once per launch by warp 0 (lane q = phase q, overlapping the PDL wait) instead of by every warp in
// every phase (the round draw, the valid-region bounds, the pair columns and rows per round).
struct PhaseGeom {
    int j0, nj, u0, nu;     // first active tile row, active rows, first pair column, pairs per row
    int i0, imin, imax, R;  // WIDE first tile column, valid tile-column range, rows per round
    uint32_t c1, c2;        // draw counter words of the phase (MCS low, STEP c2)
    int cx, oyox;           // colour column parity, tiling origin oy | ox << 1
};
__shared__ PhaseGeom sPh[4 * kMaxBlockMcs];

template <bool NARROW>
__device__ __noinline__ void build_phase_table(const BlockGeom g, int Wh, int Ww, uint32_t s32) {
    const int q = threadIdx.x;  // warp 0
    if (q >= 4 * g.nmcs) return;
    const int t = q >> 2, p = q & 3;
    const uint64_t mcs = static_cast<uint64_t>(g.mcs + t);
    const Round rp = round_params(s32, mcs);
    const int ex = margin_cols(g.nmcs) - margin_rows(g.nmcs);  // extra loaded columns
    const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
    // footprint rows [2j-oy-1, 2j-oy+2] within [3q, Wh-3q); cols within [ex+3q, Ww-ex-3q)
    const int lo = 3 * q, hiR = Wh - 3 * q, loC = ex + 3 * q, hiC = Ww - ex - 3 * q;
    const int jmin = (lo + rp.oy + 2) >> 1, jmax = (hiR - 3 + rp.oy) >> 1;
    const int imin = (loC + rp.ox + 2) >> 1, imax = (hiC - 3 + rp.ox) >> 1;
    PhaseGeom G;
    G.j0 = jmin + ((jmin ^ cy) & 1);
    G.nj = jmax >= G.j0 ? ((jmax - G.j0) >> 1) + 1 : 0;
    // items: pairs of same-colour tiles (i, i+2).  NARROW pairs are the global draw pairs (window
    // column 0 is 8-aligned); WIDE pairs are local.  A tile outside the valid region runs on the
    // scratch box (same instruction stream for every lane, results discarded).
    G.i0 = imin + ((imin ^ cx) & 1);  // first valid tile column of this colour
    if (NARROW) {
        G.u0 = (imin - cx + 1) >> 2;
        const int u1 = imax >= cx ? (imax - cx) >> 2 : -1;
        G.nu = u1 >= G.u0 ? u1 - G.u0 + 1 : 0;
    } else {
        const int ni = imax >= G.i0 ? ((imax - G.i0) >> 1) + 1 : 0;
        G.u0 = 0;
        G.nu = (ni + 1) >> 1;
    }
    G.imin = imin;
    G.imax = imax;
    G.R = G.nu > 0 ? udiv_small(static_cast<int>(blockDim.x), G.nu) : 0;
    G.c1 = static_cast<uint32_t>(mcs);
    G.c2 = ctr2(mcs, kDomStep, static_cast<uint32_t>(p), 0u);
    G.cx = cx;
    G.oyox = rp.oy | (rp.ox << 1);
    sPh[q] = G;
}

template <int ARITY, bool NARROW, bool BF>
__device__ __forceinline__ void block_phases(const BlockGeom g, const RuleArgs rule, uint32_t win0, int Wh, int Ww,
                                             int wy0, int wx0, uint32_t s32) {
    const int tid = threadIdx.x, nt = blockDim.x, P = g.P;
    const int Ty = g.Hg >> 1, Tx = g.L >> 1, TQ = g.L >> 3;
    // global tile index of window tile 0 (even; ib % 4 == 0 if NARROW)
    const int jb = ((g.row0 + wy0) % g.Hg) >> 1, ib = wx0 >> 1;
    const int ex = margin_cols(g.nmcs) - margin_rows(g.nmcs);  // extra loaded columns
    const bool big = Wh > g.Hg || Ww > g.L;  // window wraps more than once: use a true modulo
#pragma unroll 1
    for (int t = 0; t < g.nmcs; ++t) {
        const uint64_t mcs = static_cast<uint64_t>(g.mcs + t);
        const Round rp = round_params(s32, mcs);
#pragma unroll 1
        for (int p = 0; p < 4; ++p) {
            const int q = 4 * t + p;  // global phase of this launch: validity shrinks 3 cells per phase
            const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
            const PhaseCtx C = phase_ctx<ARITY, BF>(rule, NARROW, mcs, p, s32);
            const uint32_t c2 = C.c2;
            // footprint rows [2j-oy-1, 2j-oy+2] within [3q, Wh-3q); cols within [ex+3q, Ww-ex-3q)
            const int lo = 3 * q, hiR = Wh - 3 * q, loC = ex + 3 * q, hiC = Ww - ex - 3 * q;
            const int jmin = (lo + rp.oy + 2) >> 1, jmax = (hiR - 3 + rp.oy) >> 1;
            const int imin = (loC + rp.ox + 2) >> 1, imax = (hiC - 3 + rp.ox) >> 1;
            const int j0 = jmin + ((jmin ^ cy) & 1);
            const int nj = jmax >= j0 ? ((jmax - j0) >> 1) + 1 : 0;
            // items: pairs of same-colour tiles (i, i+2).  NARROW pairs are the global draw pairs
            // (window column 0 is 8-aligned); WIDE pairs are local.  A tile outside the valid region
            // runs on the scratch box (same instruction stream for every lane, results discarded).
            const int i0 = imin + ((imin ^ cx) & 1);  // first valid tile column of this colour
            int u0, nu;
            if (NARROW) {
                u0 = (imin - cx + 1) >> 2;
                const int u1 = imax >= cx ? (imax - cx) >> 2 : -1;
                nu = u1 >= u0 ? u1 - u0 + 1 : 0;
            } else {
                const int ni = imax >= i0 ? ((imax - i0) >> 1) + 1 : 0;
                u0 = 0;
                nu = (ni + 1) >> 1;
            }
            // Thread -> items: a fixed item column b (pair b of every active tile row) and rows
            // a0, a0 + R, a0 + 2R, ... with R = floor(threads / nu): the column geometry, the
            // half-warp chain order and the scratch redirection are per-phase constants, and a row
            // step is a few adds.  (Items are the same as any other enumeration; order within a
            // phase is immaterial.)
            if (nu > 0 && nj > 0) {
                const int R = udiv_small(nt, nu);
                const int a0 = udiv_small(tid, nu), b = tid - a0 * nu;
                if (a0 < R && a0 < nj) {
                    // upper half-warp runs its pair's second tile as chain 1 (bank split, tile_dual)
#ifdef ESCG_DIAG_NO_SWAP
                    const bool sw = false;
#else
                    const bool sw = (tid & 16) != 0;
#endif
                    int ia1, ia2;  // window tile columns of chain 1 / chain 2
                    uint32_t tc1, tc2;  // global tile-column part of the tile ids
                    uint32_t ctrcol = 0;  // NARROW: pair column of the draw counter
                    if (NARROW) {
                        const int u = u0 + b;
                        const int qq = big ? ((ib >> 2) + u) % TQ : wrap_down((ib >> 2) + u, TQ, false);
                        const int ia = cx + 4 * u;
                        ctrcol = static_cast<uint32_t>(qq);
                        ia1 = sw ? ia + 2 : ia;
                        ia2 = sw ? ia : ia + 2;
                        tc1 = static_cast<uint32_t>(4 * qq + cx + (sw ? 2 : 0));
                        tc2 = static_cast<uint32_t>(4 * qq + cx + (sw ? 0 : 2));
                    } else {
                        const int ia = i0 + 4 * b;
                        const uint32_t tA = static_cast<uint32_t>(big ? (ib + ia) % Tx : wrap_down(ib + ia, Tx, false));
                        const uint32_t tB =
                            static_cast<uint32_t>(big ? (ib + ia + 2) % Tx : wrap_down(ib + ia + 2, Tx, false));
                        ia1 = sw ? ia + 2 : ia;
                        ia2 = sw ? ia : ia + 2;
                        tc1 = sw ? tB : tA;
                        tc2 = sw ? tA : tB;
                    }
                    const bool ok1 = ia1 >= imin && ia1 <= imax, ok2 = ia2 >= imin && ia2 <= imax;
                    const uint32_t scr1 = sw ? g.scratch + 8 : g.scratch, scr2 = sw ? g.scratch : g.scratch + 8;
                    int j = j0 + 2 * a0;
                    int ty = big ? (jb + j) % Ty : wrap_down(jb + j, Ty, false);
                    const int dTy = big ? (2 * R) % Ty : 2 * R;  // window rows < Ty: 2R < Ty
                    uint32_t rowbase = win0 + static_cast<uint32_t>((2 * j - rp.oy) * P - rp.ox);
                    const uint32_t dRow = static_cast<uint32_t>(4 * R * P);
                    auto draw1 = [&](int ty_) {
                        return NARROW ? philox(static_cast<uint32_t>(ty_) * static_cast<uint32_t>(TQ) + ctrcol, C.c1, c2, s32)
                                      : philox(static_cast<uint32_t>(ty_) * static_cast<uint32_t>(Tx) + tc1, C.c1, c2, s32);
                    };
                    uint4 w = draw1(ty);
                    for (int a = a0; a < nj; a += R) {
                        int nty = ty + dTy;
                        nty = nty >= Ty ? nty - Ty : nty;
                        uint4 nw = make_uint4(0, 0, 0, 0);
                        if (a + R < nj) nw = draw1(nty);
                        const uint32_t trow = static_cast<uint32_t>(ty) * static_cast<uint32_t>(Tx);
                        const uint32_t base1 = ok1 ? rowbase + 2 * ia1 : scr1;
                        const uint32_t base2 = ok2 ? rowbase + 2 * ia2 : scr2;
                        if (NARROW) {
                            // pair draw: words (x, y) belong to the pair's first tile, (z, w) to its second
                            const uint32_t p0 = sw ? w.z : w.x, p1 = sw ? w.w : w.y;
                            const uint32_t q0 = sw ? w.x : w.z, q1 = sw ? w.y : w.w;
                            const uint32_t b1[4] = {p0 & 0xFFFFu, p0 >> 16, p1 & 0xFFFFu, p1 >> 16};
                            const uint32_t b2[4] = {q0 & 0xFFFFu, q0 >> 16, q1 & 0xFFFFu, q1 >> 16};
                            tile_dual_ordered<ARITY, true>(b1, base1, trow + tc1, b2, base2, trow + tc2, C);
                        } else {
                            const uint4 w2 = philox(trow + tc2, C.c1, c2, s32);
                            const uint32_t b1[4] = {w.x, w.y, w.z, w.w};
                            const uint32_t b2[4] = {w2.x, w2.y, w2.z, w2.w};
                            tile_dual_ordered<ARITY, false>(b1, base1, trow + tc1, b2, base2, trow + tc2, C);
                        }
                        ty = nty;
                        rowbase += dRow;
                        w = nw;
                    }
                }
            }
#ifdef ESCG_DIAG_TIMING
            {
                const int cta = blockIdx.x + gridDim.x * blockIdx.y;
                if (cta < 8 && (threadIdx.x & 31) == 0 && q < 16) {
                    unsigned long long tw;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw));
                    g_diag_w[(cta * 32 + (threadIdx.x >> 5)) * 16 + q] = tw;
                }
            }
#endif
#ifndef ESCG_DIAG_NO_PHASE_SYNC
            __syncthreads();
#endif
            if (t == 0) DIAG_STAMP(3 + p);
        }
    }
}

template <int ARITY, bool NARROW, bool BF>
__device__ __forceinline__ void block_phases_tab(const BlockGeom g, const RuleArgs rule, uint32_t win0, int Wh, int Ww,
                                             int wy0, int wx0, uint32_t s32) {
    const int tid = threadIdx.x, nt = blockDim.x, P = g.P;
    const int Ty = g.Hg >> 1, Tx = g.L >> 1, TQ = g.L >> 3;
    // global tile index of window tile 0 (even; ib % 4 == 0 if NARROW)
    const int jb = ((g.row0 + wy0) % g.Hg) >> 1, ib = wx0 >> 1;
    const bool big = Wh > g.Hg || Ww > g.L;  // window wraps more than once: use a true modulo
    const int ex = margin_cols(g.nmcs) - margin_rows(g.nmcs);  // extra loaded columns
    Round rp = {0, 0, 0u};
#pragma unroll 1
    for (int q = 0; q < 4 * g.nmcs; ++q) {
        const int t = q >> 2;
        // phase geometry: TAB reads the per-launch table (few items per thread: the per-phase work
        // dominates); otherwise it is recomputed in uniform registers (many items per thread: no
        // extra vector-register pressure on the item loop)
        int j0, nj, u0, nu, i0, imin, imax, R, cx, oy, ox;
        uint32_t c1, c2p;
        if (true) {
            const PhaseGeom& G = sPh[q];
            j0 = G.j0;
            nj = G.nj;
            u0 = G.u0;
            nu = G.nu;
            i0 = G.i0;
            imin = G.imin;
            imax = G.imax;
            R = G.R;
            cx = G.cx;
            oy = G.oyox & 1;
            ox = G.oyox >> 1;
            c1 = G.c1;
            c2p = G.c2;
        } else {
            const int p = q & 3;
            const uint64_t mcs = static_cast<uint64_t>(g.mcs + t);
            if (p == 0) rp = round_params(s32, mcs);
            const int cy = rp.colour(p) >> 1;
            cx = rp.colour(p) & 1;
            oy = rp.oy;
            ox = rp.ox;
            // footprint rows [2j-oy-1, 2j-oy+2] within [3q, Wh-3q); cols within [ex+3q, Ww-ex-3q)
            const int lo = 3 * q, hiR = Wh - 3 * q, loC = ex + 3 * q, hiC = Ww - ex - 3 * q;
            const int jmin = (lo + oy + 2) >> 1, jmax = (hiR - 3 + oy) >> 1;
            imin = (loC + ox + 2) >> 1;
            imax = (hiC - 3 + ox) >> 1;
            j0 = jmin + ((jmin ^ cy) & 1);
            nj = jmax >= j0 ? ((jmax - j0) >> 1) + 1 : 0;
            i0 = imin + ((imin ^ cx) & 1);
            if (NARROW) {
                u0 = (imin - cx + 1) >> 2;
                const int u1 = imax >= cx ? (imax - cx) >> 2 : -1;
                nu = u1 >= u0 ? u1 - u0 + 1 : 0;
            } else {
                const int ni = imax >= i0 ? ((imax - i0) >> 1) + 1 : 0;
                u0 = 0;
                nu = (ni + 1) >> 1;
            }
            R = nu > 0 ? udiv_small(nt, nu) : 0;
            c1 = static_cast<uint32_t>(mcs);
            c2p = ctr2(mcs, kDomStep, static_cast<uint32_t>(p), 0u);
        }
        PhaseCtx C;
        C.fast = NARROW ? rule.fast : 0u;
        C.xm = rule.xm;
        C.xi = rule.xi;
        C.bf = BF ? 1u : 0u;
        C.c1 = c1;
        C.c2 = c2p;
        C.c3 = s32;
        const uint32_t c2 = C.c2;
        // Thread -> items: a fixed item column b (pair b of every active tile row) and rows
        // a0, a0 + R, a0 + 2R, ... with R = floor(threads / nu): the column geometry, the
        // half-warp chain order and the scratch redirection are per-phase constants, and a row
        // step is a few adds.  (Items are the same as any other enumeration; order within a
        // phase is immaterial.)
        if (nu > 0 && nj > 0) {
            const int a0 = udiv_small(tid, nu), b = tid - a0 * nu;
            if (a0 < R && a0 < nj) {
                // upper half-warp runs its pair's second tile as chain 1 (bank split, tile_dual)
#ifdef ESCG_DIAG_NO_SWAP
                const bool sw = false;
#else
                const bool sw = (tid & 16) != 0;
#endif
                int ia1, ia2;  // window tile columns of chain 1 / chain 2
                uint32_t tc1, tc2;  // global tile-column part of the tile ids
                uint32_t ctrcol = 0;  // NARROW: pair column of the draw counter
                if (NARROW) {
                    const int u = u0 + b;
                    const int qq = big ? ((ib >> 2) + u) % TQ : wrap_down((ib >> 2) + u, TQ, false);
                    const int ia = cx + 4 * u;
                    ctrcol = static_cast<uint32_t>(qq);
                    ia1 = sw ? ia + 2 : ia;
                    ia2 = sw ? ia : ia + 2;
                    tc1 = static_cast<uint32_t>(4 * qq + cx + (sw ? 2 : 0));
                    tc2 = static_cast<uint32_t>(4 * qq + cx + (sw ? 0 : 2));
                } else {
                    const int ia = i0 + 4 * b;
                    const uint32_t tA = static_cast<uint32_t>(big ? (ib + ia) % Tx : wrap_down(ib + ia, Tx, false));
                    const uint32_t tB =
                        static_cast<uint32_t>(big ? (ib + ia + 2) % Tx : wrap_down(ib + ia + 2, Tx, false));
                    ia1 = sw ? ia + 2 : ia;
                    ia2 = sw ? ia : ia + 2;
                    tc1 = sw ? tB : tA;
                    tc2 = sw ? tA : tB;
                }
                const bool ok1 = ia1 >= imin && ia1 <= imax, ok2 = ia2 >= imin && ia2 <= imax;
                const uint32_t scr1 = sw ? g.scratch + 8 : g.scratch, scr2 = sw ? g.scratch : g.scratch + 8;
                int j = j0 + 2 * a0;
                int ty = big ? (jb + j) % Ty : wrap_down(jb + j, Ty, false);
                const int dTy = big ? (2 * R) % Ty : 2 * R;  // window rows < Ty: 2R < Ty
                uint32_t rowbase = win0 + static_cast<uint32_t>((2 * j - oy) * P - ox);
                const uint32_t dRow = static_cast<uint32_t>(4 * R * P);
                auto draw1 = [&](int ty_) {
                    return NARROW ? philox(static_cast<uint32_t>(ty_) * static_cast<uint32_t>(TQ) + ctrcol, C.c1, c2, s32)
                                  : philox(static_cast<uint32_t>(ty_) * static_cast<uint32_t>(Tx) + tc1, C.c1, c2, s32);
                };
                uint4 w = draw1(ty);
                for (int a = a0; a < nj; a += R) {
                    int nty = ty + dTy;
                    nty = nty >= Ty ? nty - Ty : nty;
                    uint4 nw = make_uint4(0, 0, 0, 0);
                    if (a + R < nj) nw = draw1(nty);
                    const uint32_t trow = static_cast<uint32_t>(ty) * static_cast<uint32_t>(Tx);
                    const uint32_t base1 = ok1 ? rowbase + 2 * ia1 : scr1;
                    const uint32_t base2 = ok2 ? rowbase + 2 * ia2 : scr2;
                    if (NARROW) {
                        // pair draw: words (x, y) belong to the pair's first tile, (z, w) to its second
                        const uint32_t p0 = sw ? w.z : w.x, p1 = sw ? w.w : w.y;
                        const uint32_t q0 = sw ? w.x : w.z, q1 = sw ? w.y : w.w;
                        const uint32_t b1[4] = {p0 & 0xFFFFu, p0 >> 16, p1 & 0xFFFFu, p1 >> 16};
                        const uint32_t b2[4] = {q0 & 0xFFFFu, q0 >> 16, q1 & 0xFFFFu, q1 >> 16};
                        tile_dual_ordered<ARITY, true>(b1, base1, trow + tc1, b2, base2, trow + tc2, C);
                    } else {
                        const uint4 w2 = philox(trow + tc2, C.c1, c2, s32);
                        const uint32_t b1[4] = {w.x, w.y, w.z, w.w};
                        const uint32_t b2[4] = {w2.x, w2.y, w2.z, w2.w};
                        tile_dual_ordered<ARITY, false>(b1, base1, trow + tc1, b2, base2, trow + tc2, C);
                    }
                    ty = nty;
                    rowbase += dRow;
                    w = nw;
                }
            }
        }
#ifdef ESCG_DIAG_TIMING
        {
            const int cta = blockIdx.x + gridDim.x * blockIdx.y;
            if (cta < 8 && (threadIdx.x & 31) == 0 && q < 16) {
                unsigned long long tw;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw));
                g_diag_w[(cta * 32 + (threadIdx.x >> 5)) * 16 + q] = tw;
            }
        }
#endif
#ifndef ESCG_DIAG_NO_PHASE_SYNC
        __syncthreads();
#endif
        if (t == 0) DIAG_STAMP(3 + (q & 3));
    }
}

template <int ARITY, bool NARROW, bool BF, bool TAB>
__device__ __forceinline__ void block_phases_any(const BlockGeom g, const RuleArgs rule, uint32_t win0, int Wh, int Ww,
                                                 int wy0, int wx0, uint32_t s32) {
    if constexpr (TAB)
        block_phases_tab<ARITY, NARROW, BF>(g, rule, win0, Wh, Ww, wy0, wx0, s32);
    else
        block_phases<ARITY, NARROW, BF>(g, rule, win0, Wh, Ww, wy0, wx0, s32);
}

// ---- TMA bulk copies (cp.async.bulk, Hopper+/Blackwell) ----------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx_arrive(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred done;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
        "@!done bra WAIT_%=;\n\t}" ::"r"(mbar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}

// Window load (global → shared) with periodic wrap.  TMA path: one bulk copy per row segment
// (two when the row wraps), completion tracked by one mbarrier; fallback: vector loads.
template <int VEC>
__device__ __forceinline__ void load_window(uint8_t* win, const uint8_t* src, int H, int L, int P, int Wh, int Ww,
                                            int wy0, int wx0) {
    using V = typename std::conditional<VEC == 16, uint4, uint32_t>::type;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int cpr = Ww / VEC;
    const bool bigy = Wh > H, bigx = Ww > L;
    for (int wr = warp; wr < Wh; wr += nw) {
        int gy = wy0 + wr;
        gy = bigy ? gy % H : (gy >= H ? gy - H : gy);
        const uint8_t* srow = src + static_cast<size_t>(gy) * L;
        V* drow = reinterpret_cast<V*>(win + wr * P);
        for (int c = lane; c < cpr; c += 32) {
            int gx = wx0 + VEC * c;
            gx = bigx ? gx % L : (gx >= L ? gx - L : gx);
            V v;
            if (VEC == 16) {
                const uint4 t = __ldcg(reinterpret_cast<const uint4*>(srow + gx));
                v = *reinterpret_cast<const V*>(&t);
            } else {
                const unsigned int t = __ldcg(reinterpret_cast<const unsigned int*>(srow + gx));
                v = *reinterpret_cast<const V*>(&t);
            }
            drow[c] = v;
        }
    }
}

__device__ __forceinline__ void load_window_tma(uint8_t* win, const uint8_t* src, int H, int L, int P, int Wh, int Ww,
                                                int wy0, int wx0, uint32_t mbar) {
    // caller: mbarrier initialised and expect_tx(Wh*Ww) armed by thread 0 before a __syncthreads
    const uint32_t w0 = smem_addr(win);
    for (int wr = threadIdx.x; wr < Wh; wr += blockDim.x) {
        int gy = wy0 + wr;
        gy = gy >= H ? gy - H : gy;
        const uint8_t* srow = src + static_cast<size_t>(gy) * L;
        const int n1 = (wx0 + Ww <= L) ? Ww : L - wx0;
        bulk_g2s(w0 + wr * P, srow + wx0, static_cast<uint32_t>(n1), mbar);
        if (n1 < Ww) bulk_g2s(w0 + wr * P + n1, srow, static_cast<uint32_t>(Ww - n1), mbar);
    }
}

template <int VEC>
__device__ __forceinline__ void store_block(uint8_t* dst, const uint8_t* win, int L, int P, int bh, int bw, int ry0,
                                            int rx0, int My, int Mx) {
    using V = typename std::conditional<VEC == 16, uint4, uint32_t>::type;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int cpr = bw / VEC;
    for (int y = warp; y < bh; y += nw) {
        const V* srow = reinterpret_cast<const V*>(win + (My + y) * P + Mx);
        uint8_t* drow = dst + static_cast<size_t>(ry0 + y) * L + rx0;
        for (int c = lane; c < cpr; c += 32) {
            if (VEC == 16)
                __stcg(reinterpret_cast<uint4*>(drow) + c, *reinterpret_cast<const uint4*>(srow + c));
            else
                __stcg(reinterpret_cast<unsigned int*>(drow) + c, *reinterpret_cast<const unsigned int*>(srow + c));
        }
    }
}

// ---- reflecting lattices (flux = false) on the block kernel --------------------------------------
// Windows are clipped at the lattice edge (no wrap); a clipped side needs no validity margin.  Tiles
// follow the reflect tiling of orc_crs_run (T = (n + o + 1) / 2 per axis, partial edge tiles), WIDE
// draws.  Pairs whose footprints stay inside the lattice take the fast dual path; pairs touching the
// mirror go through tile_reflect (explicit coordinates, reflected neighbours, skipped cells).
template <int ARITY, bool BF>
__device__ void block_phases_reflect(const RuleArgs& rule, uint32_t win0, int H, int L, int P, int nmcs,
                                     int64_t mcs0, int Wh, int Ww, int wy0, int wx0, int ex, uint32_t s32) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const bool top = wy0 == 0, bot = wy0 + Wh == H, lft = wx0 == 0, rgt = wx0 + Ww == L;
    const int jb = wy0 >> 1, ib = wx0 >> 1;  // window origin is even: tile parity = global parity
#pragma unroll 1
    for (int t = 0; t < nmcs; ++t) {
        const uint64_t mcs = static_cast<uint64_t>(mcs0 + t);
        const Round rp = round_params(s32, mcs);
        const int Ty = (H + rp.oy + 1) >> 1, Tx = (L + rp.ox + 1) >> 1;
#pragma unroll 1
        for (int p = 0; p < 4; ++p) {
            const int q = 4 * t + p;
            const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
            const PhaseCtx C = phase_ctx<ARITY, BF>(rule, 0, mcs, p, s32);
            const int jlo = top ? 0 : ((3 * q + rp.oy + 2) >> 1);
            const int jhi = bot ? (Ty - 1 - jb) : ((Wh - 3 * q - 3 + rp.oy) >> 1);
            const int ilo = lft ? 0 : ((ex + 3 * q + rp.ox + 2) >> 1);
            const int ihi = rgt ? (Tx - 1 - ib) : ((Ww - ex - 3 * q - 3 + rp.ox) >> 1);
            const int j0 = jlo + ((jlo ^ cy) & 1), i0 = ilo + ((ilo ^ cx) & 1);
            const int nj = jhi >= j0 ? ((jhi - j0) >> 1) + 1 : 0;
            const int ni = ihi >= i0 ? ((ihi - i0) >> 1) + 1 : 0;
            const int nu = (ni + 1) >> 1;  // pairs (i, i + 2) of a row
            const int cnt = nj * nu;
            for (int k = tid; k < cnt; k += nt) {
                const int a_ = udiv_small(k, nu), b_ = k - a_ * nu;
                const int j = j0 + 2 * a_, iA = i0 + 4 * b_, iB = iA + 2;
                const bool hasB = iB <= ihi;
                const int tg = j + jb, sA = iA + ib, sB = iB + ib;
                const int y0 = 2 * tg - rp.oy, xA = 2 * sA - rp.ox, xB = 2 * sB - rp.ox;
                const uint32_t tA = static_cast<uint32_t>(tg) * static_cast<uint32_t>(Tx) + static_cast<uint32_t>(sA);
                const uint32_t tB = tA + 2;
                const uint4 wA = philox(tA, C.c1, C.c2, s32);
                const uint4 wB = hasB ? philox(tB, C.c1, C.c2, s32) : make_uint4(0, 0, 0, 0);
                const bool inR = y0 >= 1 && y0 + 2 <= H - 1;
                const bool inA = inR && xA >= 1 && xA + 2 <= L - 1, inB = inR && xB >= 1 && xB + 2 <= L - 1;
                const uint32_t rowb = win0 + static_cast<uint32_t>((y0 - wy0) * P - wx0);
                if (inA && hasB && inB) {
                    const uint32_t b1[4] = {wA.x, wA.y, wA.z, wA.w};
                    const uint32_t b2[4] = {wB.x, wB.y, wB.z, wB.w};
                    tile_dual_ordered<ARITY, false>(b1, rowb + xA, tA, b2, rowb + xB, tB, C);
                } else {
                    tile_reflect<ARITY>(wA, win0, y0, xA, -wy0, -wx0, P, H, L, tA, C);
                    if (hasB) tile_reflect<ARITY>(wB, win0, y0, xB, -wy0, -wx0, P, H, L, tB, C);
                }
            }
            __syncthreads();
        }
    }
}

// Plain (non-wrapping) copies of a rows x cols region between global memory (pitch L) and the window
// (pitch P): 4-byte words when everything is 4-aligned, else bytes.
template <bool TO_WIN>
__device__ void copy_region(uint8_t* win, int P, uint8_t* glob, int L, int rows, int cols) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool w4 = ((L | P | cols) & 3) == 0 && ((reinterpret_cast<uintptr_t>(glob) | reinterpret_cast<uintptr_t>(win)) & 3) == 0;
    for (int y = warp; y < rows; y += nw) {
        uint8_t* g = glob + static_cast<size_t>(y) * L;
        uint8_t* w = win + y * P;
        if (w4) {
            for (int c = lane; c < (cols >> 2); c += 32) {
                if (TO_WIN)
                    reinterpret_cast<uint32_t*>(w)[c] = __ldcg(reinterpret_cast<const unsigned int*>(g) + c);
                else
                    __stcg(reinterpret_cast<unsigned int*>(g) + c, reinterpret_cast<const uint32_t*>(w)[c]);
            }
        } else {
            for (int c = lane; c < cols; c += 32) {
                if (TO_WIN)
                    w[c] = g[c];
                else
                    g[c] = w[c];
            }
        }
    }
}

// ---- periodic lattices with seams (L or H not divisible by 4) on the block kernel ---------------
// Per MCS the window's tiles are listed per axis in shared memory (global tile, local start row /
// column, 1 or 2 cells, colour), built from the seam tiling of SeamAxis/round_params_g for that MCS'
// origin; each of the 4, 6 or 9 phases then runs the (row list of colour cy) x (column list of
// colour cx) tiles whose footprints lie in the phase's valid region, as single WIDE tiles.  The
// validity region shrinks 3 cells per phase, so the margin is 3 * phases * MCS per launch.
struct SeamEntry {
    int t, start, nc, pad;
};

__device__ void seam_axis_lists(SeamEntry* lists, int* counts, int W, int w0, int n, int o, const SeamAxis ax) {
    // one warp per axis; lists[c * cap + i], cap = W / 2 + 2
    const int lane = threadIdx.x & 31, cap = W / 2 + 2;
    int cnt[3] = {0, 0, 0};
    for (int base = 0; base < W; base += 32) {
        const int y = base + lane;
        bool start = false;
        int t = 0, nc = 0, col = 0;
        if (y < W) {
            const int g = (w0 + y) % n;
            const int pos = (g + o) % n;
            start = (pos & 1) == 0;
            t = pos >> 1;
            nc = pos + 1 < n ? 2 : 1;
            col = t == ax.seam ? 2 : (t & 1);
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const unsigned m = __ballot_sync(0xffffffffu, start && col == c);
            if (start && col == c) {
                const int idx = cnt[c] + __popc(m & ((1u << lane) - 1u));
                if (idx < cap) lists[c * cap + idx] = SeamEntry{t, y, nc, 0};
            }
            cnt[c] += __popc(m);
        }
    }
    if (lane == 0)
        for (int c = 0; c < 3; ++c) counts[c] = min(cnt[c], cap);
}

template <int ARITY, bool BF>
__device__ void block_phases_seam(const RuleArgs& rule, uint32_t win0, int H, int L, int P, int nmcs, int64_t mcs0,
                                  int Wh, int Ww, int wy0, int wx0, uint32_t s32, SeamEntry* rows, SeamEntry* cols,
                                  int* counts) {
    const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5;
    const SeamAxis ay(H), ax(L);
    const int np = ay.nc * ax.nc, capy = Wh / 2 + 2, capx = Ww / 2 + 2;
#pragma unroll 1
    for (int t = 0; t < nmcs; ++t) {
        const uint64_t mcs = static_cast<uint64_t>(mcs0 + t);
        const RoundG rg = round_params_g(s32, mcs, ay.nc, ax.nc);
        if (warp == 0) seam_axis_lists(rows, counts, Wh, wy0, H, rg.oy, ay);
        if (warp == 1) seam_axis_lists(cols, counts + 3, Ww, wx0, L, rg.ox, ax);
        __syncthreads();
#pragma unroll 1
        for (int p = 0; p < np; ++p) {
            const int q = np * t + p;
            const int v = rg.colour(p), cy = v / ax.nc, cx = v - cy * ax.nc;
            const PhaseCtx C = phase_ctx<ARITY, BF>(rule, 0, mcs, p, s32);
            const int ny = counts[cy], nx = counts[3 + cx], cnt = ny * nx;
            const int lo = 3 * q, hiY = Wh - 3 * q, hiX = Ww - 3 * q;
            for (int k = tid; k < cnt; k += nt) {
                const int i = udiv_small(k, nx), j = k - i * nx;
                const SeamEntry R = rows[cy * capy + i], Cc = cols[cx * capx + j];
                // footprint [start - 1, start + nc] inside the valid region of this phase
                if (R.start - 1 < lo || R.start + R.nc > hiY - 1 || Cc.start - 1 < lo || Cc.start + Cc.nc > hiX - 1)
                    continue;
                const uint32_t tile = static_cast<uint32_t>(R.t) * static_cast<uint32_t>(ax.T) + static_cast<uint32_t>(Cc.t);
                const uint32_t base = win0 + static_cast<uint32_t>(R.start * P + Cc.start);
                tile_seam<ARITY>(philox(tile, C.c1, C.c2, s32), base, tile, R.nc == 1, Cc.nc == 1, C);
            }
            __syncthreads();
        }
    }
}

// Wrapping byte copy of a window (any L; windows may wrap several times around small axes).
__device__ void load_window_bytes(uint8_t* win, const uint8_t* src, int H, int L, int P, int Wh, int Ww, int wy0,
                                  int wx0) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int y = warp; y < Wh; y += nw) {
        const uint8_t* srow = src + static_cast<size_t>((wy0 + y) % H) * L;
        uint8_t* drow = win + y * P;
        for (int x = lane; x < Ww; x += 32) drow[x] = srow[(wx0 + x) % L];
    }
}

template <int ARITY, int BMODE, bool BF, bool TAB>
__global__ void __launch_bounds__(kBlockThreads) block_kernel(BlockArgs a) {
    constexpr bool REFLECT = BMODE == 1, SEAM = BMODE == 2;
    extern __shared__ __align__(128) uint8_t smem[];
    // Programmatic dependent launch: let the next launch's CTAs start their prologue as soon as SMs
    // free up; everything that reads the previous launch's output sits behind griddepcontrol.wait.
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#ifdef ESCG_DIAG_TIMING
    const int dslot = static_cast<int>((a.mcs / (a.nmcs > 0 ? a.nmcs : 1)) & 255);
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMin(&g_diag_span[dslot * 3 + 0], t);
    }
#endif
    const int r = blockIdx.z;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int H = a.H, L = a.L, P = a.P, S1 = a.S + 1;
    const int My = SEAM ? 3 * a.seam_np * a.nmcs : margin_rows(a.nmcs), Mx = SEAM ? My : margin_cols(a.nmcs);
    const int ry0 = a.row_split[blockIdx.y], ry1 = a.row_split[blockIdx.y + 1];
    const int rx0 = a.col_split[blockIdx.x], rx1 = a.col_split[blockIdx.x + 1];
    const int bh = ry1 - ry0, bw = rx1 - rx0;
    const int Wh = bh + 2 * My, Ww = bw + 2 * Mx;
    const size_t N = static_cast<size_t>(H) * L;
    const uint8_t* src = a.src + r * N;
    uint8_t* dst = a.dst + r * N;
    uint8_t* win = smem;
    const int woff = (Wh * P + 15) & ~15;
    uint32_t* sT = reinterpret_cast<uint32_t*>(smem + woff);
    // (256 bytes after the thresholds are reserved: block_smem's layout predates the static tables)
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(smem + woff + ((S1 * S1 * 8 + 15) & ~15) + 32 * 8);
    uint8_t* sScratch = reinterpret_cast<uint8_t*>(sCnt + kMaxSpecies + 1);  // 4 * P bytes (dummy box)
    __shared__ int sLast;
    __shared__ __align__(8) uint64_t sMbar;
    // 16-byte chunks / TMA rows when every window/block column boundary is 16-aligned in memory;
    // TMA also needs the window to wrap at most once per axis.
    const bool v16 = (L & 15) == 0 && (rx0 & 15) == 0 && (bw & 15) == 0;
    const bool tma = v16 && Wh <= H && Ww <= L;
    DIAG_STAMP(0);

    if (SEAM && a.step) {
        const uint32_t s32 = seed32(a.seeds[r]);
        const int wy0 = ((ry0 - My) % H + H) % H, wx0 = ((rx0 - Mx) % L + L) % L;
        fill_pair_thresholds<ARITY>(reinterpret_cast<uint2*>(sT), a.rule.T, S1);
        attempt_setup<ARITY>(a.rule, smem_addr(sT), S1, P);
        SeamEntry* rows = reinterpret_cast<SeamEntry*>(
            (reinterpret_cast<uintptr_t>(sScratch) + 4 * P + 15) & ~static_cast<uintptr_t>(15));
        SeamEntry* cols = rows + 3 * (Wh / 2 + 2);
        __shared__ int sSeamCnt[6];
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (a.run.status[r] != kStatusRunning) return;  // uniform per CTA
        load_window_bytes(win, src, H, L, P, Wh, Ww, wy0, wx0);
        __syncthreads();
        block_phases_seam<ARITY, BF>(a.rule, smem_addr(win), H, L, P, a.nmcs, a.mcs, Wh, Ww, wy0, wx0, s32, rows, cols,
                                 sSeamCnt);
        copy_region<false>(win + My * P + Mx, P, dst + static_cast<size_t>(ry0) * L + rx0, L, bh, bw);
    } else if (REFLECT && a.step) {
        const uint32_t s32 = seed32(a.seeds[r]);
        const int wy0 = max(0, ry0 - My), wx0 = max(0, rx0 - Mx);
        const int wh = min(H, ry1 + My) - wy0, ww = min(L, rx1 + Mx) - wx0;
        fill_pair_thresholds<ARITY>(reinterpret_cast<uint2*>(sT), a.rule.T, S1);
        attempt_setup<ARITY>(a.rule, smem_addr(sT), S1, P);
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (a.run.status[r] != kStatusRunning) return;  // uniform per CTA
        copy_region<true>(win, P, const_cast<uint8_t*>(src) + static_cast<size_t>(wy0) * L + wx0, L, wh, ww);
        __syncthreads();
        block_phases_reflect<ARITY, BF>(a.rule, smem_addr(win), H, L, P, a.nmcs, a.mcs, wh, ww, wy0, wx0, Mx - My, s32);
        copy_region<false>(win + (ry0 - wy0) * P + (rx0 - wx0), P, dst + static_cast<size_t>(ry0) * L + rx0, L, bh, bw);
    } else if (a.step) {
        const uint32_t s32 = seed32(a.seeds[r]);
        const int wy0 = a.wrap_rows ? ((ry0 - My) % H + H) % H : ry0 - My;  // bands: halo rows, no wrap
        const int wx0 = ((rx0 - Mx) % L + L) % L;
        const uint32_t mbar = smem_addr(&sMbar);
        // prologue: inputs that no earlier launch writes (rule, seeds, geometry)
        fill_pair_thresholds<ARITY>(reinterpret_cast<uint2*>(sT), a.rule.T, S1);
        attempt_setup<ARITY>(a.rule, smem_addr(sT), S1, P);
        if (TAB && tid < 32) {
            BlockGeom gt;
            gt.nmcs = a.nmcs;
            gt.mcs = a.mcs;
            if (a.narrow)
                build_phase_table<true>(gt, Wh, Ww, s32);
            else
                build_phase_table<false>(gt, Wh, Ww, s32);
        }
        // the scratch box must hold valid species codes: dummy attempts index the threshold table
        for (int i = tid; i < P; i += nt) reinterpret_cast<uint32_t*>(sScratch)[i] = 0u;
        if (tma && tid == 0) {
            mbar_init(mbar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
#ifdef ESCG_DIAG_TIMING
        if (threadIdx.x == 0) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            atomicMin(&g_diag_span[dslot * 3 + 1], t);
        }
#endif
        if (a.run.status[r] != kStatusRunning) return;  // uniform per CTA
#ifndef ESCG_DIAG_NO_LOAD
        if (tma) {
            if (tid == 0) mbar_expect_tx_arrive(mbar, static_cast<uint32_t>(Wh * Ww));
            __syncthreads();
            load_window_tma(win, src, H, L, P, Wh, Ww, wy0, wx0, mbar);
        } else if (v16) {
            load_window<16>(win, src, H, L, P, Wh, Ww, wy0, wx0);
        } else {
            load_window<4>(win, src, H, L, P, Wh, Ww, wy0, wx0);
        }
#endif
        DIAG_STAMP(1);
#ifndef ESCG_DIAG_NO_LOAD
        if (tma) mbar_wait(mbar, 0);
#endif
        __syncthreads();
        DIAG_STAMP(2);
        const uint32_t win0 = smem_addr(win);
        BlockGeom g;
        g.P = P;
        g.H = H;
        g.L = L;
        g.Hg = a.Hg;
        g.row0 = a.row0;
        g.nmcs = a.nmcs;
        g.mcs = a.mcs;
        g.scratch = smem_addr(sScratch) + static_cast<uint32_t>(P + 1);
        if (a.narrow)
            block_phases_any<ARITY, true, false, TAB>(g, a.rule, win0, Wh, Ww, wy0, wx0, s32);
        else
            block_phases_any<ARITY, false, BF, TAB>(g, a.rule, win0, Wh, Ww, wy0, wx0, s32);
#ifndef ESCG_DIAG_NO_LOAD
        if (tma) {
            // generic-proxy writes → async proxy, then one bulk store per block row
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            for (int y = tid; y < bh; y += nt)
                bulk_s2g(dst + static_cast<size_t>(ry0 + y) * L + rx0, win0 + (My + y) * P + Mx, static_cast<uint32_t>(bw));
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        } else if (v16) {
            store_block<16>(dst, win, L, P, bh, bw, ry0, rx0, My, Mx);
        } else {
            store_block<4>(dst, win, L, P, bh, bw, ry0, rx0, My, Mx);
        }
#endif
    } else {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (a.run.status[r] != kStatusRunning) return;  // uniform per CTA
    }
    if (a.count) {
        for (int v = tid; v <= kMaxSpecies; v += nt) sCnt[v] = 0;
        __syncthreads();
        if (a.step && REFLECT)
            block_count(win + (ry0 - max(0, ry0 - My)) * P + (rx0 - max(0, rx0 - Mx)), bh, bw, P, S1, sCnt);
        else if (a.step)
            block_count(win + My * P + Mx, bh, bw, P, S1, sCnt);
        else
            block_count(src + static_cast<size_t>(ry0) * L + rx0, bh, bw, L, S1, sCnt);
        __syncthreads();
        if (tid == 0) {
            for (int v = 0; v < S1; ++v)
                if (sCnt[v]) atomicAdd(&a.acc[r * S1 + v], static_cast<unsigned long long>(sCnt[v]));
            __threadfence();
            const unsigned int t = atomicAdd(&a.ticket[r], 1u);
            sLast = t == static_cast<unsigned int>(a.nby * a.nbx - 1);
        }
        __syncthreads();
        if (sLast && tid == 0) {
            __threadfence();
            uint64_t c64[kMaxSpecies + 1];
            for (int v = 0; v < S1; ++v) c64[v] = atomicExch(&a.acc[r * S1 + v], 0ull);
            a.ticket[r] = 0u;
            if (a.run.cur) a.run.cur[r] = a.step ? a.dst_index : 1 - a.dst_index;
            record_decide(c64, S1, a.mcs + (a.step ? a.nmcs : 0), r, a.run);
        }
    }
    DIAG_STAMP(8);
    // bulk stores must finish reading shared memory before the CTA exits
    if (a.step && tma) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    DIAG_STAMP(9);
#ifdef ESCG_DIAG_TIMING
    if (threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(&g_diag_span[dslot * 3 + 2], t);
    }
#endif
}

// Persistent variant: one cooperative launch runs every chunk of a run; a grid barrier replaces the
// kernel boundary.  Records: CTAs add their block counts into acc3[r % 3]; after the barrier every
// CTA reads the same totals and takes the same stop decision; CTA 0 writes the record and zeroes
// acc3[(r + 2) % 3] (last read before the previous barrier, next written after the next one).
template <int ARITY>
__global__ void __launch_bounds__(1024) block_kernel_persistent(PersistArgs pa) {
    namespace cg = cooperative_groups;
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) uint8_t smem[];
    const BlockArgs& a = pa.b;
    const int r = blockIdx.z;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int H = a.H, L = a.L, P = a.P, S1 = a.S + 1;
    const int kmax = pa.kmcs;
    const int My = margin_rows(kmax), Mx = margin_cols(kmax);
    const int ry0 = a.row_split[blockIdx.y], ry1 = a.row_split[blockIdx.y + 1];
    const int rx0 = a.col_split[blockIdx.x], rx1 = a.col_split[blockIdx.x + 1];
    const int bh = ry1 - ry0, bw = rx1 - rx0;
    const size_t N = static_cast<size_t>(H) * L;
    uint8_t* win = smem;
    const int Whm = bh + 2 * My;
    const int woff = (Whm * P + 15) & ~15;
    uint32_t* sT = reinterpret_cast<uint32_t*>(smem + woff);
    // (256 bytes after the thresholds are reserved: block_smem's layout predates the static tables)
    uint32_t* sCnt = reinterpret_cast<uint32_t*>(smem + woff + ((S1 * S1 * 8 + 15) & ~15) + 32 * 8);
    uint8_t* sScratch = reinterpret_cast<uint8_t*>(sCnt + kMaxSpecies + 1);
    __shared__ __align__(8) uint64_t sMbar;

    const uint32_t s32 = seed32(a.seeds[r]);
    fill_pair_thresholds<ARITY>(reinterpret_cast<uint2*>(sT), a.rule.T, S1);
    attempt_setup<ARITY>(a.rule, smem_addr(sT), S1, P);
    for (int i = tid; i < P; i += nt) reinterpret_cast<uint32_t*>(sScratch)[i] = 0u;
    const uint32_t mbar = smem_addr(&sMbar);
    if (tid == 0) {
        mbar_init(mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint32_t win0 = smem_addr(win);
    const RunArgs& run = a.run;
    const int64_t limit = pa.record ? run.mcs_limit : pa.mcs_end;
    int64_t mcs = pa.mcs0;
    int par = 0;       // buffer holding the lattice
    int64_t rec = 0;   // record index
    uint32_t tma_phase = 0;
    bool running = true;

    // record_and_check on the current lattice (block region in `src`, pitch `pitch`)
    auto do_record = [&](const uint8_t* base, int pitch) {
        for (int v = tid; v <= kMaxSpecies; v += nt) sCnt[v] = 0;
        __syncthreads();
        block_count(base, bh, bw, pitch, S1, sCnt);
        __syncthreads();
        unsigned long long* acc = pa.acc3 + (static_cast<size_t>(rec % 3) * gridDim.z + r) * S1;
        if (tid < S1 && sCnt[tid]) atomicAdd(&acc[tid], static_cast<unsigned long long>(sCnt[tid]));
        grid.sync();
        uint64_t c64[kMaxSpecies + 1];
        int alive = 0;
        for (int v = 0; v < S1; ++v) {
            c64[v] = *reinterpret_cast<volatile unsigned long long*>(&acc[v]);
            if (v >= 1 && c64[v] > 0) ++alive;
        }
        int st = kStatusRunning;
        if ((run.stop_flags & kStopTracked) && run.tracked >= 1 && run.tracked < S1 && c64[run.tracked] == 0)
            st = kStopped;
        else if (mcs >= run.mcs_limit)
            st = kCompleted;
        else if ((run.stop_flags & kStopStasis) && alive <= 1)
            st = kStasis;
        if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
            record_decide(c64, S1, mcs, r, run);
            if (run.cur) run.cur[r] = par;
            unsigned long long* z = pa.acc3 + (static_cast<size_t>((rec + 2) % 3) * gridDim.z + r) * S1;
            for (int v = 0; v < S1; ++v) z[v] = 0ull;
        }
        ++rec;
        running = st == kStatusRunning;
    };

    if (pa.record) do_record(pa.buf[0] + r * N + static_cast<size_t>(ry0) * L + rx0, L);
    int64_t next_rec = pa.record ? pa.mcs0 + run.interval : limit;
    while (running && mcs < limit) {
        const int64_t target = pa.record ? (next_rec < limit ? next_rec : limit) : limit;
        const int chunk = static_cast<int>((target - mcs) < kmax ? (target - mcs) : kmax);
        const int Myc = margin_rows(chunk), Mxc = margin_cols(chunk);
        const int Wh = bh + 2 * Myc, Ww = bw + 2 * Mxc;
        const int wy0 = ((ry0 - Myc) % H + H) % H;
        const int wx0 = ((rx0 - Mxc) % L + L) % L;
        const uint8_t* src = pa.buf[par] + r * N;
        uint8_t* dst = pa.buf[1 - par] + r * N;
        // generic-proxy writes of the previous chunk (other CTAs) → this CTA's async-proxy reads
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (tid == 0) mbar_expect_tx_arrive(mbar, static_cast<uint32_t>(Wh * Ww));
        if (tid < 32) {  // phase table of this chunk (the previous chunk's phases are done)
            BlockGeom gt;
            gt.nmcs = chunk;
            gt.mcs = mcs;
            if (a.narrow)
                build_phase_table<true>(gt, Wh, Ww, s32);
            else
                build_phase_table<false>(gt, Wh, Ww, s32);
        }
        __syncthreads();
        load_window_tma(win, src, H, L, P, Wh, Ww, wy0, wx0, mbar);
        mbar_wait(mbar, tma_phase);
        tma_phase ^= 1u;
        __syncthreads();
        BlockGeom g;
        g.P = P;
        g.H = H;
        g.L = L;
        g.Hg = a.Hg;
        g.row0 = a.row0;
        g.nmcs = chunk;
        g.mcs = mcs;
        g.scratch = smem_addr(sScratch) + static_cast<uint32_t>(P + 1);
        if (a.narrow)
            block_phases_any<ARITY, true, false, true>(g, a.rule, win0, Wh, Ww, wy0, wx0, s32);
        else
            block_phases_any<ARITY, false, false, true>(g, a.rule, win0, Wh, Ww, wy0, wx0, s32);
        store_block<16>(dst, win, L, P, bh, bw, ry0, rx0, Myc, Mxc);
        mcs += chunk;
        par ^= 1;
        if (pa.record && mcs == target) {
            __threadfence();
            do_record(win + Myc * P + Mxc, P);  // includes the grid barrier
            next_rec = mcs + run.interval;
        } else {
            __threadfence();
            grid.sync();
        }
    }
    if (!pa.record && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) {
        run.mcs[r] = mcs;
        if (run.cur) run.cur[r] = par;
    }
}

// ---------------------------------------------------------------------------------------------
// Helpers
// ---------------------------------------------------------------------------------------------

// Device init_lattice: lattice.hpp:53-66's transform applied to Philox INIT-domain words
// (cell pair i>>1 → 4 words: (empty, species) for the even then the odd cell).
__global__ void init_kernel(InitArgs a) {
    const int64_t pairs = (a.n + 1) >> 1;
    const int64_t total = pairs * a.nrep;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(t / pairs);
        const int64_t pi = t - static_cast<int64_t>(r) * pairs;
        uint8_t* lat = a.lat + static_cast<size_t>(r) * a.n;
        const uint32_t S = static_cast<uint32_t>(a.S);
        for (int h = 0; h < 2; ++h) {
            const int64_t i = 2 * pi + h;
            if (i >= a.n) break;
            // global cell index of local cell i (band engines start at global row row0)
            const int64_t lr = i / a.L, col = i - lr * a.L;
            const int64_t gi = ((a.row0 + lr) % a.Hg) * a.L + col;
            const uint4 w = philox(static_cast<uint32_t>(gi >> 1), 0u, ctr2(0, kDomInit, 0u, 0u), seed32(a.seeds[r]));
            const uint32_t we = (gi & 1) ? w.z : w.x, ws = (gi & 1) ? w.w : w.y;
            uint8_t v = 0;
            if (!a.all_empty && we >= a.x_empty) v = static_cast<uint8_t>(ws % S + 1u);
            lat[i] = v;
        }
    }
}

__global__ void count_kernel(const uint8_t* lat, int64_t n, int S1, unsigned long long* out) {
    __shared__ uint32_t sCnt[kMaxSpecies + 1];
    const int r = blockIdx.y;
    for (int v = threadIdx.x; v < S1; v += blockDim.x) sCnt[v] = 0;
    __syncthreads();
    const uint8_t* base = lat + static_cast<size_t>(r) * n;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        atomicAdd(&sCnt[base[i]], 1u);
    __syncthreads();
    for (int v = threadIdx.x; v < S1; v += blockDim.x)
        if (sCnt[v]) atomicAdd(&out[r * S1 + v], static_cast<unsigned long long>(sCnt[v]));
}

// Serial replay of injected reference draws (engine.cpp:104-110) with the production rule.
__global__ void replay_kernel(ReplayArgs a) {
    const uint32_t n = static_cast<uint32_t>(static_cast<int64_t>(a.H) * a.L);
    const int S1 = a.S + 1;
    for (int64_t k = 0; k < a.n_attempts; ++k) {
        const uint32_t cell = a.wc[k] % n;
        const uint32_t d = a.wd[k] % static_cast<uint32_t>(a.arity);
        int dr, dc;
        dir_rc(d, dr, dc);
        const int y = static_cast<int>(cell / static_cast<uint32_t>(a.L));
        const int x = static_cast<int>(cell % static_cast<uint32_t>(a.L));
        int ny = y + dr, nx = x + dc;
        if (a.flux) {
            ny = (ny + a.H) % a.H;
            nx = (nx + a.L) % a.L;
        } else {
            if (ny < 0) ny = -ny;
            if (ny >= a.H) ny = 2 * (a.H - 1) - ny;
            if (nx < 0) nx = -nx;
            if (nx >= a.L) nx = 2 * (a.L - 1) - nx;
        }
        const int64_t ni = static_cast<int64_t>(ny) * a.L + nx;
        // the production rule with the injected full 32-bit action word
        const uint32_t r = rule_exact(a.lat[cell], a.lat[ni], a.wa[k], a.rule.xm, a.rule.xi, a.rule.T, S1);
        a.lat[cell] = static_cast<uint8_t>(r & 0xFFu);
        a.lat[ni] = static_cast<uint8_t>(r >> 8);
    }
}

__global__ void u8_to_i32_kernel(const uint8_t* src, int32_t* dst, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

__global__ void i32_to_u8_kernel(const int32_t* src, uint8_t* dst, int64_t n, int S, int* bad) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int32_t v = src[i];
        if (v < 0 || v > S) {
            atomicExch(bad, 1);
            dst[i] = 0;
        } else {
            dst[i] = static_cast<uint8_t>(v);
        }
    }
}

int grid_for(int64_t n, int threads) {
    int64_t g = (n + threads - 1) / threads;
    if (g > 148 * 16) g = 148 * 16;
    return g < 1 ? 1 : static_cast<int>(g);
}

}  // namespace

int tile_smem_bytes(int H, int L, int S, int* pitch) {
    // pitch ≡ 0 (mod 128) keeps a tile's footprint column in one bank group (conflict-light
    // accesses); fall back to 16-byte alignment when the padded lattice would not fit.
    int P = (L + kTileC0 + 1 + 127) & ~127;
    if (tile_layout(H, L, S, P).total > max_smem_optin(0)) P = align16(L + kTileC0 + 1);
    if (pitch) *pitch = P;
    return tile_layout(H, L, S, P).total;
}

// Diagnostic: copy the block kernel's section stamps (ESCG_DIAG_TIMING builds; else returns 0).
extern "C" __attribute__((visibility("default"))) int escg_diag_spans(unsigned long long* out, int reset) {
#ifdef ESCG_DIAG_TIMING
    if (reset) {
        static unsigned long long init[256 * 3];
        for (int i = 0; i < 256; ++i) {
            init[3 * i] = ~0ull;
            init[3 * i + 1] = ~0ull;
            init[3 * i + 2] = 0ull;
        }
        return cudaMemcpyToSymbol(g_diag_span, init, sizeof(init)) == cudaSuccess ? 0 : -1;
    }
    return cudaMemcpyFromSymbol(out, g_diag_span, sizeof(unsigned long long) * 256 * 3) == cudaSuccess ? 0 : -1;
#else
    (void)out;
    (void)reset;
    return -1;
#endif
}

extern "C" __attribute__((visibility("default"))) int escg_diag_warps(unsigned long long* out, int n) {
#ifdef ESCG_DIAG_TIMING
    return cudaMemcpyFromSymbol(out, g_diag_w, sizeof(unsigned long long) * (n < 8 * 32 * 16 ? n : 8 * 32 * 16)) ==
                   cudaSuccess
               ? n
               : -1;
#else
    (void)out;
    (void)n;
    return 0;
#endif
}

extern "C" __attribute__((visibility("default"))) int escg_diag_timing(unsigned long long* out, int n) {
#ifdef ESCG_DIAG_TIMING
    return cudaMemcpyFromSymbol(out, g_diag_t, sizeof(unsigned long long) * (n < 4096 * 16 ? n : 4096 * 16)) ==
                   cudaSuccess
               ? n
               : -1;
#else
    (void)out;
    (void)n;
    return 0;
#endif
}

// Dynamic shared memory available per CTA: the opt-in limit minus a reserve for the kernels'
// static shared variables (offset table, slow-path parameters, barriers; < 1 KB).
int max_smem_optin(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return v - 1024;
}

cudaError_t launch_init(const InitArgs& a, cudaStream_t s) {
    init_kernel<<<grid_for(((a.n + 1) >> 1) * a.nrep, 256), 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_count(const uint8_t* lat, int64_t n, int nrep, int S, unsigned long long* out, cudaStream_t s) {
    cudaMemsetAsync(out, 0, sizeof(unsigned long long) * (S + 1) * nrep, s);
    dim3 grid(static_cast<unsigned>(grid_for(n, 256) > 64 ? 64 : grid_for(n, 256)), static_cast<unsigned>(nrep));
    count_kernel<<<grid, 256, 0, s>>>(lat, n, S + 1, out);
    return cudaGetLastError();
}

template <int ARITY, int MODE>
static cudaError_t tile_launch_t(const TileArgs& a, int nrep, int threads, cudaStream_t s) {
    const bool one = a.one_per_sm != 0;
    auto k = a.rule.wide_bf ? (one ? tile_kernel<ARITY, MODE, true, true> : tile_kernel<ARITY, MODE, true, false>)
                            : (one ? tile_kernel<ARITY, MODE, false, true> : tile_kernel<ARITY, MODE, false, false>);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
    if (e != cudaSuccess) return e;
    k<<<nrep, threads, a.smem_bytes, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_tile(const TileArgs& a, int nrep, int threads, cudaStream_t s) {
    const int mode = !a.flux ? kModeReflect : ((a.H % 4 == 0 && a.L % 4 == 0) ? kModePeriodic : kModeSeam);
    if (a.arity == 8) {
        if (mode == kModeReflect) return tile_launch_t<8, kModeReflect>(a, nrep, threads, s);
        if (mode == kModeSeam) return tile_launch_t<8, kModeSeam>(a, nrep, threads, s);
        return tile_launch_t<8, kModePeriodic>(a, nrep, threads, s);
    }
    if (mode == kModeReflect) return tile_launch_t<4, kModeReflect>(a, nrep, threads, s);
    if (mode == kModeSeam) return tile_launch_t<4, kModeSeam>(a, nrep, threads, s);
    return tile_launch_t<4, kModePeriodic>(a, nrep, threads, s);
}

template <int ARITY, int BMODE>
static cudaError_t block_launch_t(const BlockArgs& a, int nrep, int threads, cudaStream_t s) {
    // NARROW launches never consult the WIDE rule: one instantiation
    const bool bf = a.rule.wide_bf && !a.narrow;
    // the dynamic-smem opt-in is a per-device function attribute: remember it per device (band
    // groups drive several devices from one thread); atomics keep concurrent host threads safe
    const bool tab = a.phase_table != 0 && BMODE == 0;
    static std::atomic<int> configured[4][kMaxDevices];  // [rule form x phase table][device]
    std::atomic<int>* configured_bytes = configured[(bf ? 1 : 0) + (tab ? 2 : 0)];
    auto k = bf ? (tab ? block_kernel<ARITY, BMODE, true, true> : block_kernel<ARITY, BMODE, true, false>)
                : (tab ? block_kernel<ARITY, BMODE, false, true> : block_kernel<ARITY, BMODE, false, false>);
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDevices || configured_bytes[dev].load() < a.smem_bytes) {
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
        if (e != cudaSuccess) return e;
        if (dev >= 0 && dev < kMaxDevices) {
            int cur = configured_bytes[dev].load();
            while (cur < a.smem_bytes && !configured_bytes[dev].compare_exchange_weak(cur, a.smem_bytes)) {
            }
        }
    }
    dim3 grid(static_cast<unsigned>(a.nbx), static_cast<unsigned>(a.nby), static_cast<unsigned>(nrep));
    // programmatic dependent launch (the kernel waits with griddepcontrol.wait before touching the
    // previous launch's output); ESCG_PDL=0 turns it off
    static const bool pdl = !(std::getenv("ESCG_PDL") && std::getenv("ESCG_PDL")[0] == '0');
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = static_cast<size_t>(a.smem_bytes);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, a);
}

// Registers per thread of the periodic block kernel (the launch bound decides them).
int block_kernel_registers(int arity) {
    cudaFuncAttributes fa{};
    const void* f = arity == 8 ? reinterpret_cast<const void*>(block_kernel<8, 0, false, false>)
                               : reinterpret_cast<const void*>(block_kernel<4, 0, false, false>);
    if (cudaFuncGetAttributes(&fa, f) != cudaSuccess) return 64;
    return fa.numRegs;
}

// Concurrent tile-kernel CTAs (one per replica) the device holds at this CTA shape.
template <bool ONE>
static const void* tile_fn(int arity, int mode) {
    if (arity == 8)
        return mode == kModeReflect ? reinterpret_cast<const void*>(tile_kernel<8, kModeReflect, false, ONE>)
               : mode == kModeSeam  ? reinterpret_cast<const void*>(tile_kernel<8, kModeSeam, false, ONE>)
                                    : reinterpret_cast<const void*>(tile_kernel<8, kModePeriodic, false, ONE>);
    return mode == kModeReflect ? reinterpret_cast<const void*>(tile_kernel<4, kModeReflect, false, ONE>)
           : mode == kModeSeam  ? reinterpret_cast<const void*>(tile_kernel<4, kModeSeam, false, ONE>)
                                : reinterpret_cast<const void*>(tile_kernel<4, kModePeriodic, false, ONE>);
}

int tile_capacity(int arity, int flux, int H, int L, int threads, int smem_bytes, int device) {
    const int mode = !flux ? kModeReflect : ((H % 4 == 0 && L % 4 == 0) ? kModePeriodic : kModeSeam);
    const void* f = tile_one_per_sm(smem_bytes) ? tile_fn<true>(arity, mode) : tile_fn<false>(arity, mode);
    int per_sm = 0, sms = 0;
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, threads, smem_bytes) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return per_sm * sms;
}

int block_persistent_capacity(int arity, int threads, int smem_bytes, int device) {
    int per_sm = 0, sms = 0;
    auto k4 = block_kernel_persistent<4>;
    auto k8 = block_kernel_persistent<8>;
    const void* f = arity == 8 ? reinterpret_cast<const void*>(k8) : reinterpret_cast<const void*>(k4);
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess) return 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, threads, smem_bytes) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
    return coop ? per_sm * sms : 0;
}

cudaError_t launch_block_persistent(const PersistArgs& a, int nrep, int threads, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>(a.b.nbx), static_cast<unsigned>(a.b.nby), static_cast<unsigned>(nrep));
    void* args[] = {const_cast<PersistArgs*>(&a)};
    const void* f = a.b.arity == 8 ? reinterpret_cast<const void*>(block_kernel_persistent<8>)
                                   : reinterpret_cast<const void*>(block_kernel_persistent<4>);
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, a.b.smem_bytes);
    if (e != cudaSuccess) return e;
    return cudaLaunchCooperativeKernel(f, grid, dim3(static_cast<unsigned>(threads)), args, a.b.smem_bytes, s);
}

cudaError_t launch_block(const BlockArgs& a, int nrep, int threads, cudaStream_t s) {
    if (a.reflect)
        return a.arity == 8 ? block_launch_t<8, 1>(a, nrep, threads, s) : block_launch_t<4, 1>(a, nrep, threads, s);
    if (a.seam_np > 0)
        return a.arity == 8 ? block_launch_t<8, 2>(a, nrep, threads, s) : block_launch_t<4, 2>(a, nrep, threads, s);
    return a.arity == 8 ? block_launch_t<8, 0>(a, nrep, threads, s) : block_launch_t<4, 0>(a, nrep, threads, s);
}

cudaError_t launch_replay(const ReplayArgs& a, cudaStream_t s) {
    replay_kernel<<<1, 1, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_u8_to_i32(const uint8_t* src, int32_t* dst, int64_t n, cudaStream_t s) {
    u8_to_i32_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n);
    return cudaGetLastError();
}

cudaError_t launch_i32_to_u8(const int32_t* src, uint8_t* dst, int64_t n, int S, int* bad, cudaStream_t s) {
    i32_to_u8_kernel<<<grid_for(n, 256), 256, 0, s>>>(src, dst, n, S, bad);
    return cudaGetLastError();
}

}  // namespace escgd
