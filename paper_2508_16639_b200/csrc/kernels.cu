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
#include <cuda_runtime.h>

#include <cstdint>

#include "crs.cuh"
#include "launch.h"

namespace escgd {

namespace {

constexpr int kStatusRunning = -1;
constexpr int kCompleted = 0, kStasis = 1, kStopped = 2;
constexpr uint32_t kStopTracked = 1u, kStopStasis = 2u;

__host__ __device__ __forceinline__ int align16(int x) { return (x + 15) & ~15; }

// record_and_check (engine.cpp:47-57) for one replica, executed by a single thread.
__device__ int record_decide(const uint64_t* counts, int S1, int64_t mcs, int r, const RunArgs& run) {
    const int64_t k = run.n_rec[r];
    if (run.trace_steps != nullptr && k < run.trace_cap) {
        run.trace_steps[r * run.trace_cap + k] = mcs;
        for (int v = 0; v < S1; ++v) run.trace_counts[(r * run.trace_cap + k) * S1 + v] = counts[v];
    }
    run.n_rec[r] = k + 1;
    int alive = 0;
    for (int v = 0; v < S1; ++v) {
        run.last_counts[r * S1 + v] = counts[v];
        if (v >= 1 && counts[v] > 0) ++alive;
    }
    run.mcs[r] = mcs;
    int st = kStatusRunning;
    if ((run.stop_flags & kStopTracked) && run.tracked >= 1 && run.tracked < S1 && counts[run.tracked] == 0)
        st = kStopped;
    else if (mcs >= run.mcs_limit)
        st = kCompleted;
    else if ((run.stop_flags & kStopStasis) && alive <= 1)
        st = kStasis;
    run.status[r] = st;
    return st;
}

// Species histogram of a rows x cols region of a byte array with the given pitch into sCnt
// (shared, zeroed by the caller).  S1 <= 8 uses SIMD byte compares + popc in registers.
__device__ void block_count(const uint8_t* base, int rows, int cols, int pitch, int S1, uint32_t* sCnt) {
    const int tid = threadIdx.x, nt = blockDim.x;
    if (S1 <= 8 && (cols & 3) == 0 && (pitch & 3) == 0 && ((reinterpret_cast<uintptr_t>(base) & 3) == 0)) {
        uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const int wpr = cols >> 2;
        const int total = rows * wpr;
        for (int idx = tid; idx < total; idx += nt) {
            const int y = idx / wpr;
            const int x = idx - y * wpr;
            const uint32_t w = *reinterpret_cast<const uint32_t*>(base + y * pitch + 4 * x);
#pragma unroll
            for (int v = 0; v < 8; ++v)
                if (v < S1) c[v] += __popc(__vcmpeq4(w, 0x01010101u * static_cast<uint32_t>(v)));
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) {
            if (v < S1) {
                const uint32_t s = __reduce_add_sync(0xffffffffu, c[v]);
                if ((tid & 31) == 0 && s) atomicAdd(&sCnt[v], s >> 3);
            }
        }
    } else {
        const int total = rows * cols;
        for (int idx = tid; idx < total; idx += nt) {
            const int y = idx / cols;
            const int x = idx - y * cols;
            atomicAdd(&sCnt[base[y * pitch + x]], 1u);
        }
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
    t.snap_off = t.T_off + align16(S1 * S1 * 4);
    t.cnt_off = t.snap_off + align16(3 * (L + 3) + 3 * H);
    t.flag_off = t.cnt_off + align16((kMaxSpecies + 1) * 4);
    t.total = t.flag_off + 16;
    return t;
}

// Ghost cell k → (gy, gx) in lattice coordinates (rows {-2,-1,H} x cols [-2,L], then
// cols {-2,-1,L} x rows [0,H)).
__device__ __forceinline__ void ghost_pos(int k, int H, int L, int& gy, int& gx) {
    const int rowband = 3 * (L + 3);
    if (k < rowband) {
        const int b = k / (L + 3);
        gx = k - b * (L + 3) - 2;
        gy = b == 0 ? -2 : (b == 1 ? -1 : H);
    } else {
        const int k2 = k - rowband;
        const int b = k2 / H;
        gy = k2 - b * H;
        gx = b == 0 ? -2 : (b == 1 ? -1 : L);
    }
}

__device__ __forceinline__ int wrap(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// After a phase: a ghost that changed carries the phase's write of its physical cell (at most one
// representation of a physical cell lies in an active footprint per phase).
__device__ void ghost_fold(uint8_t* lat, const uint8_t* snap, int H, int L, int P) {
    const int G = 3 * (L + 3) + 3 * H;
    for (int k = threadIdx.x; k < G; k += blockDim.x) {
        int gy, gx;
        ghost_pos(k, H, L, gy, gx);
        const uint8_t g = lat[(gy + kTileR0) * P + gx + kTileC0];
        if (g != snap[k]) lat[(wrap(gy, H) + kTileR0) * P + wrap(gx, L) + kTileC0] = g;
    }
}

__device__ void ghost_refresh(uint8_t* lat, uint8_t* snap, int H, int L, int P) {
    const int G = 3 * (L + 3) + 3 * H;
    for (int k = threadIdx.x; k < G; k += blockDim.x) {
        int gy, gx;
        ghost_pos(k, H, L, gy, gx);
        const uint8_t v = lat[(wrap(gy, H) + kTileR0) * P + wrap(gx, L) + kTileC0];
        lat[(gy + kTileR0) * P + gx + kTileC0] = v;
        snap[k] = v;
    }
}

template <int ARITY, bool REFLECT>
__device__ void tile_round(uint8_t* lat, uint8_t* snap, const uint32_t* sT, const Rule& R, int H, int L, int P,
                           int S1, uint32_t k0, uint32_t k1, uint64_t mcs) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const Round rp = round_params(k0, k1, mcs);
    const int Ty = REFLECT ? (H + rp.oy + 1) >> 1 : H >> 1;
    const int Tx = REFLECT ? (L + rp.ox + 1) >> 1 : L >> 1;
#pragma unroll 1
    for (int p = 0; p < 4; ++p) {
        const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
        const int nty = (Ty - cy + 1) >> 1, ntx = (Tx - cx + 1) >> 1;
        const int cnt = nty * ntx;
        if (tid < cnt) {
            int i = tid / ntx, j = tid - (tid / ntx) * ntx;
            const int di = nt / ntx, dj = nt - (nt / ntx) * ntx;
            const uint32_t c2 = ctr2(mcs, kDomStep, static_cast<uint32_t>(p));
            for (int k = tid; k < cnt; k += nt) {
                const int ty = cy + 2 * i, tx = cx + 2 * j;
                const uint32_t tile = static_cast<uint32_t>(ty) * static_cast<uint32_t>(Tx) + static_cast<uint32_t>(tx);
                const uint4 w = philox(tile, static_cast<uint32_t>(mcs), c2, 0u, k0, k1);
                if (REFLECT) {
                    tile_attempts_reflect<ARITY>(lat, 2 * ty - rp.oy, 2 * tx - rp.ox, kTileR0, kTileC0, P, H, L, w, R,
                                                 sT, S1, k0, k1, tile, mcs, p);
                } else {
                    const int base = (2 * ty - rp.oy + kTileR0) * P + (2 * tx - rp.ox + kTileC0);
                    tile_attempts<ARITY>(lat, base, P, w, R, sT, S1, k0, k1, tile, mcs, p);
                }
                j += dj;
                i += di;
                if (j >= ntx) {
                    j -= ntx;
                    ++i;
                }
            }
        }
        __syncthreads();
        if (!REFLECT) {
            ghost_fold(lat, snap, H, L, P);
            __syncthreads();
            ghost_refresh(lat, snap, H, L, P);
            __syncthreads();
        }
    }
}

template <int ARITY, bool REFLECT>
__global__ void __launch_bounds__(512) tile_kernel(TileArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
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
    const uint64_t seed = a.seeds[r];
    const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);

    for (int i = tid; i < S1 * S1; i += nt) sT[i] = a.rule.T[i];
    if ((L & 3) == 0) {
        const int wpr = L >> 2;
        for (int idx = tid; idx < H * wpr; idx += nt) {
            const int y = idx / wpr, c = idx - (idx / wpr) * wpr;
            *reinterpret_cast<uint32_t*>(lat + (y + kTileR0) * P + kTileC0 + 4 * c) =
                *reinterpret_cast<const uint32_t*>(glat + static_cast<size_t>(y) * L + 4 * c);
        }
    } else {
        for (int idx = tid; idx < H * L; idx += nt) {
            const int y = idx / L, x = idx - (idx / L) * L;
            lat[(y + kTileR0) * P + kTileC0 + x] = glat[idx];
        }
    }
    __syncthreads();
    if (!REFLECT) {
        ghost_refresh(lat, snap, H, L, P);
        __syncthreads();
    }
    const Rule R{a.rule.xm, a.rule.xi, a.rule.xm >> Bits<ARITY>::LB, a.rule.xi >> Bits<ARITY>::LB};
    int64_t mcs = a.run.mcs[r];
    int status = a.run.status[r];
    for (;;) {
        int64_t adv;
        if (a.record) {
            for (int v = tid; v < S1; v += nt) sCnt[v] = 0;
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
            tile_round<ARITY, REFLECT>(lat, snap, sT, R, H, L, P, S1, k0, k1, static_cast<uint64_t>(mcs));
    }
    if ((L & 3) == 0) {
        const int wpr = L >> 2;
        for (int idx = tid; idx < H * wpr; idx += nt) {
            const int y = idx / wpr, c = idx - (idx / wpr) * wpr;
            *reinterpret_cast<uint32_t*>(glat + static_cast<size_t>(y) * L + 4 * c) =
                *reinterpret_cast<const uint32_t*>(lat + (y + kTileR0) * P + kTileC0 + 4 * c);
        }
    } else {
        for (int idx = tid; idx < H * L; idx += nt) {
            const int y = idx / L, x = idx - (idx / L) * L;
            glat[idx] = lat[(y + kTileR0) * P + kTileC0 + x];
        }
    }
    if (tid == 0 && !a.record) a.run.mcs[r] = mcs;
}

// ---------------------------------------------------------------------------------------------
// Block kernel (overlapped tiling, one MCS per launch, periodic lattices with H, L ≡ 0 mod 4)
// ---------------------------------------------------------------------------------------------

template <int ARITY>
__global__ void __launch_bounds__(1024) block_kernel(BlockArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const int r = blockIdx.z;
    if (a.run.status[r] != kStatusRunning) return;
    const int tid = threadIdx.x, nt = blockDim.x;
    const int H = a.H, L = a.L, P = a.P, S1 = a.S + 1, M = kMargin;
    const int ry0 = a.row_split[blockIdx.y], ry1 = a.row_split[blockIdx.y + 1];
    const int rx0 = a.col_split[blockIdx.x], rx1 = a.col_split[blockIdx.x + 1];
    const int bh = ry1 - ry0, bw = rx1 - rx0;
    const int Wh = bh + 2 * M, Ww = bw + 2 * M;
    const size_t N = static_cast<size_t>(H) * L;
    const uint8_t* src = a.src + r * N;
    uint8_t* dst = a.dst + r * N;
    uint8_t* win = smem;
    uint32_t* sT = reinterpret_cast<uint32_t*>(smem + align16(Wh * P));
    uint32_t* sCnt = sT + S1 * S1;
    __shared__ int sLast;

    if (a.step) {
        const uint64_t seed = a.seeds[r];
        const uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
        const uint64_t mcs = static_cast<uint64_t>(a.mcs);
        const int wy0 = ((ry0 - M) % H + H) % H;
        const int wx0 = ((rx0 - M) % L + L) % L;
        for (int i = tid; i < S1 * S1; i += nt) sT[i] = a.rule.T[i];
        {
            const int wpr = Ww >> 2;
            for (int idx = tid; idx < Wh * wpr; idx += nt) {
                const int wr = idx / wpr, c = idx - (idx / wpr) * wpr;
                const int gy = (wy0 + wr) % H;
                const int gx = (wx0 + 4 * c) % L;
                *reinterpret_cast<uint32_t*>(win + wr * P + 4 * c) =
                    __ldcg(reinterpret_cast<const unsigned int*>(src + static_cast<size_t>(gy) * L + gx));
            }
        }
        __syncthreads();
        const Rule R{a.rule.xm, a.rule.xi, a.rule.xm >> Bits<ARITY>::LB, a.rule.xi >> Bits<ARITY>::LB};
        const Round rp = round_params(k0, k1, mcs);
        const int Ty = H >> 1, Tx = L >> 1;
        const int jb = wy0 >> 1, ib = wx0 >> 1;  // global tile index of window tile 0 (even)
#pragma unroll 1
        for (int p = 0; p < 4; ++p) {
            const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
            const int lo = 3 * p, hiR = Wh - 3 * p, hiC = Ww - 3 * p;
            // footprint rows [2j-oy-1, 2j-oy+2] within [lo, hiR)
            const int jmin = (lo + rp.oy + 2) >> 1, jmax = (hiR - 3 + rp.oy) >> 1;
            const int imin = (lo + rp.ox + 2) >> 1, imax = (hiC - 3 + rp.ox) >> 1;
            const int j0 = jmin + ((jmin ^ cy) & 1), i0 = imin + ((imin ^ cx) & 1);
            const int nj = jmax >= j0 ? ((jmax - j0) >> 1) + 1 : 0;
            const int ni = imax >= i0 ? ((imax - i0) >> 1) + 1 : 0;
            const int cnt = nj * ni;
            if (tid < cnt) {
                int aa = tid / ni, bb = tid - (tid / ni) * ni;
                const int da = nt / ni, db = nt - (nt / ni) * ni;
                const uint32_t c2 = ctr2(mcs, kDomStep, static_cast<uint32_t>(p));
                for (int k = tid; k < cnt; k += nt) {
                    const int j = j0 + 2 * aa, i = i0 + 2 * bb;
                    const int ty = (jb + j) % Ty, tx = (ib + i) % Tx;
                    const uint32_t tile =
                        static_cast<uint32_t>(ty) * static_cast<uint32_t>(Tx) + static_cast<uint32_t>(tx);
                    const uint4 w = philox(tile, static_cast<uint32_t>(mcs), c2, 0u, k0, k1);
                    tile_attempts<ARITY>(win, (2 * j - rp.oy) * P + (2 * i - rp.ox), P, w, R, sT, S1, k0, k1, tile,
                                         mcs, p);
                    bb += db;
                    aa += da;
                    if (bb >= ni) {
                        bb -= ni;
                        ++aa;
                    }
                }
            }
            __syncthreads();
        }
        {
            const int wpr = bw >> 2;
            for (int idx = tid; idx < bh * wpr; idx += nt) {
                const int y = idx / wpr, c = idx - (idx / wpr) * wpr;
                __stcg(reinterpret_cast<unsigned int*>(dst + static_cast<size_t>(ry0 + y) * L + rx0 + 4 * c),
                       *reinterpret_cast<const uint32_t*>(win + (M + y) * P + M + 4 * c));
            }
        }
    }
    if (a.count) {
        for (int v = tid; v < S1; v += nt) sCnt[v] = 0;
        __syncthreads();
        if (a.step)
            block_count(win + M * P + M, bh, bw, P, S1, sCnt);
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
            for (int v = 0; v < S1; ++v) {
                c64[v] = atomicExch(&a.acc[r * S1 + v], 0ull);
            }
            a.ticket[r] = 0u;
            record_decide(c64, S1, a.mcs + a.step, r, a.run);
        }
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
        const uint64_t seed = a.seeds[r];
        const uint4 w = philox(static_cast<uint32_t>(pi), 0u, ctr2(0, kDomInit, 0u), 0u, static_cast<uint32_t>(seed),
                               static_cast<uint32_t>(seed >> 32));
        const uint32_t S = static_cast<uint32_t>(a.S);
        for (int h = 0; h < 2; ++h) {
            const int64_t i = 2 * pi + h;
            if (i >= a.n) break;
            const uint32_t we = h ? w.z : w.x, ws = h ? w.w : w.y;
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
    const Rule R{a.rule.xm, a.rule.xi, a.rule.xm >> Bits<4>::LB, a.rule.xi >> Bits<4>::LB};
    const int S1 = a.S + 1;
    for (int64_t k = 0; k < a.n_attempts; ++k) {
        const uint32_t cell = a.wc[k] % n;
        const uint32_t d = a.wd[k] % static_cast<uint32_t>(a.arity);
        const uint32_t word = a.wa[k];
        int dr, dc;
        dir_rc<8>(d, dr, dc);
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
        const uint32_t s = a.lat[cell], nb = a.lat[ni];
        uint32_t ns, nn;
        // The refine functor returns the word's own low bits: every comparison sees the full word.
        apply_rule<4>(s, nb, word, R, a.rule.T, S1, ns, nn, [&]() { return word & ((1u << Bits<4>::LB) - 1u); });
        a.lat[cell] = static_cast<uint8_t>(ns);
        a.lat[ni] = static_cast<uint8_t>(nn);
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
    const int P = align16(L + kTileC0 + 1);
    if (pitch) *pitch = P;
    return tile_layout(H, L, S, P).total;
}

int max_smem_optin(int device) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    return v;
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

template <int ARITY, bool REFLECT>
static cudaError_t tile_launch_t(const TileArgs& a, int nrep, int threads, cudaStream_t s) {
    auto k = tile_kernel<ARITY, REFLECT>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
    if (e != cudaSuccess) return e;
    k<<<nrep, threads, a.smem_bytes, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_tile(const TileArgs& a, int nrep, int threads, cudaStream_t s) {
    if (a.arity == 8) return a.flux ? tile_launch_t<8, false>(a, nrep, threads, s) : tile_launch_t<8, true>(a, nrep, threads, s);
    return a.flux ? tile_launch_t<4, false>(a, nrep, threads, s) : tile_launch_t<4, true>(a, nrep, threads, s);
}

template <int ARITY>
static cudaError_t block_launch_t(const BlockArgs& a, int nrep, int threads, cudaStream_t s) {
    static int configured_bytes = -1;
    auto k = block_kernel<ARITY>;
    if (configured_bytes < a.smem_bytes) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.smem_bytes);
        if (e != cudaSuccess) return e;
        configured_bytes = a.smem_bytes;
    }
    dim3 grid(static_cast<unsigned>(a.nbx), static_cast<unsigned>(a.nby), static_cast<unsigned>(nrep));
    k<<<grid, threads, a.smem_bytes, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_block(const BlockArgs& a, int nrep, int threads, cudaStream_t s) {
    return a.arity == 8 ? block_launch_t<8>(a, nrep, threads, s) : block_launch_t<4>(a, nrep, threads, s);
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
