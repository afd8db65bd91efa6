// ring.cu — persistent bit-sliced row-band kernel (draw format SLICED).
//
// The bit-sliced update of slice.cu — the same bit planes, the same draws, the same exact replay of
// undecided tiles, so oracle/escg_oracle.c orc_crs_run (fmt = 2 | K << 8) defines it too — without
// the overlapped-tile margins that make slice.cu recompute 1.6x the lattice at L=3200.
//
//   bands    one co-resident CTA (cooperative launch) per band [R0, R1) of full-width rows
//            (L/128 <= 32 groups: lane = group, the row wraps through the lane shuffles); the band
//            plus one halo row above and two below stay in shared memory for the whole launch.
//   slabs    in a colour phase the footprints of one tile row (anchor row w) cover exactly the rows
//            [w-1, w+2] of every column, and the tile rows of a phase are 4 rows apart: the slabs
//            partition the rows, so every row is written by exactly one CTA per phase.  A CTA
//            processes the slabs anchored in its band, one warp per slab (engine.hpp:108-141 per
//            tile, bit-parallel as in slice.cu).  Undecided tiles are replayed with the exact rule
//            by their own lane on the footprint words it holds in registers (bit l of each word is
//            tile l's cell), before the words are stored: no queue, no second pass.
//   exchange the rows a band shares with a neighbour are {R-1, R, R+1} at each boundary R; only the
//            first and the last slab of a band reach them.  After the phase the warp that wrote a
//            part of them publishes it as 64-bit words {data, phase tag} in the band's L2 mailbox;
//            the neighbour's boundary warp imports it before its next slab, polling the tags (a
//            tagged word is its own valid flag: no fence, no flag round trip).  A header word is
//            published every phase, so a side that imports nothing still waits for its neighbour —
//            bands never drift more than one phase apart, which is what makes the two mailbox
//            parities enough.  Interior warps never wait.
//   draws    the boundary slabs are the critical path of a phase, so two otherwise idle warps draw
//            the next phase's boundary slabs (the draws depend only on seed, MCS, phase and tile)
//            into shared memory while the current phase runs.
//   records  at a record MCS each warp writes its last-phase slab rows (final values, each row
//            exactly once over the grid) to a snapshot plane buffer and counts them; the last CTA
//            runs record_and_check (engine.cpp:47-57).  A CTA reaching record k first waits for
//            the decision of record k-1 and stops there if the run ended (the lattice of a stop is
//            that record's snapshot).
//   parts    (ring_kernel<..., PARTS = true>, advance only) the lattice split into parts, one launch
//            per part (one GPU each) or one launch over all parts: a part's first and last bands
//            exchange with the neighbouring part's through tagged system-scope stores into that
//            part's inbox (two sets, alternate launches), write their final rows into its planes as
//            well and flag them for its next launch; every cross-part wait is bounded
//            (kStatusRingTimeout).  DESIGN.md §7.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <type_traits>

#include "crs.cuh"
#include "launch.h"
#include "record.cuh"
#include "slice_common.cuh"

namespace escgd {
namespace {

constexpr int kRingWarps = kRingThreads / 32;
constexpr int kDrawWords = 20;  // per lane and slab: U[4], Y[4], X[4], D0[4], D1[4]

#ifdef ESCG_DIAG_RING
// diagnostic builds only (tools/ring_diag.py): per CTA, phase (32 from launch phase 800) and warp,
// clock64 at events 0-7; import poll rounds per CTA, phase and boundary warp
constexpr int kRingDiagQ0 = 800;
__device__ long long g_rdiag[160][32][8][8];
__device__ int g_rpoll[160][32][2];
#define RDIAG(q, ev, val)                                                                                   \
    do {                                                                                                   \
        const int qq_ = static_cast<int>(q) - kRingDiagQ0;                                                  \
        if (qq_ >= 0 && qq_ < 32 && (threadIdx.x & 31) == 0 && blockIdx.x < 160)                           \
            g_rdiag[blockIdx.x][qq_][threadIdx.x >> 5][ev] = (val);                                          \
    } while (0)
#else
#define RDIAG(q, ev, val)
#endif

__device__ __forceinline__ void st_tag2(unsigned long long* p, uint32_t a, uint32_t b, uint32_t tag) {
    const unsigned long long x = (static_cast<unsigned long long>(tag) << 32) | a;
    const unsigned long long y = (static_cast<unsigned long long>(tag) << 32) | b;
    asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_tag2(const unsigned long long* p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}
// the same between parts of a multi-part ring (the words cross NVLink: system scope)
__device__ __forceinline__ void st_tag2_sys(unsigned long long* p, uint32_t a, uint32_t b, uint32_t tag) {
    const unsigned long long x = (static_cast<unsigned long long>(tag) << 32) | a;
    const unsigned long long y = (static_cast<unsigned long long>(tag) << 32) | b;
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ ulonglong2 ld_tag2_sys(const unsigned long long* p) {
    ulonglong2 v;
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t tag_of(unsigned long long x) { return static_cast<uint32_t>(x >> 32); }
__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

struct RingCtx {
    uint32_t* sw;  // window [band + 3][RP]: window row y = global row R0 - 1 + y
    int RP, GL, H, Hh, R0, R1, c, nb;
    int lL, lR;  // lanes holding the left / right neighbour group (the row wraps)
    uint32_t s32, xm, xi, TK, sT;
    int S1;
    unsigned long long* mbox;
    int mbs;
    const uint32_t* T3;   // SLICED3 thresholds T, S in shared memory, null: SLICED
    const uint32_t* T3g;  // the whole SLICED3 table (global)
    // multi-part ring: this band's part (shared memory), its rows, the launch's inbox set
    const RingPart* P;    // null: single-device ring (the lattice wraps inside this launch)
    int pr0, prows, xset, cur;
    int32_t* status;          // multi-part ring: kStatusRingTimeout once any wait gave up
    unsigned long long t0;    // launch start (global timer, ns)
    unsigned long long budget;  // ns a multi-part wait may take
};

// Multi-part ring waits are bounded: past the budget (or once another CTA gave up) a wait
// returns, the launch runs out with junk rows and the status tells the host.  Checked every 64
// polls (each poll is an L2 or NVLink round trip anyway).
__device__ __forceinline__ bool ring_expired(const RingCtx& C, unsigned& polls) {
    if ((++polls & 63u) != 0u) return false;
    if (*reinterpret_cast<volatile const int32_t*>(C.status) == kStatusRingTimeout) return true;
    if (global_ns() - C.t0 > C.budget) {
        atomicExch(C.status, kStatusRingTimeout);
        return true;
    }
    return false;
}

// Inbox (set, side: 0 rows from the part above, 1 from below, parity) of a part, and its flags
// (the neighbour's final boundary rows of the previous launch are in this part's planes).
__device__ __forceinline__ unsigned long long* inbox_slot(unsigned long long* base, int set, int side, int par,
                                                          int mbs) {
    return base + static_cast<size_t>((set * 2 + side) * 2 + par) * static_cast<size_t>(mbs);
}
__device__ __forceinline__ unsigned long long* inbox_flag(unsigned long long* base, int set, int side, int mbs) {
    return base + static_cast<size_t>(8) * static_cast<size_t>(mbs) + set * 2 + side;
}

// Mailbox of band `cta`, direction dir (0: rows shared with the band above, 1: below), parity par.
__device__ __forceinline__ unsigned long long* mailbox(const RingCtx& C, int cta, int dir, int par) {
    return C.mbox + static_cast<size_t>((cta * 2 + dir) * 2 + par) * static_cast<size_t>(C.mbs);
}
// words 0-1: header; (shared row s in 0..2, plane p, group g, quad k) at 2 + ((s NPL + p) GL + g) 4 + k
template <int NPL>
__device__ __forceinline__ int mslot(const RingCtx& C, int s, int p, int g) {
    return 2 + ((s * NPL + p) * C.GL + g) * 4;
}

// Publish shared rows s_lo..s_hi (window rows wrow0 + s) into this band's mailbox, then the header.
template <int NPL, bool PARTS>
__device__ __forceinline__ void ring_publish(const RingCtx& C, int dir, int wrow0, int s_lo, int s_hi, int par,
                                             uint32_t tag) {
    const int lane = threadIdx.x & 31;
    // the band above / below in another part: into that part's inbox (peer memory)
    const bool cross = PARTS && (dir == 0 ? C.c == 0 : C.c == C.nb - 1);
    unsigned long long* mb =
        !cross ? mailbox(C, C.c, dir, par)
               : (dir == 0 ? inbox_slot(C.P->up_inbox, C.xset, 1, par, C.mbs) : inbox_slot(C.P->dn_inbox, C.xset, 0, par, C.mbs));
    if (lane < C.GL) {
        for (int s = s_lo; s <= s_hi; ++s) {
#pragma unroll
            for (int p = 0; p < NPL; ++p) {
                const uint4 v = lds128(C.sw + (wrow0 + s) * C.RP + (p * C.GL + lane) * 4);
                unsigned long long* d = mb + mslot<NPL>(C, s, p, lane);
                ESCG_CHECK(s >= 0 && s < 3 && mslot<NPL>(C, s, p, lane) + 3 < C.mbs && wrow0 + s <= C.R1 - C.R0 + 2);
                if (cross) {
                    st_tag2_sys(d, v.x, v.y, tag);
                    st_tag2_sys(d + 2, v.z, v.w, tag);
                } else {
                    st_tag2(d, v.x, v.y, tag);
                    st_tag2(d + 2, v.z, v.w, tag);
                }
            }
        }
    }
    if (lane == 0) {  // header: this band finished the phase
        if (cross)
            st_tag2_sys(mb, 0u, 0u, tag);
        else
            st_tag2(mb, 0u, 0u, tag);
    }
}

// Import the neighbour's shared rows s_lo..s_hi of the previous phase (tag) into window rows
// wrow0 + s; with nothing to import, wait for its header.  Polls until every word carries the tag.
template <int NPL, bool PARTS>
__device__ __forceinline__ void ring_import(const RingCtx& C, int src, int dir, int wrow0, int s_lo, int s_hi, int par,
                                         uint32_t tag, int diag_q) {
    const int lane = threadIdx.x & 31;
    const bool cross = PARTS && (dir == 1 ? C.c == 0 : C.c == C.nb - 1);
    const unsigned long long* mb =
        cross ? inbox_slot(C.P->inbox, C.xset, dir == 1 ? 0 : 1, par, C.mbs) : mailbox(C, src, dir, par);
    unsigned polls = 0;
    if (s_lo > s_hi) {
        if (lane == 0)
            while (tag_of((cross ? ld_tag2_sys(mb) : ld_tag2(mb)).x) != tag) {
                if constexpr (PARTS)
                    if (cross && ring_expired(C, polls)) break;
            }
        __syncwarp();
        return;
    }
    if (lane < C.GL) {
        uint32_t pend = 0;
        for (int s = s_lo; s <= s_hi; ++s)
            for (int p = 0; p < NPL; ++p) pend |= 1u << (s * NPL + p);
#ifdef ESCG_DIAG_RING
        int rounds = 0;
#endif
        while (pend) {
#ifdef ESCG_DIAG_RING
            ++rounds;
#endif
            if constexpr (PARTS)
                if (cross && ring_expired(C, polls)) break;
            ulonglong2 v[3 * NPL][2];
#pragma unroll
            for (int e = 0; e < 3 * NPL; ++e)
                if ((pend >> e) & 1u) {
                    const unsigned long long* a = mb + mslot<NPL>(C, e / NPL, e % NPL, lane);
                    if (cross) {
                        v[e][0] = ld_tag2_sys(a);
                        v[e][1] = ld_tag2_sys(a + 2);
                    } else {
                        v[e][0] = ld_tag2(a);
                        v[e][1] = ld_tag2(a + 2);
                    }
                }
#pragma unroll
            for (int e = 0; e < 3 * NPL; ++e)
                if ((pend >> e) & 1u) {
                    if (tag_of(v[e][0].x) == tag && tag_of(v[e][0].y) == tag && tag_of(v[e][1].x) == tag &&
                        tag_of(v[e][1].y) == tag) {
                        const int s = e / NPL, p = e % NPL;
                        sts128(C.sw + (wrow0 + s) * C.RP + (p * C.GL + lane) * 4,
                               make_uint4(static_cast<uint32_t>(v[e][0].x), static_cast<uint32_t>(v[e][0].y),
                                          static_cast<uint32_t>(v[e][1].x), static_cast<uint32_t>(v[e][1].y)));
                        pend &= ~(1u << e);
                    }
                }
        }
#ifdef ESCG_DIAG_RING
        if (lane == 0 && blockIdx.x < 160 && diag_q >= 0 && diag_q < 32) g_rpoll[blockIdx.x][diag_q][dir] = rounds;
#endif
    }
    __syncwarp();
}

// footprint word at column offset DX of a row (slice.cu fetch/put with explicit, wrapping lanes)
template <int XR, int DX>
__device__ __forceinline__ uint32_t rfetch(const uint32_t (&q4)[4], int lL, int lR) {
    constexpr int t = XR + DX, q = t & 3, s = t < 0 ? -1 : (t >> 2);
    if constexpr (s == 0) {
        return q4[q];
    } else if constexpr (s < 0) {
        const uint32_t l = __shfl_sync(kFull, q4[3], lL);
        return __funnelshift_l(l, q4[3], 1);
    } else {
        const uint32_t r = __shfl_sync(kFull, q4[q], lR);
        return __funnelshift_r(q4[q], r, 1);
    }
}
template <int XR, int DX>
__device__ __forceinline__ void rput(uint32_t (&q4)[4], uint32_t f, int lL, int lR) {
    constexpr int t = XR + DX, q = t & 3, s = t < 0 ? -1 : (t >> 2);
    if constexpr (s == 0) {
        q4[q] = f;
    } else if constexpr (s < 0) {
        const uint32_t r = __shfl_sync(kFull, f, lR);
        q4[3] = __funnelshift_r(f, r, 1);
    } else {
        const uint32_t l = __shfl_sync(kFull, f, lL);
        q4[q] = __funnelshift_l(l, f, 1);
    }
}

// All 12 footprint words of a slab item from its 4 rows of quad words (and back), for anchor
// column residue XR; the kernel switches on XR once per slab, so only these shuffle patterns are
// instantiated four times (a compact kernel keeps the phase loop in the instruction cache).
template <int NPL, int XR>
__device__ __forceinline__ void fetch_all(const uint32_t (&Q)[4][NPL][4], uint32_t (&F)[4][4][NPL], int lL, int lR) {
#define ESCG_RFET(rr, c) \
    _Pragma("unroll") for (int p = 0; p < NPL; ++p) F[rr][c][p] = rfetch<XR, (c)-1>(Q[rr][p], lL, lR);
    ESCG_RFET(0, 1) ESCG_RFET(0, 2)
    ESCG_RFET(1, 0) ESCG_RFET(1, 1) ESCG_RFET(1, 2) ESCG_RFET(1, 3)
    ESCG_RFET(2, 0) ESCG_RFET(2, 1) ESCG_RFET(2, 2) ESCG_RFET(2, 3)
    ESCG_RFET(3, 1) ESCG_RFET(3, 2)
#undef ESCG_RFET
}
template <int NPL, int XR>
__device__ __forceinline__ void put_all(uint32_t (&Q)[4][NPL][4], const uint32_t (&F)[4][4][NPL], int lL, int lR) {
#define ESCG_RPUT(rr, c) \
    _Pragma("unroll") for (int p = 0; p < NPL; ++p) rput<XR, (c)-1>(Q[rr][p], F[rr][c][p], lL, lR);
    ESCG_RPUT(0, 1) ESCG_RPUT(0, 2)
    ESCG_RPUT(1, 0) ESCG_RPUT(1, 1) ESCG_RPUT(1, 2) ESCG_RPUT(1, 3)
    ESCG_RPUT(2, 0) ESCG_RPUT(2, 1) ESCG_RPUT(2, 2) ESCG_RPUT(2, 3)
    ESCG_RPUT(3, 1) ESCG_RPUT(3, 2)
#undef ESCG_RPUT
}

// The SLICED draws of one item (slice.cu slice_phase, LPI = 1): K action words AND-ed into the
// undecided masks U, then the choice planes (cell row, cell column, direction bits) per attempt.
template <int K>
__device__ __forceinline__ void slab_draws(uint32_t item, uint32_t c1, uint32_t c2s, uint32_t s32, const uint32_t* T3,
                                           const uint32_t* T3g, uint32_t (&D)[kDrawWords]) {
    if (T3 != nullptr) {  // SLICED3: the undecided masks drawn directly (slice_common.cuh)
        uint32_t U[4];
        slice3_masks(item, c1, c2s, s32, T3, T3g, U);
#pragma unroll
        for (int a = 0; a < 4; ++a) D[a] = U[a];
    } else {
#pragma unroll
        for (int a = 0; a < 4; ++a) D[a] = ~0u;
#pragma unroll
        for (int jj = 0; jj < K; ++jj) {
            const uint4 v = philox(item, c1, c2s | (static_cast<uint32_t>(4 + jj) << 24), s32);
            const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) D[(4 * jj + c) / K] &= vw[c];
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint4 v = philox(item, c1, c2s | (static_cast<uint32_t>(a) << 24), s32);
        D[4 + a] = v.x;
        D[8 + a] = v.y;
        D[12 + a] = v.z;
        D[16 + a] = v.w;
    }
}

// The draws of one slab item into shared memory ([word][lane]); out of line so the kernel holds a
// single copy of the Philox code.
template <int K>
__device__ __noinline__ void draws_to_smem(uint32_t item, uint32_t c1, uint32_t c2s, uint32_t s32, const uint32_t* T3,
                                           const uint32_t* T3g, uint32_t* t) {
    uint32_t D[kDrawWords];
    slab_draws<K>(item, c1, c2s, s32, T3, T3g, D);
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int i = 0; i < kDrawWords; ++i) t[i * 32 + lane] = D[i];
}

// Exact replay (engine.hpp:108-141) of tile l's four attempts on its 12 footprint cells, read from
// and written back to bit l of the footprint words F (the tile took no part in the bit-parallel
// pass; no other tile's footprint overlaps it).  Positions k as in slice_replay_group.
template <int NPL>
__device__ __forceinline__ void tile_replay_regs(uint32_t (&F)[4][4][NPL], int l, uint32_t code, const uint4 rf,
                                                 const RingCtx& C) {
    constexpr int CB = NPL == 2 ? 2 : 3;  // bits per packed cell
    using Pack = typename std::conditional<NPL == 2, uint32_t, uint64_t>::type;
    constexpr uint32_t kCellPos = 0x8473u;
    constexpr uint64_t kNbrPos = 0x95847362b8a74130ull;
    constexpr int kR[12] = {0, 0, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3};
    constexpr int kC[12] = {1, 2, 0, 1, 2, 3, 0, 1, 2, 3, 1, 2};
    Pack cells = 0;
#pragma unroll
    for (int k = 0; k < 12; ++k)
#pragma unroll
        for (int p = 0; p < NPL; ++p) cells |= static_cast<Pack>((F[kR[k]][kC[k]][p] >> l) & 1u) << (CB * k + p);
    const Pack cells0 = cells;
    const uint32_t rw[4] = {rf.x, rf.y, rf.z, rf.w};
    constexpr Pack M = (static_cast<Pack>(1) << CB) - 1;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t cb = (code >> (4 * a)) & 15u;
        const uint32_t ps = (kCellPos >> (4 * (cb & 3u))) & 15u, pn = static_cast<uint32_t>(kNbrPos >> (4 * cb)) & 15u;
        const uint32_t s = static_cast<uint32_t>(cells >> (CB * ps)) & M, n = static_cast<uint32_t>(cells >> (CB * pn)) & M;
        const bool und = (code >> (16 + a)) & 1u;
        const uint32_t x = C.TK | (rw[a] & ~C.TK);
        const bool mig = !und || x < C.xm, rep = und && x >= C.xi;
        const bool inter = !mig && !rep && s != 0u && n != 0u && s != n;
        const uint32_t t1 = lds32_if(inter, C.sT + 4u * (s * C.S1 + n), 0u);
        const uint32_t t2 = lds32_if(inter, C.sT + 4u * (n * C.S1 + s), 0u);
        const bool kn = inter && x < t1, ks = inter && !(x < t1) && x < t2;
        const bool r1 = rep && n == 0u, r2 = rep && n != 0u && s == 0u;
        const uint32_t ns = mig ? n : (ks ? 0u : (r2 ? n : s));
        const uint32_t nn = mig ? s : (kn ? 0u : (r1 ? s : n));
        cells = (cells & ~((M << (CB * ps)) | (M << (CB * pn)))) | (static_cast<Pack>(ns) << (CB * ps)) |
                (static_cast<Pack>(nn) << (CB * pn));
    }
    const Pack delta = cells ^ cells0;
#pragma unroll
    for (int k = 0; k < 12; ++k)
#pragma unroll
        for (int p = 0; p < NPL; ++p) F[kR[k]][kC[k]][p] ^= static_cast<uint32_t>((delta >> (CB * k + p)) & 1u) << l;
}

struct Exchange {  // one boundary warp's import before / publish after its slab
    int imp, src, idir, iwrow0, is_lo, is_hi, ipar;
    uint32_t itag;
    int pub, pdir, pwrow0, ps_lo, ps_hi, ppar;
    uint32_t ptag;
    uint32_t q;  // launch phase (diagnostics)
};

// One slab: the tile row anchored at global row w (every group, anchor column residue XR), by one
// warp.  tbl: this slab's draws precomputed in shared memory ([word][lane]), or null.
// dst: write the slab's rows there afterwards (and count them into cnt when `count`).
template <int NPL, int K, bool PARTS>
__device__ __forceinline__ void ring_slab(const RingCtx& C, int w, int oy, int xr, uint32_t c1, uint32_t c2s,
                                          uint32_t c2r, const Exchange& X, const uint32_t* tbl, uint32_t* scratch,
                                          uint32_t* dst, bool count, uint32_t (&cnt)[1 << NPL]) {
    const int lane = threadIdx.x & 31;
    const bool valid = lane < C.GL;
    const int wl = w - C.R0 + 1;  // window row of the anchor
    ESCG_CHECK(wl >= 1 && wl + 2 <= C.R1 - C.R0 + 2 && C.GL <= 32);
    int j = (w + oy) >> 1;
    j = j >= C.Hh ? j - C.Hh : j;
    const uint32_t item = static_cast<uint32_t>(j) * static_cast<uint32_t>(C.GL) + static_cast<uint32_t>(lane);
    RDIAG(X.q, 0, clock64());

    if (tbl == nullptr) {  // not drawn ahead by a producer warp: draw now (this warp's scratch)
        draws_to_smem<K>(item, c1, c2s, C.s32, C.T3, C.T3g, scratch);
        __syncwarp();
        tbl = scratch;
    }
    RDIAG(X.q, 1, clock64());
    // the draws do not depend on the lattice: the neighbour's rows are awaited only now (before the
    // draw words are loaded, so that few registers are live while polling)
    if (X.imp) ring_import<NPL, PARTS>(C, X.src, X.idir, X.iwrow0, X.is_lo, X.is_hi, X.ipar, X.itag,
                                   static_cast<int>(X.q) - 800);
    RDIAG(X.q, 2, clock64());
    uint32_t D[kDrawWords];
#pragma unroll
    for (int i = 0; i < kDrawWords; ++i) D[i] = tbl[i * 32 + lane];
    const uint32_t Dm = valid ? (D[0] | D[1] | D[2] | D[3]) : 0u;
    const uint32_t act = ~Dm;
    // the exact low action bits of the lane's first undecided tile, drawn ahead of the footprint
    // loads and the bit-parallel pass (its Philox latency would otherwise open the replay)
    uint4 rf0 = make_uint4(0u, 0u, 0u, 0u);
    if (Dm != 0u) rf0 = philox(item, c1, c2r | (static_cast<uint32_t>(__ffs(Dm) - 1) << 24), C.s32);

    uint32_t Q[4][NPL][4];
    uint32_t* rowp = C.sw + (wl - 1) * C.RP + lane * 4;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) {
#pragma unroll
        for (int p = 0; p < NPL; ++p) {
            uint4 t = make_uint4(0u, 0u, 0u, 0u);
            if (valid) t = lds128(rowp + rr * C.RP + p * C.GL * 4);
            Q[rr][p][0] = t.x;
            Q[rr][p][1] = t.y;
            Q[rr][p][2] = t.z;
            Q[rr][p][3] = t.w;
        }
    }
    uint32_t F[4][4][NPL];
    switch (xr) {
        case 0: fetch_all<NPL, 0>(Q, F, C.lL, C.lR); break;
        case 1: fetch_all<NPL, 1>(Q, F, C.lL, C.lR); break;
        case 2: fetch_all<NPL, 2>(Q, F, C.lL, C.lR); break;
        default: fetch_all<NPL, 3>(Q, F, C.lL, C.lR); break;
    }

#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t y = D[4 + a], x = D[8 + a], d0 = D[12 + a], d1 = D[16 + a];
        // direction 0 up, 1 down, 2 left, 3 right (params.hpp:81); masked exchanges (slice.cu)
        const uint32_t up = act & ~(d1 | d0), dn = act & ~d1 & d0, lf = act & d1 & ~d0, rt = act & d1 & d0;
        const uint32_t ny = ~y, nx = ~x;
        const uint32_t vm = (ny & dn) | (y & up);
        const uint32_t hm = (nx & rt) | (x & lf);
        const uint32_t mV0[2] = {ny & nx & up, ny & x & up};
        const uint32_t mV1[2] = {nx & vm, x & vm};
        const uint32_t mV2[2] = {y & nx & dn, y & x & dn};
        const uint32_t mH[2][3] = {{ny & nx & lf, ny & hm, ny & x & rt}, {y & nx & lf, y & hm, y & x & rt}};
#pragma unroll
        for (int p = 0; p < NPL; ++p) {
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
    RDIAG(X.q, 3, clock64() + (F[1][1][0] == 0x12345u));
    // undecided tiles (rare: ~4 per 1024 tile-phases at P(migration) 0.999): their four attempts,
    // exactly, by the owning lane on its registers (the order among disjoint tiles is immaterial)
    for (uint32_t dm = Dm; dm != 0u; dm &= dm - 1u) {
        const int l = __ffs(dm) - 1;
        uint32_t code = 0;
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            code |= (((D[4 + a] >> l) & 1u) | (((D[8 + a] >> l) & 1u) << 1) | (((D[12 + a] >> l) & 1u) << 2) |
                     (((D[16 + a] >> l) & 1u) << 3))
                    << (4 * a);
            code |= ((D[a] >> l) & 1u) << (16 + a);
        }
        const uint4 rf = dm == Dm ? rf0 : philox(item, c1, c2r | (static_cast<uint32_t>(l) << 24), C.s32);
        tile_replay_regs<NPL>(F, l, code, rf, C);
    }
    RDIAG(X.q, 4, clock64() + (F[1][1][0] == 0x12345u));
    switch (xr) {
        case 0: put_all<NPL, 0>(Q, F, C.lL, C.lR); break;
        case 1: put_all<NPL, 1>(Q, F, C.lL, C.lR); break;
        case 2: put_all<NPL, 2>(Q, F, C.lL, C.lR); break;
        default: put_all<NPL, 3>(Q, F, C.lL, C.lR); break;
    }
    if (valid) {
#pragma unroll
        for (int rr = 0; rr < 4; ++rr)
#pragma unroll
            for (int p = 0; p < NPL; ++p)
                sts128(rowp + rr * C.RP + p * C.GL * 4, make_uint4(Q[rr][p][0], Q[rr][p][1], Q[rr][p][2], Q[rr][p][3]));
    }
    __syncwarp();
    RDIAG(X.q, 5, clock64());

    if (X.pub) ring_publish<NPL, PARTS>(C, X.pdir, X.pwrow0, X.ps_lo, X.ps_hi, X.ppar, X.ptag);
    if (dst != nullptr && valid) {
        // the slab's rows are final for this phase: snapshot (global rows w-1 .. w+2) and count
#pragma unroll
        for (int rr = 0; rr < 4; ++rr) {
            int gy = w - 1 + rr;
            if constexpr (PARTS) {
                // multi-part ring: local row of this part's planes; rows within one of a part
                // boundary go to the neighbour's planes as well (it reads them at its next launch)
                ESCG_CHECK(gy - C.pr0 + 2 >= 1 && gy - C.pr0 + 2 < C.prows + 4);
#pragma unroll
                for (int p = 0; p < NPL; ++p) {
                    const uint4 v = make_uint4(Q[rr][p][0], Q[rr][p][1], Q[rr][p][2], Q[rr][p][3]);
                    const size_t col = static_cast<size_t>(p * C.GL + lane) * 4;
                    const size_t rw = static_cast<size_t>(NPL) * C.GL * 4;
                    __stcg(reinterpret_cast<uint4*>(dst + static_cast<size_t>(gy - C.pr0 + 2) * rw + col), v);
                    if (C.c == 0 && gy <= C.pr0 + 1)
                        __stcg(reinterpret_cast<uint4*>(C.P->up_pl[C.cur ^ 1] +
                                                         static_cast<size_t>(gy - C.pr0 + C.P->up_rows + 2) * rw + col), v);
                    if (C.c == C.nb - 1 && gy >= C.pr0 + C.prows - 1)
                        __stcg(reinterpret_cast<uint4*>(C.P->dn_pl[C.cur ^ 1] +
                                                         static_cast<size_t>(gy - C.pr0 - C.prows + 2) * rw + col), v);
                }
                continue;
            }
            gy = gy < 0 ? gy + C.H : (gy >= C.H ? gy - C.H : gy);
            ESCG_CHECK(gy >= 0 && gy < C.H);
#pragma unroll
            for (int p = 0; p < NPL; ++p)
                __stcg(reinterpret_cast<uint4*>(dst + ((static_cast<size_t>(gy) * NPL + p) * C.GL + lane) * 4),
                       make_uint4(Q[rr][p][0], Q[rr][p][1], Q[rr][p][2], Q[rr][p][3]));
            if (count) {
#pragma unroll
                for (int v = 1; v < (1 << NPL); ++v) {
                    uint32_t n = 0;
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        uint32_t m = ~0u;
#pragma unroll
                        for (int p = 0; p < NPL; ++p) m &= ((v >> p) & 1) ? Q[rr][p][k] : ~Q[rr][p][k];
                        n += __popc(m);
                    }
                    cnt[v] += n;
                }
            }
        }
    }
    RDIAG(X.q, 6, clock64());
}

// Geometry of one colour phase in a band: tile residues and the slab anchors.
struct PhaseGeo {
    int oy, yr, xr, w0, ns;
};
__device__ __forceinline__ PhaseGeo phase_geo(const Round& rp, int p, int R0, int R1) {
    PhaseGeo g;
    const int cy = rp.colour(p) >> 1, cx = rp.colour(p) & 1;
    g.oy = rp.oy;
    g.yr = (2 * cy - rp.oy) & 3;
    g.xr = (2 * cx - rp.ox) & 3;
    g.w0 = R0 + ((g.yr - R0) & 3);   // first anchor row of the band
    g.ns = (R1 - 1 - g.w0) / 4 + 1;  // slabs (>= 2: bands have >= 8 rows)
    return g;
}

template <int NPL, int K, bool PARTS>
__global__ void __launch_bounds__(kRingThreads, 1) ring_kernel(RingArgs a) {
    extern __shared__ __align__(16) uint32_t sw[];
    __shared__ uint32_t sTh[(kMaxSliceSpecies + 1) * (kMaxSliceSpecies + 1)];
    __shared__ uint32_t sDraw[2][2][kDrawWords * 32];  // [phase parity][top, bottom slab][word][lane]
    __shared__ uint32_t sScr[kRingWarps][kDrawWords * 32];  // slab warps' own draws
    __shared__ uint32_t sCnt[1 << NPL];
    __shared__ int sStop;
    __shared__ uint32_t sT3[64];
    __shared__ RingPart sPart;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int H = a.H, GL = a.L >> 7, S1 = a.S + 1;
    // multi-part ring: this CTA's part (by first CTA index) and its band within the part
    int pi = 0;
#pragma unroll
    for (int i = 1; i < kMaxRingParts; ++i)
        if (i < a.nparts && a.part[i].cta0 <= static_cast<int>(blockIdx.x)) pi = i;
    constexpr bool parts = PARTS;  // multi-part ring instantiation (a.nparts > 0)
    if (parts && tid == 0) {
#pragma unroll
        for (int i = 0; i < kMaxRingParts; ++i)
            if (i == pi) sPart = a.part[i];
    }
    __syncthreads();
    const int c = parts ? static_cast<int>(blockIdx.x) - sPart.cta0 : static_cast<int>(blockIdx.x);
    const int nb = parts ? sPart.nb : static_cast<int>(gridDim.x);
    const int pr0 = parts ? sPart.r0 : 0, prows = parts ? sPart.rows : H;
    const int R0 = pr0 + static_cast<int>(static_cast<int64_t>(c) * prows / nb);
    const int R1 = pr0 + static_cast<int>(static_cast<int64_t>(c + 1) * prows / nb);
    const int band = R1 - R0, RP = NPL * GL * 4, per_row = NPL * GL;
    if (tid < (1 << NPL)) sCnt[tid] = 0u;
    for (int i = tid; i < S1 * S1; i += nt) sTh[i] = a.rule.T[i];
    if (a.T3 != nullptr && tid < 64) sT3[tid] = a.T3[tid];
    if (*reinterpret_cast<volatile const int32_t*>(a.run.status) != kStatusRunning) return;  // uniform

    const unsigned long long t_start = global_ns();
    if (parts && a.wait_snap && tid == 0) {
        // the neighbour parts' last launch wrote the rows they finished in this part's range into
        // these planes; their flags (release, system scope) say those stores are visible
        RingCtx T{};
        T.status = a.run.status;
        T.t0 = t_start;
        T.budget = a.timeout_ns;
        unsigned polls = 0;
        if (c == 0)
            while (ld_acquire_sys_u64(inbox_flag(sPart.inbox, a.xset, 0, a.mbs)) != a.epoch)
                if (ring_expired(T, polls)) break;
        if (c == nb - 1)
            while (ld_acquire_sys_u64(inbox_flag(sPart.inbox, a.xset, 1, a.mbs)) != a.epoch)
                if (ring_expired(T, polls)) break;
    }
    __syncthreads();
    for (int idx = tid; idx < (band + 3) * per_row; idx += nt) {  // rows R0-1 .. R1+1 (mod H)
        const int y = idx / per_row, rem = idx - y * per_row;
        int gy = R0 - 1 + y;
        const uint32_t* src;
        if (parts) {
            // halo rows: after a ring launch the neighbours' final rows are already in these planes
            // (flagged above); after a host write they are read from the neighbours' own rows
            const uint32_t* base = sPart.pl[a.cur];
            int lr = gy - pr0 + 2;
            if (!a.wait_snap && gy < pr0) {
                base = sPart.up_pl[a.cur];
                lr = gy - pr0 + sPart.up_rows + 2;
            } else if (!a.wait_snap && gy >= pr0 + prows) {
                base = sPart.dn_pl[a.cur];
                lr = gy - pr0 - prows + 2;
            }
            src = base + (static_cast<size_t>(lr) * per_row + rem) * 4;
        } else {
            gy = gy < 0 ? gy + H : (gy >= H ? gy - H : gy);
            src = a.pin + (static_cast<size_t>(gy) * per_row + rem) * 4;
        }
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(src));
        sts128(sw + y * RP + rem * 4, v);
    }
    __syncthreads();

    RingCtx C;
    C.sw = sw;
    C.RP = RP;
    C.GL = GL;
    C.H = H;
    C.Hh = H >> 1;
    C.R0 = R0;
    C.R1 = R1;
    C.c = c;
    C.nb = nb;
    C.P = parts ? &sPart : nullptr;
    C.pr0 = pr0;
    C.prows = prows;
    C.xset = a.xset;
    C.cur = a.cur;
    C.status = a.run.status;
    C.t0 = t_start;
    C.budget = a.timeout_ns;
    C.lL = lane < GL ? (lane == 0 ? GL - 1 : lane - 1) : lane;
    C.lR = lane < GL ? (lane == GL - 1 ? 0 : lane + 1) : lane;
    C.s32 = seed32(a.seeds[0]);
    C.xm = a.rule.xm;
    C.xi = a.rule.xi;
    C.TK = ~0u << (32 - K);
    C.sT = smem_addr(sTh);
    C.S1 = S1;
    C.mbox = parts ? sPart.mbox : a.mbox;
    C.mbs = a.mbs;
    C.T3 = a.T3 != nullptr ? sT3 : nullptr;
    C.T3g = a.T3;
    const int up = c == 0 ? nb - 1 : c - 1, down = c == nb - 1 ? 0 : c + 1;
    const int64_t interval = a.run.interval > 0 ? a.run.interval : 1;
    // two warps beyond the most slabs a phase can have draw the next phase's boundary slabs
    const int ns_max = (band - 1) / 4 + 1;
    const bool pre = ns_max <= kRingWarps - 2;
    const int wtop = kRingWarps - 2, wbot = kRingWarps - 1;

    int dT_prev = 0, dB_prev = 0, rec_k = 0;
    uint32_t q = 0;  // phases executed in this launch (mailbox tags are q + 1)
    Round rp = round_params(C.s32, static_cast<uint64_t>(a.mcs0));
#pragma unroll 1
    for (int64_t m = a.mcs0; m < a.mcs_end; ++m) {
        const bool rec = a.record ? (((m + 1 - a.mcs0) % interval) == 0 || m + 1 == a.mcs_end) : false;
        const bool last = m + 1 == a.mcs_end;
        const Round rn = round_params(C.s32, static_cast<uint64_t>(m + 1));  // next MCS (producers)
#pragma unroll 1
        for (int p = 0; p < 4; ++p, ++q) {
            const PhaseGeo g = phase_geo(rp, p, R0, R1);
            const int ns = g.ns;
            const int dT = R0 + 3 - g.w0;                   // top shared rows: mine are slots 3-dT .. 2
            const int dB = R1 - 1 - (g.w0 + 4 * (ns - 1));  // bottom: mine are slots 0 .. 2-dB
            const uint32_t c1 = static_cast<uint32_t>(m);
            const uint32_t c2s = ctr2(static_cast<uint64_t>(m), kDomSlice, static_cast<uint32_t>(p), 0u);
            const uint32_t c2r = ctr2(static_cast<uint64_t>(m), kDomSliceRef, static_cast<uint32_t>(p), 0u);
            const bool snap = p == 3 && (a.record ? rec : last);
            if (snap && a.record && rec_k >= 1) {
                // record k = rec_k + 1 >= 2 overwrites the buffer of record k - 2 (the input for k = 2):
                // first the decision of record k - 1, taken after every band contributed to it
                if (tid == 0) {
                    while (ld_acquire_u32(a.decided) < static_cast<unsigned>(rec_k)) {
                    }
                    sStop = *reinterpret_cast<volatile const int32_t*>(a.run.status) != kStatusRunning;
                }
                __syncthreads();
                if (sStop) return;  // the run ended at record k - 1 (its snapshot is the lattice)
            }
            uint32_t* dst = snap ? (parts ? sPart.pl[a.cur ^ 1] : (a.record ? a.pbuf[(rec_k + 1) & 1] : a.pbuf[1]))
                                 : nullptr;
            // a multi-part ring does not publish its last phase: nothing would read it, and so no
            // store into a neighbour's inbox outlives the launch
            const int pub = !(parts && snap);
            uint32_t cnt[1 << NPL];
#pragma unroll
            for (int v = 0; v < (1 << NPL); ++v) cnt[v] = 0u;
            const int par = static_cast<int>(q & 1u);
            const bool have_tbl = pre && q > 0;
            if (warp < kRingWarps - 2 || !pre) {
#pragma unroll 1
                for (int s = warp == 0 ? 0 : (warp == 1 ? ns - 1 : 1 + (warp - 2)); s < ns;
                     s += (warp < 2 ? ns : kRingWarps - 2)) {
                    if (warp >= 2 && s >= ns - 1) break;
                    Exchange X{};
                    const uint32_t* tbl = nullptr;
                    if (s == 0 && warp == 0) {
                        X.imp = q > 0;  // the band above's part of the top rows from the last phase
                        X.src = up;
                        X.idir = 1;
                        X.iwrow0 = 0;
                        X.is_lo = 0;
                        X.is_hi = 2 - dT_prev;
                        X.ipar = par ^ 1;
                        X.itag = q;
                        X.pub = pub;
                        X.pdir = 0;
                        X.pwrow0 = 0;
                        X.ps_lo = 3 - dT;
                        X.ps_hi = 2;
                        X.ppar = par;
                        X.ptag = q + 1;
                        if (have_tbl) tbl = sDraw[par][0];
                    } else if (s == ns - 1 && warp == 1) {
                        X.imp = q > 0;
                        X.src = down;
                        X.idir = 0;
                        X.iwrow0 = band;
                        X.is_lo = 3 - dB_prev;
                        X.is_hi = 2;
                        X.ipar = par ^ 1;
                        X.itag = q;
                        X.pub = pub;
                        X.pdir = 1;
                        X.pwrow0 = band;
                        X.ps_lo = 0;
                        X.ps_hi = 2 - dB;
                        X.ppar = par;
                        X.ptag = q + 1;
                        if (have_tbl) tbl = sDraw[par][1];
                    }
                    X.q = q;
                    const int w = g.w0 + 4 * s;
                    const bool cp = snap && a.record;
                    ring_slab<NPL, K, PARTS>(C, w, g.oy, g.xr, c1, c2s, c2r, X, tbl, sScr[warp], dst, cp, cnt);
                    if (parts && snap && ((s == 0 && warp == 0 && c == 0) || (s == ns - 1 && warp == 1 && c == nb - 1))) {
                        // this band's final rows in the neighbour part's range are stored: flag them
                        // for the neighbour's next launch (its inbox set of that launch)
                        __threadfence_system();
                        __syncwarp();
                        if (lane == 0) {
                            __threadfence_system();
                            st_release_sys_u64(warp == 0 ? inbox_flag(sPart.up_inbox, a.xset ^ 1, 1, a.mbs)
                                                         : inbox_flag(sPart.dn_inbox, a.xset ^ 1, 0, a.mbs),
                                               static_cast<unsigned long long>(a.epoch) + 1ull);
                        }
                    }
                }
            } else if (!(p == 3 && last)) {
                // producer warps: the next phase's boundary slab draws (top: wtop, bottom: wbot)
                const Round& rq = p == 3 ? rn : rp;
                const int pn = (p + 1) & 3;
                const int64_t mn = p == 3 ? m + 1 : m;
                const PhaseGeo gn = phase_geo(rq, pn, R0, R1);
                const int w = warp == wtop ? gn.w0 : gn.w0 + 4 * (gn.ns - 1);
                int j = (w + gn.oy) >> 1;
                j = j >= C.Hh ? j - C.Hh : j;
                const uint32_t item = static_cast<uint32_t>(j) * static_cast<uint32_t>(GL) + static_cast<uint32_t>(lane);
                draws_to_smem<K>(item, static_cast<uint32_t>(mn),
                                 ctr2(static_cast<uint64_t>(mn), kDomSlice, static_cast<uint32_t>(pn), 0u), C.s32, C.T3, C.T3g,
                                 sDraw[par ^ 1][warp == wtop ? 0 : 1]);
            }
            if (snap && a.record) {
#pragma unroll
                for (int v = 1; v < (1 << NPL); ++v) {
                    const uint32_t tsum = __reduce_add_sync(kFull, cnt[v]);
                    if (lane == 0 && tsum) atomicAdd(&sCnt[v], tsum);
                }
            }
            dT_prev = dT;
            dB_prev = dB;
            __syncthreads();
            RDIAG(q, 7, clock64());
            if (snap && a.record) {
                ++rec_k;
                if (tid == 0) {
                    uint32_t nz = 0;
                    for (int v = 1; v < (1 << NPL); ++v) nz += sCnt[v];
                    sCnt[0] = static_cast<uint32_t>(4 * ns) * static_cast<uint32_t>(a.L) - nz;
                    for (int v = 0; v < S1; ++v)
                        if (sCnt[v]) atomicAdd(&a.acc[v], static_cast<unsigned long long>(sCnt[v]));
                    for (int v = 0; v < (1 << NPL); ++v) sCnt[v] = 0u;
                    __threadfence();
                    const unsigned tk = atomicAdd(a.ticket, 1u);
                    if (tk == static_cast<unsigned>(nb - 1)) {
                        __threadfence();
                        uint64_t c64[kMaxSpecies + 1];
                        for (int v = 0; v < S1; ++v) c64[v] = atomicExch(&a.acc[v], 0ull);
                        *a.ticket = 0u;
                        a.run.cur[0] = 2 + (rec_k & 1);
                        record_decide(c64, S1, m + 1, 0, a.run);
                        __threadfence();
                        atomicAdd(a.decided, 1u);
                    }
                }
            }
        }
        rp = rn;
    }
}

template <int NPL, int K, bool PARTS>
cudaError_t ring_launch_t(const RingArgs& a, int nb, cudaStream_t s) {
    auto k = ring_kernel<NPL, K, PARTS>;
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
    RingArgs arg = a;
    void* args[] = {&arg};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(k), dim3(static_cast<unsigned>(nb)),
                                       dim3(kRingThreads), args, static_cast<size_t>(a.smem_bytes), s);
}

template <int NPL, bool PARTS>
cudaError_t ring_launch_npl(const RingArgs& a, int nb, cudaStream_t s) {
    switch (a.K) {
        case 6: return ring_launch_t<NPL, 6, PARTS>(a, nb, s);
        case 8: return ring_launch_t<NPL, 8, PARTS>(a, nb, s);
        case 10: return ring_launch_t<NPL, 10, PARTS>(a, nb, s);
        case 12: return ring_launch_t<NPL, 12, PARTS>(a, nb, s);
        case 14: return ring_launch_t<NPL, 14, PARTS>(a, nb, s);
        case 16: return ring_launch_t<NPL, 16, PARTS>(a, nb, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_ring(const RingArgs& a, int nb, cudaStream_t s) {
    // the multi-part ring is its own instantiation: the single-device kernel keeps its code
    if (a.nparts > 0) {
        if (a.npl == 2) return ring_launch_npl<2, true>(a, nb, s);
        if (a.npl == 3) return ring_launch_npl<3, true>(a, nb, s);
    } else {
        if (a.npl == 2) return ring_launch_npl<2, false>(a, nb, s);
        if (a.npl == 3) return ring_launch_npl<3, false>(a, nb, s);
    }
    return cudaErrorInvalidValue;
}

// Diagnostic: copy the ring kernel's stamps (ESCG_DIAG_RING builds; else returns -1).
extern "C" __attribute__((visibility("default"))) int escg_diag_ring(long long* out, int reset) {
#ifdef ESCG_DIAG_RING
    if (reset) {
        static long long z[160 * 32 * 8 * 8];
        static int zp[160 * 32 * 2];
        if (cudaMemcpyToSymbol(g_rpoll, zp, sizeof(zp)) != cudaSuccess) return -1;
        return cudaMemcpyToSymbol(g_rdiag, z, sizeof(z)) == cudaSuccess ? 0 : -1;
    }
    if (cudaMemcpyFromSymbol(out + 160 * 32 * 8 * 8, g_rpoll, sizeof(int) * 160 * 32 * 2) != cudaSuccess) return -1;
    return cudaMemcpyFromSymbol(out, g_rdiag, sizeof(long long) * 160 * 32 * 8 * 8) == cudaSuccess ? 0 : -1;
#else
    (void)out;
    (void)reset;
    return -1;
#endif
}

int ring_smem_bytes(int H, int L, int npl, int nb) {
    const int band_max = (H + nb - 1) / nb;
    return (band_max + 3) * npl * (L / 128) * 4 * 4;
}

int ring_capacity(int npl, int smem_bytes, int device) {
    const void* f = npl == 3 ? reinterpret_cast<const void*>(ring_kernel<3, 10, false>)
                             : reinterpret_cast<const void*>(ring_kernel<2, 10, false>);
    if (cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes) != cudaSuccess) return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, f, kRingThreads, static_cast<size_t>(smem_bytes)) !=
        cudaSuccess)
        return 0;
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 0;
    return per_sm * sms;
}

}  // namespace escgd
