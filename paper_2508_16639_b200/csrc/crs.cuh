// crs.cuh — device core of the coloured random-sequential (CRS) Monte Carlo schedule.
//
// One MCS = one round of four colour phases.  Per round a Philox draw picks the 2x2 tiling origin
// (oy, ox) and the colour order; in each phase every tile of that colour performs 4 sequential
// elementary steps (engine.hpp:108-141) with cell, direction and action drawn from one Philox
// call keyed by (seed) and countered by (tile, mcs, phase).  Same-colour tiles have disjoint
// footprints, so each phase is an exact random-sequential update of its tiles in any order.
// oracle/escg_oracle.c:orc_crs_run is the sequential definition these kernels reproduce bit-exactly.
#pragma once
#include <cstdint>

namespace escgd {

constexpr uint32_t kDomStep = 0, kDomRefine = 1, kDomRound = 2, kDomInit = 3;

// Philox4x32-10 (Salmon et al. SC'11).  mul.wide.u32 → one IMAD.WIDE.U32 per product.
__device__ __forceinline__ uint4 philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                        uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = static_cast<uint64_t>(c0) * 0xD2511F53u;
        const uint64_t p1 = static_cast<uint64_t>(c2) * 0xCD9E8D57u;
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

// Counter word 2: mcs bits 32..47 | domain | low field.
__device__ __forceinline__ uint32_t ctr2(uint64_t mcs, uint32_t dom, uint32_t low) {
    return (static_cast<uint32_t>((mcs >> 32) & 0xFFFFu) << 16) | (dom << 8) | low;
}

// Integer form of the reference's action bucketing (engine.hpp:117-123): migration iff x < xm,
// interaction iff xm <= x < xi, reproduction iff x >= xi.  Coarse copies (x >> LB) let the hot
// loop decide with the 28/27 high bits of the step word; a word whose coarse part equals a
// threshold's coarse part draws its low LB bits from the REFINE domain (exact, rare).
struct Rule {
    uint32_t xm, xi;      // full thresholds
    uint32_t xm_c, xi_c;  // coarse thresholds
};

// Round parameters (orc_crs_round): origin (oy, ox) and the four colours in phase order.
struct Round {
    int oy, ox;
    uint32_t order;  // colour of phase p in bits 2p..2p+1
    __device__ __forceinline__ int colour(int p) const { return static_cast<int>((order >> (2 * p)) & 3u); }
};

__device__ __forceinline__ Round round_params(uint32_t k0, uint32_t k1, uint64_t mcs) {
    // Lexicographic permutations of {0,1,2,3}, packed 2 bits per colour (phase 0 in bits 0-1).
    constexpr uint8_t kPerm[24] = {0xE4, 0xB4, 0xD8, 0x78, 0x9C, 0x6C, 0xE1, 0xB1, 0xC9, 0x39, 0x8D, 0x2D,
                                   0xD2, 0x72, 0xC6, 0x36, 0x4E, 0x1E, 0x93, 0x63, 0x87, 0x27, 0x4B, 0x1B};
    const uint4 w = philox(0u, static_cast<uint32_t>(mcs), ctr2(mcs, kDomRound, 0u), 0u, k0, k1);
    Round r;
    r.oy = static_cast<int>(w.x & 1u);
    r.ox = static_cast<int>((w.x >> 1) & 1u);
    const uint32_t pi = static_cast<uint32_t>((static_cast<uint64_t>(w.y) * 24u) >> 32);
    r.order = kPerm[pi];
    return r;
}

// (drow, dcol) of direction d (params.hpp:81: up, down, left, right, ul, ur, dl, dr).
template <int ARITY>
__device__ __forceinline__ void dir_rc(uint32_t d, int& dr, int& dc) {
    dr = (d < 4u) ? ((d < 2u) ? ((d & 1u) ? 1 : -1) : 0) : ((d & 2u) ? 1 : -1);
    dc = (d < 4u) ? ((d < 2u) ? 0 : ((d & 1u) ? 1 : -1)) : ((d & 1u) ? 1 : -1);
}

// Neighbour offset in a row-major window of pitch P.
template <int ARITY>
__device__ __forceinline__ int dir_offset(uint32_t d, int P) {
    if (ARITY == 4) {
        const int m = (d & 2u) ? 1 : P;
        return (d & 1u) ? m : -m;
    } else {
        int dr, dc;
        dir_rc<ARITY>(d, dr, dc);
        return dr * P + dc;
    }
}

template <int ARITY>
struct Bits {
    static constexpr int DB = ARITY == 8 ? 3 : 2;  // direction bits
    static constexpr int LB = DB + 2;              // low bits (direction + cell) = refine width
};

// Low LB bits of attempt `a` of a tile, from the REFINE domain.
template <int ARITY>
__device__ __noinline__ uint32_t refine_bits(uint32_t k0, uint32_t k1, uint32_t tile, uint64_t mcs, int phase,
                                             int a) {
    const uint4 r = philox(tile, static_cast<uint32_t>(mcs),
                           ctr2(mcs, kDomRefine, (static_cast<uint32_t>(phase) << 2) | static_cast<uint32_t>(a)), 0u,
                           k0, k1);
    return r.x & ((1u << Bits<ARITY>::LB) - 1u);
}

// The rule on one (cell, neighbour) pair with action word x (engine.hpp:111-140).  sT is the
// (S+1)^2 interaction-threshold table: u < D[a][b] (engine.hpp:125-131) ⇔ x < sT[a*S1+b].
// `x` holds the coarse word; `refine()` supplies the exact low bits when a comparison needs them.
template <int ARITY, class Refine>
__device__ __forceinline__ void apply_rule(uint32_t s, uint32_t n, uint32_t word, const Rule& R,
                                           const uint32_t* __restrict__ sT, int S1, uint32_t& ns, uint32_t& nn,
                                           Refine refine) {
    constexpr int LB = Bits<ARITY>::LB;
    const uint32_t coarse = word >> LB;
    uint32_t x = coarse << LB;
    bool exact = false;
    if ((coarse == R.xm_c) | (coarse == R.xi_c)) {
        x |= refine();
        exact = true;
    }
    ns = s;
    nn = n;
    if (x < R.xm) {  // migration: exchange (engine.hpp:118-122)
        ns = n;
        nn = s;
    } else if (x >= R.xi) {  // reproduction into an empty site (engine.hpp:134-140)
        if (n == 0u)
            nn = s;
        else if (s == 0u)
            ns = n;
    } else if ((s != 0u) & (n != 0u) & (s != n)) {  // interaction (engine.hpp:123-133)
        const uint32_t t1 = sT[s * S1 + n], t2 = sT[n * S1 + s];
        if (!exact && ((coarse == (t1 >> LB)) | (coarse == (t2 >> LB)))) x |= refine();
        if (x < t1)
            nn = 0u;
        else if (x < t2)
            ns = 0u;
    }
}

// Four sequential attempts of one tile whose (0,0) cell sits at window offset `base`
// (periodic / contiguous-window addressing: every footprint cell is at base + small offset).
template <int ARITY>
__device__ __forceinline__ void tile_attempts(uint8_t* __restrict__ lat, int base, int P, const uint4 w,
                                              const Rule& R, const uint32_t* __restrict__ sT, int S1, uint32_t k0,
                                              uint32_t k1, uint32_t tile, uint64_t mcs, int phase) {
    constexpr int DB = Bits<ARITY>::DB;
    const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t word = words[a];
        const uint32_t d = word & (ARITY - 1);
        const int sa = base + static_cast<int>((word >> DB) & 1u) * P + static_cast<int>((word >> (DB + 1)) & 1u);
        const int na = sa + dir_offset<ARITY>(d, P);
        const uint32_t s = lat[sa], n = lat[na];
        uint32_t ns, nn;
        apply_rule<ARITY>(s, n, word, R, sT, S1, ns, nn,
                          [&]() { return refine_bits<ARITY>(k0, k1, tile, mcs, phase, a); });
        lat[sa] = static_cast<uint8_t>(ns);
        lat[na] = static_cast<uint8_t>(nn);
    }
}

// Mirror-reflect variant (flux=false, lattice.hpp:42-47): tile cells outside the lattice are
// skipped (partial edge tiles), neighbours reflect one step inward.  (y0, x0) are the global
// coordinates of the tile's (0,0) cell; the window maps global (y, x) to (y+R0)*P + x + C0.
template <int ARITY>
__device__ __forceinline__ void tile_attempts_reflect(uint8_t* __restrict__ lat, int y0, int x0, int R0, int C0,
                                                      int P, int H, int L, const uint4 w, const Rule& R,
                                                      const uint32_t* __restrict__ sT, int S1, uint32_t k0,
                                                      uint32_t k1, uint32_t tile, uint64_t mcs, int phase) {
    constexpr int DB = Bits<ARITY>::DB;
    const uint32_t words[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t word = words[a];
        const uint32_t d = word & (ARITY - 1);
        const int y = y0 + static_cast<int>((word >> DB) & 1u);
        const int x = x0 + static_cast<int>((word >> (DB + 1)) & 1u);
        if (y < 0 || y >= H || x < 0 || x >= L) continue;
        int dr, dc;
        dir_rc<ARITY>(d, dr, dc);
        int ny = y + dr, nx = x + dc;
        if (ny < 0) ny = -ny;
        if (ny >= H) ny = 2 * (H - 1) - ny;
        if (nx < 0) nx = -nx;
        if (nx >= L) nx = 2 * (L - 1) - nx;
        const int sa = (y + R0) * P + x + C0;
        const int na = (ny + R0) * P + nx + C0;
        const uint32_t s = lat[sa], n = lat[na];
        uint32_t ns, nn;
        apply_rule<ARITY>(s, n, word, R, sT, S1, ns, nn,
                          [&]() { return refine_bits<ARITY>(k0, k1, tile, mcs, phase, a); });
        lat[sa] = static_cast<uint8_t>(ns);
        lat[na] = static_cast<uint8_t>(nn);
    }
}

}  // namespace escgd
