/*
 * escg_oracle.c — CPU restatement of the reference ESCG Monte Carlo step path.
 *
 *   *** TEST INFRASTRUCTURE ONLY ***
 *   Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 *   legs may load this library, and only as the checker (or the timed CPU baseline).
 *   The product path (paper_2508_16639_b200/) never links, loads or calls it.
 *
 * Parity is pinned two ways:
 *   1. against the reference's own sources compiled unmodified into oracle/_ref/ (ref_shim.cpp),
 *      on the same seeds: MT19937 words, initial lattices, serial trajectories, rule outcomes;
 *   2. against the SPEC known-answer vectors (MT19937 KATs SPEC.md:155,164; neighbor_index
 *      SPEC.md:86-88; align_num_randoms SPEC.md:191-193) and the Random123 Philox4x32-10 KATs.
 *
 * Part A restates the reference (MT19937 serial path).  Part B restates the device schedule
 * ("coloured random-sequential", CRS) with the *reference's* double-precision elementary_step,
 * so the GPU kernels' integer-threshold rule and parallel schedule are checked bit-for-bit
 * against the reference's arithmetic.  Every function cites the reference file:line it follows;
 * paths are relative to /root/reference/proj/.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------------------------ */
/* Part A — reference restatement                                                             */
/* ------------------------------------------------------------------------------------------ */

/* include/escg/mt19937.hpp:9-16 */
EXPORT uint32_t orc_murmur_finalize(uint32_t x) {
    x ^= x >> 16;
    x *= 0x85ebca6bu;
    x ^= x >> 13;
    x *= 0xc2b2ae35u;
    x ^= x >> 16;
    return x;
}

/* include/escg/mt19937.hpp:20-22 */
EXPORT uint32_t orc_seed_mix(uint32_t seed, uint32_t stream_id) { return orc_murmur_finalize(seed ^ stream_id); }

typedef struct orc_mt {
    uint32_t s[624];
    int32_t idx;
} orc_mt;

/* include/escg/mt19937.hpp:44-49 (reseed) */
EXPORT void orc_mt_seed(orc_mt* g, uint32_t seed) {
    g->s[0] = seed;
    for (int i = 1; i < 624; ++i) g->s[i] = 1812433253u * (g->s[i - 1] ^ (g->s[i - 1] >> 30)) + (uint32_t)i;
    g->idx = 624;
}

/* include/escg/mt19937.hpp:81-89 (twist) */
static void orc_mt_twist(orc_mt* g) {
    for (int i = 0; i < 624; ++i) {
        uint32_t y = (g->s[i] & 0x80000000u) | (g->s[(i + 1) % 624] & 0x7fffffffu);
        uint32_t next = y >> 1;
        if (y & 1u) next ^= 0x9908b0dfu;
        g->s[i] = g->s[(i + 397) % 624] ^ next;
    }
    g->idx = 0;
}

/* include/escg/mt19937.hpp:51-59 (extract + tempering 11/7/15/18) */
EXPORT uint32_t orc_mt_extract(orc_mt* g) {
    if (g->idx >= 624) orc_mt_twist(g);
    uint32_t y = g->s[g->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* include/escg/mt19937.hpp:62 — float(x) / 4294967295.0f (the divisor rounds to 2^32) */
EXPORT float orc_unit(uint32_t x) { return (float)x / 4294967295.0f; }

EXPORT float orc_mt_next_unit(orc_mt* g) { return orc_unit(orc_mt_extract(g)); }

/* include/escg/mt19937.hpp:64-66 */
EXPORT void orc_mt_discard(orc_mt* g, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) orc_mt_extract(g);
}

/* include/escg/random_batch.hpp:44-53 — stream k = seed_mix(u32(seed + k), k), burn-in 50000
 * (mt19937.hpp:26 kDefaultBurnIn). */
EXPORT void orc_stream_init(orc_mt* g, uint64_t global_seed, int k, uint64_t burn_in) {
    orc_mt_seed(g, orc_seed_mix((uint32_t)(global_seed + (uint64_t)k), (uint32_t)k));
    orc_mt_discard(g, burn_in);
}

EXPORT int64_t orc_sizeof_mt(void) { return (int64_t)sizeof(orc_mt); }

/* include/escg/random_batch.hpp:32-38 — returns -1 on ConfigError */
EXPORT int64_t orc_align_num_randoms(int64_t requested, int64_t cells) {
    if (cells < 1 || requested < cells) return -1;
    return requested / cells * cells;
}

/* include/escg/params.hpp:61-70 — out = {mu, sigma, epsilon, total} */
EXPORT void orc_action_rates(double mobility, int64_t cells, double* out) {
    out[0] = 1.0;
    out[1] = 1.0;
    out[2] = 2.0 * mobility * (double)cells;
    out[3] = out[0] + out[1] + out[2];
}

/* include/escg/params.hpp:81 — (drow, dcol): up, down, left, right, ul, ur, dl, dr */
static const int kOff[8][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {-1, -1}, {-1, 1}, {1, -1}, {1, 1}};

/* include/escg/lattice.hpp:31-49 — returns -1 for an out-of-range direction (ConfigError) */
EXPORT int64_t orc_neighbor_index(int64_t i, int dir, int arity, int length, int height, int flux) {
    if (dir < 0 || dir >= arity) return -1;
    int row = (int)(i / length);
    int col = (int)(i % length);
    row += kOff[dir][0];
    col += kOff[dir][1];
    if (flux) {
        row = (row + height) % height;
        col = (col + length) % length;
    } else {
        if (row < 0) row = -row;
        if (row >= height) row = 2 * (height - 1) - row;
        if (col < 0) col = -col;
        if (col >= length) col = 2 * (length - 1) - col;
    }
    return (int64_t)row * length + col;
}

/* include/escg/lattice.hpp:53-66 — uniform initial lattice from one MT stream */
EXPORT void orc_init_lattice(int length, int height, int species, double empty_prob, orc_mt* g, int32_t* cells) {
    int64_t n = (int64_t)length * height;
    memset(cells, 0, sizeof(int32_t) * (size_t)n);
    if (empty_prob >= 1.0) return;
    for (int64_t i = 0; i < n; ++i) {
        if (empty_prob > 0.0 && (double)orc_mt_next_unit(g) < empty_prob) {
            cells[i] = 0;
            continue;
        }
        cells[i] = (int32_t)(orc_mt_extract(g) % (uint32_t)species) + 1;
    }
}

typedef struct orc_ctx {
    int32_t length, height, species, arity, flux;
    const double* dom; /* S*S, row = attacker-1 (include/escg/dominance.hpp:20) */
    double mu, sigma, epsilon, total;
} orc_ctx;

/* include/escg/engine.hpp:108-141 — elementary_step<PlainCellAccess>.
 * Returns 0, or 5 (EngineError) on a corrupt lattice value. */
static int orc_step(int32_t* cells, const orc_ctx* c, int64_t cell, int dir, float action) {
    const int64_t ni = orc_neighbor_index(cell, dir, c->arity, c->length, c->height, c->flux);
    const int32_t s = cells[cell];
    const int32_t n = cells[ni];
    if (s == n) return 0;
    if (s > c->species || n > c->species || s < 0 || n < 0) return 5;
    const double r = (double)action * c->total;
    if (r < c->epsilon) {
        cells[cell] = n;
        cells[ni] = s;
    } else if (r < c->epsilon + c->mu) {
        if (n != 0 && s != 0) {
            const double u = (r - c->epsilon) / c->mu;
            const double fwd = c->dom[(size_t)(s - 1) * c->species + (n - 1)];
            if (fwd > 0.0 && u < fwd) {
                cells[ni] = 0;
            } else {
                const double bwd = c->dom[(size_t)(n - 1) * c->species + (s - 1)];
                if (bwd > 0.0 && u < bwd) cells[cell] = 0;
            }
        }
    } else {
        if (n == 0) {
            cells[ni] = s;
        } else if (s == 0) {
            cells[cell] = n;
        }
    }
    return 0;
}

static void orc_ctx_make(orc_ctx* c, int length, int height, int species, int arity, int flux, const double* dom,
                         double mobility) {
    double r[4];
    c->length = length;
    c->height = height;
    c->species = species;
    c->arity = arity;
    c->flux = flux;
    c->dom = dom;
    orc_action_rates(mobility, (int64_t)length * height, r);
    c->mu = r[0];
    c->sigma = r[1];
    c->epsilon = r[2];
    c->total = r[3];
}

/* One elementary step on a caller lattice (rule KAT).  Returns 0 / 5. */
EXPORT int orc_elementary_step(int32_t* cells, int length, int height, int species, int arity, int flux,
                               const double* dom, double mobility, int64_t cell, int dir, float action) {
    orc_ctx c;
    orc_ctx_make(&c, length, height, species, arity, flux, dom, mobility);
    return orc_step(cells, &c, cell, dir, action);
}

/* Bucket of an action word under the reference's double comparisons (engine.hpp:117-123):
 * 0 migration, 1 interaction, 2 reproduction. */
EXPORT int orc_bucket(uint32_t x, double mobility, int64_t cells) {
    double r4[4];
    orc_action_rates(mobility, cells, r4);
    const double r = (double)orc_unit(x) * r4[3];
    if (r < r4[2]) return 0;
    if (r < r4[2] + r4[0]) return 1;
    return 2;
}

/* Interaction outcome for attacker s vs neighbour n under word x (engine.hpp:124-133):
 * 0 no change, 1 neighbour cleared, 2 cell cleared. Only meaningful in the interaction bucket. */
EXPORT int orc_interaction(uint32_t x, double mobility, int64_t cells, const double* dom, int species, int s, int n) {
    double r4[4];
    orc_action_rates(mobility, cells, r4);
    const double r = (double)orc_unit(x) * r4[3];
    const double u = (r - r4[2]) / r4[0];
    const double fwd = dom[(size_t)(s - 1) * species + (n - 1)];
    if (fwd > 0.0 && u < fwd) return 1;
    const double bwd = dom[(size_t)(n - 1) * species + (s - 1)];
    if (bwd > 0.0 && u < bwd) return 2;
    return 0;
}

/* Count mismatches between integer thresholds and the reference's double bucketing over the
 * word range [lo, hi] with the given stride (stride 1 + full range = exhaustive over 2^32).
 * thr = {X_mig, X_int}.  Used to validate the product's host-side threshold precompute. */
EXPORT int64_t orc_check_bucket_thresholds(const uint32_t* thr, double mobility, int64_t cells, uint64_t lo,
                                           uint64_t hi, uint64_t stride) {
    double r4[4];
    int64_t bad = 0;
    orc_action_rates(mobility, cells, r4);
    const double e = r4[2], em = r4[2] + r4[0], t = r4[3];
    for (uint64_t v = lo; v <= hi; v += stride) {
        const uint32_t x = (uint32_t)v;
        const double r = (double)((float)x / 4294967295.0f) * t;
        const int ref = r < e ? 0 : (r < em ? 1 : 2);
        const int dev = x < thr[0] ? 0 : (x < thr[1] ? 1 : 2);
        bad += ref != dev;
    }
    return bad;
}

/* include/src engine.cpp:70-94 — densities(); returns 5 on a corrupt value */
EXPORT int orc_densities(const int32_t* cells, int64_t n, int species, uint64_t* counts) {
    memset(counts, 0, sizeof(uint64_t) * (size_t)(species + 1));
    for (int64_t i = 0; i < n; ++i) {
        const int32_t v = cells[i];
        if (v < 0 || v > species) return 5;
        ++counts[v];
    }
    return 0;
}

/* engine.cpp:14-19 — geometric snapshot schedule */
EXPORT int orc_is_save_mcs(int64_t mcs, int64_t limit) {
    if (mcs == 0 || mcs == limit) return 1;
    int64_t lead = mcs;
    while (lead >= 10 && lead % 10 == 0) lead /= 10;
    return lead == 1 || lead == 2 || lead == 5;
}

/* Status codes: engine.hpp:20 RunStatus {Completed, Stasis, Stopped} */
enum { ORC_COMPLETED = 0, ORC_STASIS = 1, ORC_STOPPED = 2 };

/* engine.cpp:47-57 record_and_check (without console/on_save observers).  The on_record hook is
 * restated as the predicate the experiments harness installs (experiments.cpp:107-113):
 * stop when counts[tracked] == 0 (tracked < 1 disables it). Returns -1 to continue. */
static int orc_record(const int32_t* cells, int64_t n, int species, int64_t mcs, int64_t limit, int tracked,
                      int64_t* steps, uint64_t* counts, int64_t cap, int64_t* n_rec, int* err) {
    uint64_t local[65];
    *err = orc_densities(cells, n, species, local);
    if (*err) return -2;
    if (*n_rec < cap) {
        steps[*n_rec] = mcs;
        memcpy(counts + (size_t)(*n_rec) * (species + 1), local, sizeof(uint64_t) * (size_t)(species + 1));
    }
    ++*n_rec;
    if (tracked >= 1 && local[tracked] == 0) return ORC_STOPPED;
    if (mcs >= limit) return ORC_COMPLETED;
    int alive = 0;
    for (int s = 1; s <= species; ++s) alive += local[s] > 0;
    if (alive <= 1) return ORC_STASIS; /* engine.hpp:40-43 */
    return -1;
}

/* engine.cpp:96-113 run_serial, driven as simulate(..., Serial) does (engine.cpp:194-240):
 * StreamSet(seed, 1) → init_lattice(stream 0) (unless init_cells given) → loop.
 * Returns status (>=0) or -5 on EngineError. */
EXPORT int orc_run_serial(int length, int height, int species, int arity, int flux, const double* dom,
                          double mobility, double empty_prob, int64_t mcs_limit, uint64_t seed,
                          const int32_t* init_cells, int tracked, int32_t* out_cells, int64_t* steps,
                          uint64_t* counts, int64_t cap, int64_t* n_rec) {
    orc_ctx c;
    orc_mt* g = (orc_mt*)malloc(sizeof(orc_mt));
    const int64_t n = (int64_t)length * height;
    int err = 0, st;
    orc_ctx_make(&c, length, height, species, arity, flux, dom, mobility);
    orc_stream_init(g, seed, 0, 50000);
    if (init_cells)
        memcpy(out_cells, init_cells, sizeof(int32_t) * (size_t)n);
    else
        orc_init_lattice(length, height, species, empty_prob, g, out_cells);
    *n_rec = 0;
    for (int64_t mcs = 0;; ++mcs) {
        st = orc_record(out_cells, n, species, mcs, mcs_limit, tracked, steps, counts, cap, n_rec, &err);
        if (st == -2) break;
        if (st >= 0) {
            free(g);
            return st;
        }
        for (uint32_t i = 0; i < (uint32_t)n; ++i) {
            const int64_t cell = orc_mt_extract(g) % (uint32_t)n;
            const int dir = (int)(orc_mt_extract(g) % (uint32_t)arity);
            const float action = orc_mt_next_unit(g);
            if (orc_step(out_cells, &c, cell, dir, action)) {
                free(g);
                return -5;
            }
        }
    }
    free(g);
    return -5;
}

/* Serial draw injection (north_star "injected identical random draw sequence"): the initial
 * lattice and the raw 3-word-per-attempt MT stream that run_serial would consume
 * (engine.cpp:104-110) after init_lattice on StreamSet(seed,1) stream 0. */
EXPORT void orc_serial_draws(int length, int height, int species, double empty_prob, uint64_t seed,
                             int32_t* init_cells, int64_t n_attempts, uint32_t* w_cell, uint32_t* w_dir,
                             uint32_t* w_act) {
    orc_mt* g = (orc_mt*)malloc(sizeof(orc_mt));
    orc_stream_init(g, seed, 0, 50000);
    orc_init_lattice(length, height, species, empty_prob, g, init_cells);
    for (int64_t i = 0; i < n_attempts; ++i) {
        w_cell[i] = orc_mt_extract(g);
        w_dir[i] = orc_mt_extract(g);
        w_act[i] = orc_mt_extract(g);
    }
    free(g);
}

/* Apply injected words with the reference rule exactly as run_serial does
 * (cell = w % N, dir = w % arity, action = next_unit(w); engine.cpp:106-109). */
EXPORT int orc_apply_draws(int32_t* cells, int length, int height, int species, int arity, int flux,
                           const double* dom, double mobility, const uint32_t* w_cell, const uint32_t* w_dir,
                           const uint32_t* w_act, int64_t n_attempts) {
    orc_ctx c;
    const uint32_t n = (uint32_t)((int64_t)length * height);
    orc_ctx_make(&c, length, height, species, arity, flux, dom, mobility);
    for (int64_t i = 0; i < n_attempts; ++i) {
        int e = orc_step(cells, &c, w_cell[i] % n, (int)(w_dir[i] % (uint32_t)arity), orc_unit(w_act[i]));
        if (e) return e;
    }
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* Part B — device schedule restated with the reference rule (shadow replay)                  */
/* ------------------------------------------------------------------------------------------ */

/* Philox4x32-10 (Salmon et al., SC'11; Random123 philox.h round/bumpkey), KAT-checked. */
EXPORT void orc_philox(const uint32_t* ctr_in, const uint32_t* key_in, uint32_t* out) {
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        c0 = hi1 ^ c1 ^ k0;
        c1 = lo1;
        c2 = hi0 ^ c3 ^ k1;
        c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0;
    out[1] = c1;
    out[2] = c2;
    out[3] = c3;
}

/* Draw spec of the device schedule, version 2:
 *   key  = (0xA4093822, 0x299F31D0)  (fixed: round keys become immediates on the device)
 *   c0   = tile id | tile-pair id | cell pair | 0  (by domain)
 *   c1   = mcs bits 0..31
 *   c2   = mcs bits 32..47 | domain << 16 | phase << 20 | attempt << 24
 *   c3   = seed32 = u32(seed) ^ murmur_finalize(u32(seed >> 32))  (= u32(seed) for seeds < 2^32) */
enum { DOM_STEP = 0, DOM_REFINE = 1, DOM_ROUND = 2, DOM_INIT = 3, DOM_SLICE = 4, DOM_SLICE_REF = 5 };
static const uint32_t kKey0 = 0xA4093822u, kKey1 = 0x299F31D0u;

EXPORT uint32_t orc_seed32(uint64_t seed) {
    return (uint32_t)seed ^ orc_murmur_finalize((uint32_t)(seed >> 32));
}

static void crs_draw(uint64_t seed, uint32_t c0, uint64_t mcs, uint32_t dom, uint32_t phase, uint32_t attempt,
                     uint32_t* out) {
    uint32_t ctr[4], key[2];
    ctr[0] = c0;
    ctr[1] = (uint32_t)mcs;
    ctr[2] = ((uint32_t)(mcs >> 32) & 0xFFFFu) | (dom << 16) | (phase << 20) | (attempt << 24);
    ctr[3] = orc_seed32(seed);
    key[0] = kKey0;
    key[1] = kKey1;
    orc_philox(ctr, key, out);
}

/* Lexicographic permutations of the four colours {0,1,2,3}; colour c = (cy<<1)|cx. */
static const uint8_t kPerm[24][4] = {
    {0, 1, 2, 3}, {0, 1, 3, 2}, {0, 2, 1, 3}, {0, 2, 3, 1}, {0, 3, 1, 2}, {0, 3, 2, 1}, {1, 0, 2, 3}, {1, 0, 3, 2},
    {1, 2, 0, 3}, {1, 2, 3, 0}, {1, 3, 0, 2}, {1, 3, 2, 0}, {2, 0, 1, 3}, {2, 0, 3, 1}, {2, 1, 0, 3}, {2, 1, 3, 0},
    {2, 3, 0, 1}, {2, 3, 1, 0}, {3, 0, 1, 2}, {3, 0, 2, 1}, {3, 1, 0, 2}, {3, 1, 2, 0}, {3, 2, 0, 1}, {3, 2, 1, 0}};

/* Round parameters of MCS `mcs`: tiling origin (oy, ox) ∈ {0,1}² and the colour order. */
EXPORT void orc_crs_round(uint64_t seed, uint64_t mcs, int* oy, int* ox, int* perm) {
    uint32_t w[4];
    crs_draw(seed, 0u, mcs, DOM_ROUND, 0, 0, w);
    *oy = (int)(w[0] & 1u);
    *ox = (int)((w[0] >> 1) & 1u);
    const uint32_t pi = (uint32_t)(((uint64_t)w[1] * 24u) >> 32);
    for (int k = 0; k < 4; ++k) perm[k] = kPerm[pi][k];
}

static int crs_tiles(int n, int o, int periodic) {
    if (periodic) return (n % 4 == 0) ? n / 2 : (n + 1) / 2;
    return (n + o + 1) / 2;
}

/* Periodic axis of length n >= 4.  n % 4 == 0: T = n/2 tiles, colours t & 1.
 * Otherwise T = ceil(n/2) tiles (the last one holds one cell when n is odd) and one seam tile takes
 * a third colour: the tile ring then has odd length (n % 4 in {1, 2}: seam = T-1) or, for n % 4 == 3,
 * a chord between tiles T-2 and 0 (their footprints meet across the 1-cell tile; seam = T-2).
 * Returns the number of colours; *seam = seam tile (or -1). */
static int crs_axis(int n, int* seam) {
    const int T = (n + 1) / 2;
    if (n % 4 == 0) {
        *seam = -1;
        return 2;
    }
    *seam = (n % 4 == 3) ? T - 2 : T - 1;
    return 3;
}

static int crs_colour(int t, int seam) { return t == seam ? 2 : (t & 1); }

/* Phase order of an MCS for cy x cx colours.  4 colours: the lexicographic permutation table of
 * orc_crs_round (unchanged).  6 or 9: Fisher-Yates over colour ids v = cy * ncx + cx driven by the
 * 16-bit halves of a second ROUND draw (attempt field 1): j = (half_k * (i + 1)) >> 16 for
 * i = np-1 .. 1, k = np-1-i. */
EXPORT void orc_crs_round_g(uint64_t seed, uint64_t mcs, int ncy, int ncx, int* oy, int* ox, int* perm) {
    int p4[4];
    orc_crs_round(seed, mcs, oy, ox, p4);
    const int np = ncy * ncx;
    if (np == 4) {
        for (int k = 0; k < 4; ++k) perm[k] = p4[k];
        return;
    }
    uint32_t w[4];
    crs_draw(seed, 0u, mcs, DOM_ROUND, 0, 1, w);
    for (int k = 0; k < np; ++k) perm[k] = k;
    for (int i = np - 1, k = 0; i >= 1; --i, ++k) {
        const uint32_t half = (w[k >> 1] >> (16 * (k & 1))) & 0xFFFFu;
        const int j = (int)((half * (uint32_t)(i + 1)) >> 16);
        const int t = perm[i];
        perm[i] = perm[j];
        perm[j] = t;
    }
}

/* Device init_lattice (the device counterpart of lattice.hpp:53-66): the same transformation of
 * two uniform words per cell (empty test via next_unit, species via % S + 1), drawn from the
 * Philox INIT domain (cell pair i>>1) instead of the MT stream. */
EXPORT void orc_crs_init(int length, int height, int species, double empty_prob, uint64_t seed, int32_t* cells) {
    const int64_t n = (int64_t)length * height;
    uint32_t w[4];
    for (int64_t i = 0; i < n; ++i) {
        cells[i] = 0;
        if (empty_prob >= 1.0) continue;
        crs_draw(seed, (uint32_t)(i >> 1), 0, DOM_INIT, 0, 0, w);
        const uint32_t we = (i & 1) ? w[2] : w[0];
        const uint32_t ws = (i & 1) ? w[3] : w[1];
        if (empty_prob > 0.0 && (double)orc_unit(we) < empty_prob) continue;
        cells[i] = (int32_t)(ws % (uint32_t)species) + 1;
    }
}

/* Draw formats.  LB = direction bits + 2 (cell bits) = 4 (VN4) / 5 (Moore8).
 *  WIDE   one STEP draw per 2x2 tile (c0 = tile id); attempt a uses 32-bit word a:
 *         bits [0,LB) direction/cell, action x = (word >> LB) << LB | (REFINE(tile,p,a).x & (2^LB-1)).
 *  NARROW one STEP draw per pair of same-colour tiles (tx, tx+2) of a row (c0 = ty*ceil(Tx/4) + tx/4);
 *         tile half h = (tx>>1)&1 uses words 2h, 2h+1; attempt a uses 16-bit half (a&1) of word
 *         2h+(a>>1): bits [0,LB) direction/cell, action x = (half >> LB) << (32-(16-LB))
 *         | (REFINE(tile,p,a).x & (2^(16+LB)-1)).
 *  SLICED (fmt = 2 | K << 8; periodic, VN4, L % 128 == 0, H % 4 == 0, X_mig >= 2^32 - 2^(32-K)):
 *         bit-plane draws shared by the 32 same-colour tiles whose anchor (top-left) cell (y, x)
 *         = (2ty - oy, 2tx - ox) mod (H, L) lies in columns [128g, 128g + 128) of tile row ty:
 *         item id c0 = ty * (L / 128) + g, lane l = (x mod 128) >> 2.  Words W[4j .. 4j+3] =
 *         SLICE draw j (attempt field j) for j < 4 + K; attempt a reads bit l of W[4a] (cell row),
 *         W[4a+1] (cell column), W[4a+2] | W[4a+3] << 1 (direction) and of W[16 + aK + i], i < K,
 *         as bit 31-i of the action word; its low 32-K bits are word a of SLICE_REF draw
 *         (c0 = item, attempt field l).
 *  SLICED3 (fmt = 3 | K << 8; as SLICED): the undecided mask U_a of attempt a (bit l set:
 *         tile l's action word has its top K bits all one, i.i.d. with probability q = 2^-K) is
 *         drawn by inversion instead of as the AND of K words.  Tables (integer recurrences, so
 *         engine and oracle agree bit for bit; each probability within 2^-27 of the exact power):
 *           T[g], g = 1..32: T[0] = 2^32, T[g] = floor(T[g-1] (2^K-1) / 2^K)      ~ 2^32 (1-q)^g
 *           S[G], G = 0..31: T[G+1] + r_{31-G}, r_0 = T[G] - T[G+1], r_i = floor(r_{i-1} (2^K-1)/2^K)
 *           C[m][g], m = 1..31, g = 1..m-1: floor((T[g] - T[m]) 2^32 / (2^32 - T[m]))
 *         u = word a of SLICE draw 4: u >= T[32] gives the first set bit G = #{g in 1..32 : u < T[g]}
 *         (U = 0 when u < T[32]); u < S[G] means it is the only one (the common case: one word per
 *         attempt).  Otherwise at least one more follows among the m = 31 - G positions after G: the
 *         next word (word a of SLICE draw 5) places it at G + 1 + #{g in 1..m-1 : w < C[m][g]} (the
 *         run conditioned on a set bit), and the bits after it are runs of T drawn from words a of
 *         SLICE draws 6, 7, ...: #{g in 1..r : w < T[g]} decided tiles, r = the positions left,
 *         r meaning none.  Choice words as SLICED (SLICE draws 0..3); an undecided attempt's action
 *         word is TK | (word a of the SLICE_REF draw & ~TK), TK = the K leading ones; a decided
 *         attempt is a migration.
 * In every format the action word is a uniform 32-bit value assembled from disjoint Philox bits (for
 * SLICED3: each decision of the undecided mask within 2^-27 of its probability, the reference's own
 * float action quantisation being 2^-24), so the rule sees the reference's action distribution. */

static void crs_attempt_bits(int narrow, int lb, const uint32_t* w, int h, int a, uint32_t* low, uint32_t* hi_part,
                             int* hi_shift) {
    if (!narrow) {
        *low = w[a] & ((1u << lb) - 1u);
        *hi_part = w[a] >> lb;
        *hi_shift = lb;
    } else {
        const uint32_t half = (w[2 * h + (a >> 1)] >> (16 * (a & 1))) & 0xFFFFu;
        *low = half & ((1u << lb) - 1u);
        *hi_part = half >> lb;
        *hi_shift = 32 - (16 - lb);
    }
}

/* SLICED3 tables: out[0..31] = T[1..32], out[32..63] = S[0..31], out[64 + 32 (m-1) + g] = C[m][g]. */
EXPORT void orc_slice3_table(int K, uint32_t* out) {
    const uint64_t num = (1ull << K) - 1ull;
    uint64_t T[33];
    T[0] = 1ull << 32;
    for (int g = 1; g <= 32; ++g) T[g] = (T[g - 1] * num) >> K;
    for (int g = 1; g <= 32; ++g) out[g - 1] = (uint32_t)T[g];
    for (int G = 0; G < 32; ++G) {
        uint64_t r = T[G] - T[G + 1];
        for (int i = 0; i < 31 - G; ++i) r = (r * num) >> K;
        out[32 + G] = (uint32_t)(T[G + 1] + r);
    }
    for (int i = 0; i < 31 * 32; ++i) out[64 + i] = 0u;
    for (int m = 1; m <= 31; ++m)
        for (int g = 1; g < m; ++g) out[64 + 32 * (m - 1) + g] = (uint32_t)(((T[g] - T[m]) << 32) / ((1ull << 32) - T[m]));
}

/* #{g in 1..n : u < t[g]} for a decreasing threshold list t[1..n] (t given from index 1). */
static int slice3_run(uint32_t u, const uint32_t* t1, int n) {
    int g = 0;
    while (g < n && u < t1[g]) ++g; /* t1[g] = threshold of run length g + 1 */
    return g;
}

/* SLICED3 undecided mask of attempt a of an item (see above); tab = orc_slice3_table. */
static uint32_t slice3_mask(uint64_t seed, uint32_t item, uint64_t mcs, uint32_t p, int a, uint32_t u,
                            const uint32_t* tab) {
    const uint32_t* T = tab;        /* T[g-1] */
    const uint32_t* S = tab + 32;   /* S[G] */
    if (u < T[31]) return 0u;
    const int G = slice3_run(u, T, 32);
    uint32_t U = 1u << G;
    if (u < S[G]) return U;
    uint32_t w4[4];
    crs_draw(seed, item, mcs, DOM_SLICE, p, 5u, w4);
    const int m = 31 - G;
    int pos = G + 1 + slice3_run(w4[a], tab + 64 + 32 * (m - 1) + 1, m - 1);
    U |= 1u << pos;
    ++pos;
    for (uint32_t k = 6; pos < 32; ++k) {
        crs_draw(seed, item, mcs, DOM_SLICE, p, k, w4);
        const int r = 32 - pos, g = slice3_run(w4[a], T, r);
        if (g == r) break;
        pos += g;
        U |= 1u << pos;
        ++pos;
    }
    return U;
}

/* Test hook: the SLICED3 undecided mask of attempt a of item `item` in phase p of MCS mcs. */
EXPORT uint32_t orc_slice3_mask(uint64_t seed, uint32_t item, uint64_t mcs, uint32_t p, int a, int K) {
    uint32_t T3[64 + 31 * 32], w4[4];
    orc_slice3_table(K, T3);
    crs_draw(seed, item, mcs, DOM_SLICE, p, 4u, w4);
    return slice3_mask(seed, item, mcs, p, a, w4[a], T3);
}

/* n_mcs rounds of the coloured random-sequential schedule starting at MCS mcs0, applying the
 * reference elementary_step (engine.hpp:108-141) with full 32-bit action words.  Tiles of one
 * colour have disjoint footprints, so the order within a phase is immaterial; this loop is the
 * sequential definition the GPU kernels must reproduce bit-for-bit.  Returns 0 / 5 / 2. */
EXPORT int orc_crs_run(int32_t* cells, int length, int height, int species, int arity, int flux,
                       const double* dom, double mobility, uint64_t seed, int64_t mcs0, int64_t n_mcs, int fmt) {
    orc_ctx c;
    const int periodic = flux != 0;
    const int db = arity == 8 ? 3 : 2;
    const int lb = db + 2;
    if (periodic && (length < 4 || height < 4)) return 2;
    int seam_y = -1, seam_x = -1;
    const int ncy = periodic ? crs_axis(height, &seam_y) : 2, ncx = periodic ? crs_axis(length, &seam_x) : 2;
    const int narrow = (fmt & 0xFF) == 1, sliced = (fmt & 0xFF) == 2 || (fmt & 0xFF) == 3, K = fmt >> 8;
    const int sliced3 = (fmt & 0xFF) == 3;
    if (narrow && (ncy != 2 || ncx != 2 || length % 8 != 0)) return 2;
    if (sliced && (ncy != 2 || ncx != 2 || length % 128 != 0 || arity != 4 || K < 1 || K > 24)) return 2;
    uint32_t T3[64 + 31 * 32];
    if (sliced3) orc_slice3_table(K, T3);
    const uint32_t TK = K >= 32 ? ~0u : ~((1u << (32 - K)) - 1u);
    orc_ctx_make(&c, length, height, species, arity, flux, dom, mobility);
    for (int64_t mcs = mcs0; mcs < mcs0 + n_mcs; ++mcs) {
        int oy, ox, perm[9];
        orc_crs_round_g(seed, (uint64_t)mcs, ncy, ncx, &oy, &ox, perm);
        const int ty_n = crs_tiles(height, oy, periodic), tx_n = crs_tiles(length, ox, periodic);
        const int tq = (tx_n + 3) / 4;
        for (int p = 0; p < ncy * ncx; ++p) {
            const int cy = perm[p] / ncx, cx = perm[p] % ncx;
            for (int ty = 0; ty < ty_n; ++ty) {
                if ((periodic ? crs_colour(ty, seam_y) : (ty & 1)) != cy) continue;
                for (int tx = 0; tx < tx_n; ++tx) {
                    if ((periodic ? crs_colour(tx, seam_x) : (tx & 1)) != cx) continue;
                    const uint32_t tile = (uint32_t)ty * (uint32_t)tx_n + (uint32_t)tx;
                    const uint32_t sid = narrow ? (uint32_t)ty * (uint32_t)tq + (uint32_t)(tx >> 2) : tile;
                    const int h = (tx >> 1) & 1;
                    uint32_t w[4], sw[4 * (4 + 24)], srf[4], U3[4] = {0, 0, 0, 0};
                    int lane = 0;
                    if (sliced) {
                        const int ax = ((2 * tx - ox) % length + length) % length;
                        const uint32_t item = (uint32_t)ty * (uint32_t)(length / 128) + (uint32_t)(ax >> 7);
                        lane = (ax & 127) >> 2;
                        for (int j = 0; j < (sliced3 ? 5 : 4 + K); ++j)
                            crs_draw(seed, item, (uint64_t)mcs, DOM_SLICE, (uint32_t)p, (uint32_t)j, sw + 4 * j);
                        if (sliced3)
                            for (int a = 0; a < 4; ++a)
                                U3[a] = slice3_mask(seed, item, (uint64_t)mcs, (uint32_t)p, a, sw[16 + a], T3);
                        crs_draw(seed, item, (uint64_t)mcs, DOM_SLICE_REF, (uint32_t)p, (uint32_t)lane, srf);
                    } else {
                        crs_draw(seed, sid, (uint64_t)mcs, DOM_STEP, (uint32_t)p, 0, w);
                    }
                    for (int a = 0; a < 4; ++a) {
                        uint32_t rf[4], low, hi_part;
                        int hi_shift;
                        uint32_t x;
                        int dir, dy, dx;
                        if (sliced) {
                            dy = (int)((sw[4 * a] >> lane) & 1u);
                            dx = (int)((sw[4 * a + 1] >> lane) & 1u);
                            dir = (int)(((sw[4 * a + 2] >> lane) & 1u) | (((sw[4 * a + 3] >> lane) & 1u) << 1));
                            if (sliced3) {
                                /* decided: a certain migration (action word 0); undecided: the exact word */
                                x = ((U3[a] >> lane) & 1u) ? (TK | (srf[a] & ~TK)) : 0u;
                            } else {
                                uint32_t hi = 0;
                                for (int i = 0; i < K; ++i) hi = (hi << 1) | ((sw[16 + a * K + i] >> lane) & 1u);
                                x = (hi << (32 - K)) | (srf[a] & ((1u << (32 - K)) - 1u));
                            }
                        } else {
                            crs_attempt_bits(narrow, lb, w, h, a, &low, &hi_part, &hi_shift);
                            dir = (int)(low & (uint32_t)(arity - 1));
                            dy = (int)((low >> db) & 1u);
                            dx = (int)((low >> (db + 1)) & 1u);
                            crs_draw(seed, tile, (uint64_t)mcs, DOM_REFINE, (uint32_t)p, (uint32_t)a, rf);
                            x = (hi_part << hi_shift) | (rf[0] & ((1u << hi_shift) - 1u));
                        }
                        int y = 2 * ty - oy + dy, xc = 2 * tx - ox + dx;
                        if (periodic) {
                            /* the missing half of an odd axis' last tile: no attempt */
                            if (2 * ty + dy >= height || 2 * tx + dx >= length) continue;
                            y = (y + height) % height;
                            xc = (xc + length) % length;
                        } else if (y < 0 || y >= height || xc < 0 || xc >= length) {
                            continue;
                        }
                        const int e = orc_step(cells, &c, (int64_t)y * length + xc, dir, orc_unit(x));
                        if (e) return e;
                    }
                }
            }
        }
    }
    return 0;
}
