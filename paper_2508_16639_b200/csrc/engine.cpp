// engine.cpp — host side of the B200 ESCG engine and its C ABI (include/escg_dev.h).
//
// Mirrors the reference's dispatcher/driver layer (engine.cpp:194-240 simulate, :96-192 run loops,
// :47-57 record_and_check) around the sm_100a kernels in kernels.cu.  Validation mirrors
// params.hpp:37-48 and dominance.cpp:8-21 with the same messages; errors become int codes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <string>
#include <vector>

#include "../../include/escg_dev.h"
#include "launch.h"

namespace {

thread_local std::string g_last_error;

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void config_error(const std::string& m) { throw Error(ESCG_ECONFIG, m); }
[[noreturn]] void engine_error(const std::string& m) { throw Error(ESCG_EENGINE, m); }

#define CK(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess) engine_error(std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <class F>
int guarded(F&& f) {
    try {
        f();
        g_last_error.clear();
        return ESCG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "out of host memory";
        return ESCG_EENGINE;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return ESCG_EENGINE;
    }
}

// ---- validation (params.hpp:37-48, dominance.cpp:8-21) ---------------------------------------

void validate_params(const escg_params& p) {
    if (p.length < 2 || p.height < 2) config_error("lattice dimensions must be at least 2x2");
    if (p.mcs_limit < 0) config_error("mcs limit must be non-negative");
    if (p.print_frequency < 1) config_error("print frequency must be positive");
    if (!(p.mobility >= 0.0)) config_error("mobility must be non-negative");
    if (p.species < 1 || p.species > 64) config_error("species count must be in [1, 64]");
    if (static_cast<int64_t>(p.length) * p.height > (int64_t{1} << 31))
        config_error("lattice exceeds the supported cell count");
    if (!(p.empty_prob >= 0.0 && p.empty_prob <= 1.0)) config_error("empty probability must be in [0, 1]");
    if (p.num_randoms < 1) config_error("numRandoms must be positive");
    if (p.neighbourhood != 4 && p.neighbourhood != 8) config_error("neighbourhood must be 4 or 8");
}

void validate_dominance(const double* dom, int S, int kind) {
    if (S < 1 || S > 64) config_error("dominance size must be in [1, 64]");
    if (!dom) config_error("dominance entry count does not match size");
    for (int i = 0; i < S; ++i)
        if (dom[static_cast<size_t>(i) * S + i] != 0.0)
            config_error("dominance diagonal must be zero (species " + std::to_string(i + 1) + ")");
    for (int i = 0; i < S * S; ++i) {
        const double v = dom[i];
        if (!(v >= 0.0 && v <= 1.0)) config_error("dominance entries must lie in [0, 1]");
        if (kind == ESCG_DOM_BINARY && v != 0.0 && v != 1.0) config_error("binary dominance entries must be 0 or 1");
    }
}

// ---- exact integer thresholds ------------------------------------------------------------------
// r(x) = double(float(x) / 4294967295.0f) * total is monotone non-decreasing in the raw word x
// (mt19937.hpp:62, engine.hpp:117), so every double comparison of the rule is a threshold on x.

double r_of(uint32_t x, double total) { return static_cast<double>(static_cast<float>(x) / 4294967295.0f) * total; }

// min{x in [lo, hi) : pred(x)} for a monotone predicate; hi when none.
template <class Pred>
uint64_t lower_bound_u32(uint64_t lo, uint64_t hi, Pred pred) {
    while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (pred(static_cast<uint32_t>(mid)))
            hi = mid;
        else
            lo = mid + 1;
    }
    return lo;
}

struct Thresholds {
    uint32_t xm = 0, xi = 0;
    std::vector<uint32_t> T;  // (S+1)^2
};

Thresholds compute_thresholds(double mobility, int64_t cells, const double* dom, int S) {
    // action_rates (params.hpp:61-70)
    const double mu = 1.0, sigma = 1.0, eps = 2.0 * mobility * static_cast<double>(cells);
    const double total = mu + sigma + eps;
    const double em = eps + mu;
    Thresholds t;
    const uint64_t xm = lower_bound_u32(0, uint64_t{1} << 32, [&](uint32_t x) { return r_of(x, total) >= eps; });
    const uint64_t xi = lower_bound_u32(0, uint64_t{1} << 32, [&](uint32_t x) { return r_of(x, total) >= em; });
    // r(2^32-1) = total >= eps + mu, so both exist.
    t.xm = static_cast<uint32_t>(std::min<uint64_t>(xm, 0xFFFFFFFFull));
    t.xi = static_cast<uint32_t>(std::min<uint64_t>(xi, 0xFFFFFFFFull));
    const int S1 = S + 1;
    t.T.assign(static_cast<size_t>(S1) * S1, t.xm);
    for (int a = 1; a <= S; ++a) {
        for (int b = 1; b <= S; ++b) {
            const double d = dom[static_cast<size_t>(a - 1) * S + (b - 1)];
            uint32_t T = t.xm;  // forward > 0.0 guard (engine.hpp:127,131): D == 0 never fires
            if (d > 0.0) {
                // u(x) = (r(x) - eps) / mu < d  ⇔  x < T  on [xm, xi)
                const uint64_t v = lower_bound_u32(t.xm, t.xi, [&](uint32_t x) { return (r_of(x, total) - eps) / mu >= d; });
                T = static_cast<uint32_t>(v);
            }
            t.T[static_cast<size_t>(a) * S1 + b] = T;
        }
    }
    return t;
}

// min{x : double(float(x)/4294967295.0f) >= p0} — the empty test of init_lattice (lattice.hpp:59).
// SLICED3 tables (oracle/escg_oracle.c orc_slice3_table, the definition): out[0..31] = T[1..32],
// T[0] = 2^32, T[g] = floor(T[g-1] (2^K-1) / 2^K); out[32..63] = S[0..31], the single-tile part of
// each first-tile interval; out[64 + 32 (m-1) + g] = C[m][g], the runs conditioned on a set bit.
constexpr int kSlice3Words = 64 + 31 * 32;
void slice3_table(int K, uint32_t* out) {
    const uint64_t num = (1ull << K) - 1ull;
    uint64_t T[33];
    T[0] = 1ull << 32;
    for (int g = 1; g <= 32; ++g) T[g] = (T[g - 1] * num) >> K;
    for (int g = 1; g <= 32; ++g) out[g - 1] = static_cast<uint32_t>(T[g]);
    for (int G = 0; G < 32; ++G) {
        uint64_t r = T[G] - T[G + 1];
        for (int i = 0; i < 31 - G; ++i) r = (r * num) >> K;
        out[32 + G] = static_cast<uint32_t>(T[G + 1] + r);
    }
    for (int i = 0; i < 31 * 32; ++i) out[64 + i] = 0u;
    for (int m = 1; m <= 31; ++m)
        for (int g = 1; g < m; ++g)
            out[64 + 32 * (m - 1) + g] = static_cast<uint32_t>(((T[g] - T[m]) << 32) / ((1ull << 32) - T[m]));
}

uint32_t empty_threshold(double p0) {
    if (!(p0 > 0.0)) return 0u;
    const uint64_t v = lower_bound_u32(0, uint64_t{1} << 32, [&](uint32_t x) {
        return static_cast<double>(static_cast<float>(x) / 4294967295.0f) >= p0;
    });
    return static_cast<uint32_t>(std::min<uint64_t>(v, 0xFFFFFFFFull));
}

int64_t align_num_randoms_or_throw(int64_t requested, int64_t cells) {
    if (cells < 1) config_error("cell count must be positive");
    if (requested < cells)
        config_error("numRandoms (" + std::to_string(requested) + ") must be at least the cell count (" +
                     std::to_string(cells) + ")");
    return requested / cells * cells;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        free();
        if (count == 0) return;
        CK(cudaMalloc(&p, sizeof(T) * count));
        n = count;
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { free(); }
};

}  // namespace

struct escg_dev {
    escg_params p{};
    int S = 0, S1 = 0, kind = 0, arity = 4, flux = 1, H = 0, L = 0;
    int64_t N = 0;
    int device = 0;
    int nrep = 1;
    int kernel = ESCG_KERNEL_TILE;
    int threads = 512;
    int smem = 0;
    int P = 0;
    int nby = 1, nbx = 1;
    int narrow = 0;  // draw format: 0 WIDE, 1 NARROW, 2 SLICED (bit-sliced block kernel)
    int K = 0;       // SLICED: action bit planes
    int npl = 2;     // SLICED: species-code bit planes
    int lpi = 1;     // SLICED: lanes per item (slice.cu)
    int qcap = 0;    // SLICED: deferred-tile queue capacity override (tests)
    bool sliced3 = false;  // SLICED3 draws (undecided masks drawn directly)
    int kmcs = 1;    // block kernel: MCS per launch (temporal blocking)
    bool persist = false;  // block kernel runs as one persistent cooperative launch per run/advance
    // SLICED single lattices on the persistent ring kernel (ring.cu): bands, shared memory, mailboxes
    bool ring = false;
    int ring_nb = 0, ring_smem = 0, ring_mbs = 0;
    // one part of a multi-part ring (escg_dev_create_ring_part): a row band whose ring kernel
    // exchanges boundary rows with the neighbouring parts' kernels through their inboxes
    bool ring_part = false, ring_connected = false;
    bool ring_chain = false;  // the state is a ring launch's: the neighbours flag their rows into it
    uint32_t ring_epoch = 0;  // ring launches since creation (identical on every part of a ring)
    escgd::RingPart rpart{};
    int bh_max = 0, bw_max = 0;
    int seam_np = 0;  // block kernel on a periodic lattice with seams: colour phases per MCS (4, 6, 9)
    int phase_table = 0;  // block kernel: per-launch phase-geometry table (few items per thread)
    // row-band engines (one band of a lattice sharded by rows): the local buffer holds
    // halo + band_rows + halo rows; local row r is global row (row0 + r) mod Hg
    int Hg = 0, row0 = 0, wrap_rows = 1;
    int nbands = 1, band = 0, band_start = 0, band_rows = 0, halo = 0;
    int rows_begin = 0, rows_count = 0;  // rows of the local buffer the engine owns (blocks, I/O)
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;  // the engine's stream; `stream` may be a caller's (escg_dev_set_stream)
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev_poll = nullptr;
    int32_t* h_status = nullptr;  // pinned, status polling of the block path
    Thresholds th;
    uint32_t x_empty = 0;
    std::vector<uint64_t> seeds;
    std::vector<int64_t> mcs;  // host mirror per replica
    std::vector<int> cur;      // block path: buffer holding replica r's lattice
    DevBuf<uint8_t> lat[2];
    DevBuf<uint32_t> pl[2];  // SLICED: bit-plane lattices during run/advance (slice.cu)
    bool planes_live = false;  // SLICED band engines between band steps: the state is pl[cur], not lat[cur]
    DevBuf<uint64_t> d_seeds, d_last;
    DevBuf<uint32_t> d_T;
    DevBuf<int64_t> d_mcs, d_nrec, d_tsteps;
    DevBuf<int32_t> d_status;
    DevBuf<uint64_t> d_tcounts;
    DevBuf<unsigned long long> d_acc;
    DevBuf<unsigned int> d_ticket;
    DevBuf<int> d_rows, d_cols, d_bad;
    DevBuf<int32_t> d_cur;
    DevBuf<unsigned long long> d_acc3;
    DevBuf<int32_t> d_i32;
    DevBuf<unsigned long long> d_mbox;
    DevBuf<unsigned int> d_decided;
    DevBuf<uint32_t> d_T3;
    int64_t trace_cap = 0;
    bool traced = false;
    double last_ms = 0.0;
    int64_t last_launches = 0;

    ~escg_dev() {
        if (h_status) cudaFreeHost(h_status);
        if (ev_poll) cudaEventDestroy(ev_poll);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        if (own_stream) cudaStreamDestroy(own_stream);
    }
};

namespace {

// Block-kernel decomposition: row splits at multiples of 4, column splits at multiples of 8 when
// L % 8 == 0 (keeps NARROW tile pairs aligned), minimising waves x computed window area.
size_t block_smem(int bh, int bw, int S1, int k, int* pitch, int seam_np = 0) {
    if (seam_np > 0) {
        // seam mode: margin 3 * phases * k on every side, byte-granular window, per-axis tile lists
        const int m = 3 * seam_np * k;
        const int Wh = bh + 2 * m, Ww = bw + 2 * m;
        const int P = (Ww + 15) & ~15;
        if (pitch) *pitch = P;
        return static_cast<size_t>(((Wh * P + 15) & ~15) + ((S1 * S1 * 8 + 15) & ~15) + 32 * 8 +
                                   (escgd::kMaxSpecies + 1) * 4 + 4 * P + 64 + 16 +
                                   3 * 16 * ((Wh / 2 + 2) + (Ww / 2 + 2)));
    }
    // pitch ≡ 0 (mod 128 bytes): see tile_dual (bank-conflict-light half-warp split)
    const int P = ((bw + 2 * escgd::margin_cols(k)) + 127) & ~127;
    if (pitch) *pitch = P;
    return static_cast<size_t>((((bh + 2 * escgd::margin_rows(k)) * P + 15) & ~15) + ((S1 * S1 * 8 + 15) & ~15) +
                               32 * 8 + (escgd::kMaxSpecies + 1) * 4 + 4 * P + 64);  // + scratch box
}

// Block-kernel decomposition: row splits at multiples of 4, column splits at multiples of 16 (8, 4)
// when L allows (TMA rows, NARROW pairs), and k MCS per launch (temporal blocking).  Model per MCS:
// waves x (mean valid area over the 4k phases + launch/load overhead / k), in cell units.
void plan_blocks(escg_dev* h, int sms, int smem_cap, int kmax, bool fixk) {
    // CTAs resident per SM by registers (65536 per SM, allocated in units of 8 per thread)
    const int regs = (escgd::block_kernel_registers(h->arity) + 7) / 8 * 8;
    const int cta_per_sm = std::max(1, std::min(2, 65536 / std::max(1, regs * h->threads)));
    sms *= cta_per_sm;
    smem_cap = std::min(smem_cap, (228 * 1024) / cta_per_sm - 1024);
    const int cu = (h->L % 16 == 0) ? 16 : ((h->L % 8 == 0) ? 8 : 4);
    // units: rows in 4s, columns in cu; a remainder (reflecting lattices of any size) joins the last
    // block, so split boundaries stay even (window origins even: tile parity = global parity)
    const int uy = std::max(1, h->rows_count / 4), ux = std::max(1, h->L / cu);
    const int ry_extra = h->rows_count - uy * 4, rx_extra = h->L - ux * cu;
    double best = 1e300;
    int bnby = 1, bnbx = 1, bk = 1;
    // launch + window load/store per launch, in cell units (measured on B200): 4e4 for
    // the L=3200-size blocks; smaller windows load faster, so the weight falls with the window
    // (15000 + 0.3 cells per window cell, capped at 4e4): one L=1000 lattice then runs 2 MCS per
    // launch (8.7e10 vs 8.0e10 attempts/s at 4), one L=200 lattice 3 (6.0e9 vs 5.7e9)
    const double kOverheadCells = 40000.0;
    // band engines keep the chunk they were created for (its halo depth, and every band of a lattice
    // must exchange halos at the same cadence); ESCG_BLOCK_K is an experiment knob for the rest
    const int kforce = fixk ? kmax : (std::getenv("ESCG_BLOCK_K") ? std::atoi(std::getenv("ESCG_BLOCK_K")) : 0);
    for (int k = 1; k <= kmax; ++k) {
        if (kforce > 0 && k != kforce) continue;
        for (int nby = 1; nby <= std::min(uy, 128); ++nby) {
            for (int nbx = 1; nbx <= std::min(ux, 128); ++nbx) {
                const int bh = ((uy + nby - 1) / nby) * 4 + std::max(0, ry_extra),
                          bw = ((ux + nbx - 1) / nbx) * cu + std::max(0, rx_extra);
                if (block_smem(bh, bw, h->S1, k, nullptr, h->seam_np) > static_cast<size_t>(smem_cap)) continue;
                const int64_t ctas = static_cast<int64_t>(nby) * nbx * h->nrep;
                const int64_t waves = (ctas + sms - 1) / sms;
                const double grow = 3.0 * (h->seam_np > 0 ? h->seam_np : 4) * k + 3.0;  // validity margin
                const double area = (bh + grow) * (bw + grow);
                const double win = static_cast<double>(bh + 2 * escgd::margin_rows(k)) * (bw + 2 * escgd::margin_cols(k));
                const double over = std::min(kOverheadCells, 15000.0 + 0.3 * win);
                const double cost = static_cast<double>(waves) * (area + over / k);
                if (cost < best * 0.999) {
                    best = cost;
                    bnby = nby;
                    bnbx = nbx;
                    bk = k;
                }
            }
        }
    }
    if (best == 1e300)
        config_error("no block decomposition of the " + std::to_string(h->rows_count) + "x" + std::to_string(h->L) +
                     " lattice fits the shared-memory budget");
    h->nby = bnby;
    h->nbx = bnbx;
    h->kmcs = bk;
    std::vector<int> rows(bnby + 1), cols(bnbx + 1);
    for (int i = 0; i <= bnby; ++i) rows[i] = h->rows_begin + static_cast<int>(static_cast<int64_t>(uy) * i / bnby) * 4;
    for (int i = 0; i <= bnbx; ++i) cols[i] = static_cast<int>(static_cast<int64_t>(ux) * i / bnbx) * cu;
    rows[bnby] = h->rows_begin + h->rows_count;
    cols[bnbx] = h->L;
    int bh = 0, bw = 0;
    for (int i = 0; i < bnby; ++i) bh = std::max(bh, rows[i + 1] - rows[i]);
    for (int i = 0; i < bnbx; ++i) bw = std::max(bw, cols[i + 1] - cols[i]);
    h->smem = static_cast<int>(block_smem(bh, bw, h->S1, bk, &h->P, h->seam_np));
    {
        // per-launch phase-geometry table: with 640-thread CTAs (96 registers) it wins at every size
        // measured (L=1000 +6%, 2048 +7%, 3200 +5%, 16384 +2%); the recomputing path stays for
        // comparison (ESCG_PHASE_TABLE=0)
        h->phase_table = 1;
        if (const char* pt = std::getenv("ESCG_PHASE_TABLE")) h->phase_table = std::atoi(pt) ? 1 : 0;
    }
    h->bh_max = bh;
    h->bw_max = bw;
    h->d_rows.alloc(rows.size());
    h->d_cols.alloc(cols.size());
    CK(cudaMemcpy(h->d_rows.p, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_cols.p, cols.data(), sizeof(int) * cols.size(), cudaMemcpyHostToDevice));
}

// Bit-sliced block decomposition (slice.cu): row splits at multiples of 4, column blocks of whole
// 128-column groups (block i covers [128 s_i + 64, 128 s_{i+1} + 64), its window the s_{i+1} - s_i + 1
// groups from s_i), k MCS per launch.  Work per CTA and MCS ~ (rows + 12k) x window width: the
// bit-parallel items cover whole groups whether or not their columns are valid.
void plan_slices(escg_dev* h, int sms, int smem_cap, int kmax, bool fixk) {
    const int nthr = escgd::slice_threads(h->lpi);
    const int regs = (escgd::slice_kernel_registers(h->npl, h->lpi) + 7) / 8 * 8;
    const int cta_per_sm = std::max(1, std::min(4, 65536 / std::max(1, regs * nthr)));
    sms *= cta_per_sm;
    const int GL = h->L / 128, uy = h->rows_count / 4;  // band engines: the band's rows only
    double best = 1e300;
    int bnby = 1, bnbx = 1, bk = 1;
    // launch + window load/store + wave tail, in cell units; fitted on B200 with the TMA window
    // load at L=16384: k = 1 1.52e12, k = 2 1.67e12 attempts/s; 1e5-2e5 picks k = 2, 3.8e5 k = 4
    // (1.49e12), the old 2e4 k = 1
    double overhead = 120000.0;
    if (const char* o = std::getenv("ESCG_SLICE_OVERHEAD")) overhead = std::atof(o);
    const int kforce = fixk ? kmax : (std::getenv("ESCG_BLOCK_K") ? std::atoi(std::getenv("ESCG_BLOCK_K")) : 0);
    for (int k = 1; k <= kmax; ++k) {
        if (kforce > 0 && k != kforce) continue;
        for (int nbx = 1; nbx <= GL; ++nbx) {
            const int Gw = (GL + nbx - 1) / nbx + 1;
            if (Gw > 32) continue;  // a warp holds whole window rows (lanes = groups)
            // lanes of a warp: floor(32 / (lpi Gw)) tile rows x Gw groups x lpi; the rest idle
            if ((32 / h->lpi) / Gw < 1) continue;
            const double lanes = 32.0 / (((32 / h->lpi) / Gw) * Gw * h->lpi);
            for (int nby = 1; nby <= std::min(uy, 512); ++nby) {
                const int bh = ((uy + nby - 1) / nby) * 4;
                const size_t smem = static_cast<size_t>(bh + 2 * escgd::margin_rows(k)) *
                                    escgd::slice_row_words(h->npl, Gw) * 4;
                if (smem > static_cast<size_t>(smem_cap)) continue;
                const int64_t ctas = static_cast<int64_t>(nby) * nbx * h->nrep;
                const int64_t waves = (ctas + sms - 1) / sms;
                const double area = (bh + 12.0 * k + 3.0) * 128.0 * Gw * lanes;
                const double cost = static_cast<double>(waves) * (area + overhead / k);
                if (cost < best * 0.999) {
                    best = cost;
                    bnby = nby;
                    bnbx = nbx;
                    bk = k;
                }
            }
        }
    }
    if (const char* sp = std::getenv("ESCG_SLICE_SPLIT")) {  // tests/experiments: "nby,nbx"
        int y = 0, x = 0;
        if (std::sscanf(sp, "%d,%d", &y, &x) == 2 && y >= 1 && y <= uy && x >= 1 && x <= GL &&
            (GL + x - 1) / x + 1 <= 32 &&
            static_cast<size_t>(((uy + y - 1) / y) * 4 + 2 * escgd::margin_rows(bk)) *
                    escgd::slice_row_words(h->npl, (GL + x - 1) / x + 1) * 4 <=
                static_cast<size_t>(smem_cap)) {
            bnby = y;
            bnbx = x;
        }
    }
    if (best == 1e300)
        config_error("no bit-sliced decomposition of the " + std::to_string(h->rows_count) + "x" + std::to_string(h->L) +
                     " lattice fits the shared-memory budget");
    h->nby = bnby;
    h->nbx = bnbx;
    h->kmcs = bk;
    std::vector<int> rows(bnby + 1), cols(bnbx + 1);
    for (int i = 0; i <= bnby; ++i) rows[i] = h->rows_begin + static_cast<int>(static_cast<int64_t>(uy) * i / bnby) * 4;
    for (int i = 0; i <= bnbx; ++i) cols[i] = static_cast<int>(static_cast<int64_t>(GL) * i / bnbx);
    int bh = 0, gw = 0;
    for (int i = 0; i < bnby; ++i) bh = std::max(bh, rows[i + 1] - rows[i]);
    for (int i = 0; i < bnbx; ++i) gw = std::max(gw, cols[i + 1] - cols[i] + 1);
    h->smem = (bh + 2 * escgd::margin_rows(bk)) * escgd::slice_row_words(h->npl, gw) * 4;
    h->bh_max = bh;
    h->bw_max = 128 * (gw - 1);
    h->threads = nthr;
    h->d_rows.alloc(rows.size());
    h->d_cols.alloc(cols.size());
    CK(cudaMemcpy(h->d_rows.p, rows.data(), sizeof(int) * rows.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->d_cols.p, cols.data(), sizeof(int) * cols.size(), cudaMemcpyHostToDevice));
}

escgd::RuleArgs rule_args(escg_dev* h) {
    const int LB = h->arity == 8 ? 5 : 4;
    // WIDE rule form (crs.cuh rule_wide, a kernel template parameter): branch-free unless
    // migrations dominate so much that whole warps usually take the migration branch (measured
    // crossovers: block kernel between P(migration) 0.968 and 0.990, tile kernel between 0.941 and
    // 0.976 — tools/wide_rule_sweep.py; branch-free is 23% faster at 0.8, branchy 27% at 0.99)
    uint32_t bf = static_cast<double>(h->th.xm) < 0.97 * 4294967296.0 ? 1u : 0u;
    if (const char* f = std::getenv("ESCG_WIDE_RULE")) bf = std::strcmp(f, "branchy") == 0 ? 0u : 1u;
    return escgd::RuleArgs{h->th.xm, h->th.xi, h->d_T.p, (h->th.xm >> (16 + LB)) << LB, bf};
}

escgd::RunArgs run_args(escg_dev* h, int64_t limit, int64_t interval, uint32_t flags, int tracked, bool trace) {
    escgd::RunArgs r{};
    r.mcs = h->d_mcs.p;
    r.status = h->d_status.p;
    r.last_counts = h->d_last.p;
    r.n_rec = h->d_nrec.p;
    r.trace_steps = trace ? h->d_tsteps.p : nullptr;
    r.trace_counts = trace ? h->d_tcounts.p : nullptr;
    r.trace_cap = trace ? h->trace_cap : 0;
    r.cur = h->d_cur.p;
    r.mcs_limit = limit;
    r.interval = interval;
    r.stop_flags = flags;
    r.tracked = tracked;
    return r;
}

void upload_mcs(escg_dev* h) {
    CK(cudaMemcpyAsync(h->d_mcs.p, h->mcs.data(), sizeof(int64_t) * h->nrep, cudaMemcpyHostToDevice, h->stream));
}

// Block path: bring every replica's lattice into buffer 0 so one launch serves all replicas.
// A single bit-sliced lattice (overlapped-tile kernel) keeps its state in bit planes between
// run/advance calls (pl[cur]); byte readers convert on demand (band_sync_bytes).
bool planes_resident(const escg_dev* h) {
    return h->narrow == 2 && !h->ring && h->nbands <= 1 && h->nrep == 1 && h->kernel == ESCG_KERNEL_BLOCK;
}

void normalize_buffers(escg_dev* h) {
    if (h->kernel != ESCG_KERNEL_BLOCK || h->planes_live) return;  // live planes: the bytes are stale
    for (int r = 0; r < h->nrep; ++r) {
        if (h->cur[r] != 0) {
            CK(cudaMemcpyAsync(h->lat[0].p + static_cast<size_t>(r) * h->N, h->lat[1].p + static_cast<size_t>(r) * h->N,
                               h->N, cudaMemcpyDeviceToDevice, h->stream));
            h->cur[r] = 0;
        }
    }
    for (int r = 1; r < h->nrep; ++r)
        if (h->mcs[r] != h->mcs[0]) config_error("block kernel requires all replicas at the same MCS");
}

uint8_t* replica_lat(escg_dev* h, int r) {
    return h->lat[h->kernel == ESCG_KERNEL_BLOCK ? h->cur[r] : 0].p + static_cast<size_t>(r) * h->N;
}

// The rows an engine owns (whole lattice, or the band of a band engine): I/O and counts use these.
uint8_t* owned_lat(escg_dev* h, int r) { return replica_lat(h, r) + static_cast<size_t>(h->rows_begin) * h->L; }
int64_t owned_cells(escg_dev* h) { return static_cast<int64_t>(h->rows_count) * h->L; }

// Bit-sliced band engines stepped one process per GPU (escg_dev_band_rows / escg_dev_band_step)
// stay in plane form between steps; byte readers convert back first.
void band_sync_bytes(escg_dev* h) {
    if (!h->planes_live) return;
    const int c = h->cur[0];
    CK(escgd::launch_from_planes(h->pl[0].p, h->pl[1].p, nullptr, c, h->lat[c].p, h->H, h->L, h->npl, 1, h->stream));
    // a ring part's planes stay the state (its neighbours read and write them across devices)
    if (!h->ring_part) h->planes_live = false;
}
void band_sync_planes(escg_dev* h) {
    if (h->planes_live) return;
    const int c = h->cur[0];
    CK(escgd::launch_to_planes(h->lat[c].p, h->pl[c].p, h->H, h->L, h->npl, 1, h->stream));
    h->planes_live = true;
}

// A ring part's state set from the host: planes now (a neighbour's next launch reads this part's
// rows from them), and no boundary-row flags to wait for at the next launch.
void ring_part_fresh(escg_dev* h) {
    if (!h->ring_part) return;
    CK(cudaMemsetAsync(h->d_status.p, 0xFF, sizeof(int32_t), h->stream));
    band_sync_planes(h);
    CK(cudaStreamSynchronize(h->stream));
    h->ring_chain = false;
}

void check_replica(escg_dev* h, int r) {
    if (r < 0 || r >= h->nrep) config_error("replica index out of range");
}

void timed_begin(escg_dev* h) { CK(cudaEventRecord(h->ev0, h->stream)); }
void timed_end(escg_dev* h, int64_t launches) {
    CK(cudaEventRecord(h->ev1, h->stream));
    CK(cudaEventSynchronize(h->ev1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, h->ev0, h->ev1));
    h->last_ms = ms;
    h->last_launches = launches;
}

// Block path: enqueue MCS [t, t+n) in launches of at most kmcs MCS, density record after the
// last one when `count_last`.  `launch_no` counts launches since the run start (buffer parity).
int64_t enqueue_block_steps(escg_dev* h, int64_t t, int64_t n, bool count_last, const escgd::RunArgs& run,
                            int64_t& launch_no) {
    escgd::BlockArgs a{};
    a.seeds = h->d_seeds.p;
    a.rule = rule_args(h);
    a.run = run;
    a.H = h->H;
    a.L = h->L;
    a.S = h->S;
    a.P = h->P;
    a.arity = h->arity;
    a.narrow = h->narrow;
    a.Hg = h->Hg;
    a.row0 = h->row0;
    a.wrap_rows = h->wrap_rows;
    a.reflect = h->flux ? 0 : 1;
    a.seam_np = h->seam_np;
    a.phase_table = h->phase_table;
    a.nby = h->nby;
    a.nbx = h->nbx;
    a.row_split = h->d_rows.p;
    a.col_split = h->d_cols.p;
    a.acc = h->d_acc.p;
    a.ticket = h->d_ticket.p;
    a.smem_bytes = h->smem;
    a.K = h->K;
    a.npl = h->npl;
    a.lpi = h->lpi;
    a.qcap = h->qcap;
    a.T3 = h->sliced3 ? h->d_T3.p : nullptr;
    a.step = 1;
    int64_t launches = 0;
    for (int64_t done = 0; done < n;) {
        const int k = static_cast<int>(std::min<int64_t>(h->kmcs, n - done));
        const int par = static_cast<int>(launch_no & 1);
        a.src = h->lat[par].p;
        a.dst = h->lat[1 - par].p;
        a.psrc = h->pl[par].p;
        a.pdst = h->pl[1 - par].p;
        a.dst_index = 1 - par;
        a.mcs = t + done;
        a.nmcs = k;
        done += k;
        a.count = (count_last && done == n) ? 1 : 0;
        if (h->narrow == 2)
            CK(escgd::launch_slice(a, h->nrep, h->stream));
        else
            CK(escgd::launch_block(a, h->nrep, h->threads, h->stream));
        ++launch_no;
        ++launches;
    }
    return launches;
}

// Ring path: the whole advance (record = 0; final lattice in plane buffer 1) or run (records at
// t0 + k*interval and at the limit; record k in plane buffer k & 1, named by cur) in one launch.
// A ring part whose launch gave up waiting for a neighbour (kStatusRingTimeout): raise.
void ring_part_check(escg_dev* h) {
    if (!h->ring_part) return;
    int32_t st = 0;
    CK(cudaMemcpyAsync(&st, h->d_status.p, sizeof(int32_t), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (st == escgd::kStatusRingTimeout)
        engine_error("multi-part ring: a neighbour part stopped answering (exchange timed out); the lattice is "
                     "invalid until set_lattice / init_lattice on every part");
}

// Ring launches of parts p[0..n): `together` = all on one device in ONE cooperative launch (the
// single-GPU form of the multi-GPU ring: the same kernel, cross-part traffic through the same
// inbox and plane pointers); otherwise one launch per part on its own device and stream, nothing
// synchronised between them (the kernels meet through their tagged inbox words).
void ring_parts_advance(escg_dev** p, int n, int64_t n_mcs, bool together) {
    if (n_mcs < 0) config_error("mcs count must be non-negative");
    for (int g = 0; g < n; ++g) {
        escg_dev* h = p[g];
        if (!h || !h->ring_part) config_error("not a ring part");
        if (!h->ring_connected) config_error("ring part not connected to its neighbours (escg_dev_ring_part_connect)");
        if (h->mcs[0] != p[0]->mcs[0] || h->cur[0] != p[0]->cur[0] || h->ring_epoch != p[0]->ring_epoch ||
            h->ring_chain != p[0]->ring_chain)
            config_error("ring parts are out of step");
    }
    if (n_mcs == 0) return;
    if (n_mcs > (int64_t{1} << 29)) config_error("ring launch too long (tags count 4 phases per MCS in 31 bits)");
    escgd::RingArgs a{};
    auto fill = [&](escg_dev* h) {
        a.seeds = h->d_seeds.p;
        a.rule = rule_args(h);
        a.run = run_args(h, 0, 1, 0, 0, false);
        a.H = h->Hg;  // the draws use global rows
        a.L = h->L;
        a.S = h->S;
        a.npl = h->npl;
        a.K = h->K;
        a.mcs0 = h->mcs[0];
        a.mcs_end = h->mcs[0] + n_mcs;
        a.record = 0;
        a.mbs = h->ring_mbs;
        a.acc = h->d_acc.p;
        a.ticket = h->d_ticket.p;
        a.T3 = nullptr;
        a.cur = h->cur[0];
        a.xset = static_cast<int>(h->ring_epoch & 1u);
        a.epoch = h->ring_epoch;
        a.wait_snap = h->ring_chain ? 1 : 0;
        a.timeout_ns = escgd::kRingPartTimeoutNs;
        if (const char* tv = std::getenv("ESCG_RING_TIMEOUT_S"))
            a.timeout_ns = static_cast<unsigned long long>(std::max(0.001, std::atof(tv)) * 1e9);
    };
    // per part: planes current, local mailboxes cleared, and the inbox set of the NEXT launch
    // cleared (the neighbours write it from their next launch on; this launch's set was cleared
    // by the previous one, before any neighbour could have started this launch)
    for (int g = 0; g < n; ++g) {
        escg_dev* h = p[g];
        CK(cudaSetDevice(h->device));
        band_sync_planes(h);
        const size_t local = static_cast<size_t>(h->ring_nb) * 4 * h->ring_mbs;
        const int nx = static_cast<int>((h->ring_epoch + 1) & 1u);
        CK(cudaMemsetAsync(h->d_mbox.p, 0, sizeof(unsigned long long) * local, h->stream));
        CK(cudaMemsetAsync(h->rpart.inbox + static_cast<size_t>(nx) * 4 * h->ring_mbs, 0,
                           sizeof(unsigned long long) * 4 * h->ring_mbs, h->stream));
        CK(cudaMemsetAsync(h->rpart.inbox + static_cast<size_t>(8) * h->ring_mbs + nx * 2, 0,
                           sizeof(unsigned long long) * 2, h->stream));
        // (the status stays as the last launch left it: a timed-out ring keeps failing until reset)
    }
    if (together) {
        int smem = 0, ctas = 0;
        for (int g = 0; g < n; ++g) {
            if (p[g]->device != p[0]->device) config_error("a single-launch ring group needs one device");
            smem = std::max(smem, p[g]->ring_smem);
            CK(cudaSetDevice(p[g]->device));
            CK(cudaStreamSynchronize(p[g]->stream));
        }
        fill(p[0]);
        a.nparts = n;
        a.smem_bytes = smem;
        for (int g = 0; g < n; ++g) {
            a.part[g] = p[g]->rpart;
            a.part[g].cta0 = ctas;
            ctas += p[g]->ring_nb;
        }
        CK(cudaSetDevice(p[0]->device));
        if (ctas > escgd::ring_capacity(p[0]->npl, smem, p[0]->device))
            config_error("ring group does not fit one device (" + std::to_string(ctas) + " co-resident CTAs): fewer CTAs per part");
        timed_begin(p[0]);
        CK(escgd::launch_ring(a, ctas, p[0]->stream));
        timed_end(p[0], 1);
        ring_part_check(p[0]);
    } else {
        for (int g = 0; g < n; ++g) {
            escg_dev* h = p[g];
            CK(cudaSetDevice(h->device));
            fill(h);
            a.nparts = 1;
            a.smem_bytes = h->ring_smem;
            a.part[0] = h->rpart;
            a.part[0].cta0 = 0;
            if (n == 1) timed_begin(h);
            CK(escgd::launch_ring(a, h->ring_nb, h->stream));
        }
        if (n == 1) {
            // one rank's part: device-ordered, the host does not wait (timings read lazily)
            CK(cudaEventRecord(p[0]->ev1, p[0]->stream));
            p[0]->last_launches = 1;
        } else {
            for (int g = 0; g < n; ++g) {
                CK(cudaSetDevice(p[g]->device));
                CK(cudaStreamSynchronize(p[g]->stream));
                ring_part_check(p[g]);
            }
        }
    }
    CK(cudaGetLastError());
    for (int g = 0; g < n; ++g) {
        escg_dev* h = p[g];
        h->cur[0] ^= 1;
        h->mcs[0] += n_mcs;
        ++h->ring_epoch;
        h->ring_chain = true;
        h->planes_live = true;
    }
}

void enqueue_ring(escg_dev* h, int64_t t0, int64_t t1, int record, const escgd::RunArgs& run) {
    escgd::RingArgs a{};
    a.pin = h->pl[0].p;
    a.pbuf[0] = h->pl[0].p;
    a.pbuf[1] = h->pl[1].p;
    a.seeds = h->d_seeds.p;
    a.rule = rule_args(h);
    a.run = run;
    a.H = h->H;
    a.L = h->L;
    a.S = h->S;
    a.npl = h->npl;
    a.K = h->K;
    a.mcs0 = t0;
    a.mcs_end = t1;
    a.record = record;
    a.mbox = h->d_mbox.p;
    a.mbs = h->ring_mbs;
    a.decided = h->d_decided.p;
    a.acc = h->d_acc.p;
    a.ticket = h->d_ticket.p;
    a.smem_bytes = h->ring_smem;
    a.qcap = h->qcap;
    a.T3 = h->sliced3 ? h->d_T3.p : nullptr;
    CK(cudaMemsetAsync(h->d_mbox.p, 0, sizeof(unsigned long long) * h->d_mbox.n, h->stream));
    CK(cudaMemsetAsync(h->d_decided.p, 0, sizeof(unsigned int), h->stream));
    CK(escgd::launch_ring(a, h->ring_nb, h->stream));
}

escgd::PersistArgs persist_args(escg_dev* h, const escgd::RunArgs& run) {
    escgd::PersistArgs pa{};
    escgd::BlockArgs& a = pa.b;
    a.seeds = h->d_seeds.p;
    a.rule = rule_args(h);
    a.run = run;
    a.H = h->H;
    a.L = h->L;
    a.S = h->S;
    a.P = h->P;
    a.arity = h->arity;
    a.narrow = h->narrow;
    a.Hg = h->Hg;
    a.row0 = h->row0;
    a.wrap_rows = h->wrap_rows;
    a.reflect = h->flux ? 0 : 1;
    a.seam_np = h->seam_np;
    a.phase_table = h->phase_table;
    a.nby = h->nby;
    a.nbx = h->nbx;
    a.row_split = h->d_rows.p;
    a.col_split = h->d_cols.p;
    a.smem_bytes = h->smem;
    pa.buf[0] = h->lat[0].p;
    pa.buf[1] = h->lat[1].p;
    pa.kmcs = h->kmcs;
    pa.acc3 = h->d_acc3.p;
    return pa;
}

void ensure_trace(escg_dev* h, int64_t records) {
    const int64_t cap = std::max<int64_t>(records, 1);
    const double bytes = static_cast<double>(cap) * h->nrep * (h->S1 * 8 + 8);
    if (bytes > 8e9) config_error("density trace too large for device memory; disable record_trace");
    if (h->trace_cap < cap) {
        h->d_tsteps.alloc(static_cast<size_t>(cap) * h->nrep);
        h->d_tcounts.alloc(static_cast<size_t>(cap) * h->nrep * h->S1);
        h->trace_cap = cap;
    }
}

void run_impl(escg_dev* h, int64_t limit, int64_t interval, uint32_t flags, int tracked, bool trace,
              int32_t* status_out) {
    if (interval < 1) config_error("sample interval must be positive");
    if (tracked < 0 || tracked > h->S) config_error("tracked species out of range");
    normalize_buffers(h);
    for (int r = 0; r < h->nrep; ++r)
        if (h->mcs[r] > limit) config_error("run limit is below the current MCS");
    int64_t span = 0;
    for (int r = 0; r < h->nrep; ++r) span = std::max(span, limit - h->mcs[r]);
    if (trace) ensure_trace(h, span / interval + 2);
    h->traced = trace;
    CK(cudaMemsetAsync(h->d_status.p, 0xFF, sizeof(int32_t) * h->nrep, h->stream));  // ESCG_RUNNING
    CK(cudaMemsetAsync(h->d_nrec.p, 0, sizeof(int64_t) * h->nrep, h->stream));
    upload_mcs(h);
    const escgd::RunArgs run = run_args(h, limit, interval, flags, tracked, trace);
    int64_t launches = 0;
    timed_begin(h);
    if (h->kernel == ESCG_KERNEL_TILE) {
        escgd::TileArgs a{};
        a.lat = h->lat[0].p;
        a.seeds = h->d_seeds.p;
        a.rule = rule_args(h);
        a.run = run;
        a.H = h->H;
        a.L = h->L;
        a.S = h->S;
        a.P = h->P;
        a.arity = h->arity;
        a.flux = h->flux;
        a.narrow = h->narrow;
        a.record = 1;
        a.smem_bytes = h->smem;
        a.one_per_sm = escgd::tile_one_per_sm(h->smem) ? 1 : 0;
        CK(escgd::launch_tile(a, h->nrep, h->threads, h->stream));
        launches = 1;
    } else if (h->persist) {
        CK(cudaMemsetAsync(h->d_acc3.p, 0, sizeof(unsigned long long) * 3 * h->S1 * h->nrep, h->stream));
        escgd::PersistArgs pa = persist_args(h, run);
        pa.mcs0 = h->mcs[0];
        pa.mcs_end = limit;
        pa.record = 1;
        CK(escgd::launch_block_persistent(pa, h->nrep, h->threads, h->stream));
        launches = 1;
    } else {
        CK(cudaMemsetAsync(h->d_acc.p, 0, sizeof(unsigned long long) * h->S1 * h->nrep, h->stream));
        CK(cudaMemsetAsync(h->d_ticket.p, 0, sizeof(unsigned int) * h->nrep, h->stream));
        const int64_t t0 = h->mcs[0];
        // a resident plane state (planes_resident) starts from its own buffer, with no conversion
        const bool live = h->planes_live && h->narrow == 2 && !h->ring;
        const int pc = live ? h->cur[0] : 0;
        int64_t launch_no = h->narrow == 2 ? pc : 0;
        // record at the starting MCS (record_and_check before any step, engine.cpp:181)
        escgd::BlockArgs a{};
        a.src = h->lat[0].p;
        a.dst = h->lat[1].p;
        a.seeds = h->d_seeds.p;
        a.rule = rule_args(h);
        a.run = run;
        a.H = h->H;
        a.L = h->L;
        a.S = h->S;
        a.P = h->P;
        a.arity = h->arity;
        a.narrow = h->narrow;
        a.Hg = h->Hg;
        a.row0 = h->row0;
        a.wrap_rows = h->wrap_rows;
        a.reflect = h->flux ? 0 : 1;
        a.seam_np = h->seam_np;
        a.phase_table = h->phase_table;
        a.nby = h->nby;
        a.nbx = h->nbx;
        a.row_split = h->d_rows.p;
        a.col_split = h->d_cols.p;
        a.mcs = t0;
        a.nmcs = 1;
        a.dst_index = 1;  // count-only: the lattice stays in buffer 0
        a.step = 0;
        a.count = 1;
        a.acc = h->d_acc.p;
        a.ticket = h->d_ticket.p;
        a.smem_bytes = h->smem;
        if (h->narrow == 2) {
            // SLICED: the run works on bit planes; the record at the start counts them
            if (!live) {
                CK(escgd::launch_to_planes(h->lat[0].p, h->pl[0].p, h->H, h->L, h->npl, h->nrep, h->stream));
                ++launches;
            }
            a.psrc = h->pl[pc].p;
            a.pdst = h->pl[1 - pc].p;
            a.dst_index = 1 - pc;  // count-only: the record names buffer pc
            a.K = h->K;
            a.npl = h->npl;
            a.lpi = h->lpi;
            a.qcap = h->qcap;
            CK(escgd::launch_slice(a, h->nrep, h->stream));
            ++launches;
        } else {
            CK(escgd::launch_block(a, h->nrep, h->threads, h->stream));
            ++launches;
        }
        if (h->ring) {
            // one persistent launch for the whole run (records and stop decisions on device)
            if (limit > t0) {
                enqueue_ring(h, t0, limit, 1, run);
                ++launches;
            }
            CK(escgd::launch_from_planes(h->pl[0].p, h->pl[1].p, h->d_cur.p, 0, h->lat[0].p, h->H, h->L, h->npl,
                                         h->nrep, h->stream));
            ++launches;
            timed_end(h, launches);
            CK(cudaGetLastError());
            std::vector<int32_t> st(h->nrep);
            CK(cudaMemcpy(h->mcs.data(), h->d_mcs.p, sizeof(int64_t) * h->nrep, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(st.data(), h->d_status.p, sizeof(int32_t) * h->nrep, cudaMemcpyDeviceToHost));
            if (status_out) std::memcpy(status_out, st.data(), sizeof(int32_t) * h->nrep);
            return;
        }
        // Poll the device status every few chunks so a stasis/stop does not leave thousands of
        // no-op launches queued; the poll lags one chunk behind the enqueue front.
        int32_t* hstat = h->h_status;
        cudaEvent_t polled = h->ev_poll;
        bool poll_pending = false;
        int64_t t = t0, since_poll = 0;
        const int64_t kChunk = 512;
        while (t < limit) {
            const int64_t adv = std::min(interval, limit - t);
            launches += enqueue_block_steps(h, t, adv, true, run, launch_no);
            t += adv;
            since_poll += adv;
            if (since_poll >= kChunk) {
                since_poll = 0;
                if (poll_pending) {
                    CK(cudaEventSynchronize(polled));
                    bool all_done = true;
                    for (int r = 0; r < h->nrep; ++r) all_done &= hstat[r] != ESCG_RUNNING;
                    if (all_done) break;
                }
                CK(cudaMemcpyAsync(hstat, h->d_status.p, sizeof(int32_t) * h->nrep, cudaMemcpyDeviceToHost, h->stream));
                CK(cudaEventRecord(polled, h->stream));
                poll_pending = true;
            }
        }
        if (h->narrow == 2 && !planes_resident(h)) {
            // back to bytes: the plane buffer named by the last record (cur = 2 + index)
            CK(escgd::launch_from_planes(h->pl[0].p, h->pl[1].p, h->d_cur.p, 0, h->lat[0].p, h->H, h->L, h->npl,
                                         h->nrep, h->stream));
            ++launches;
        }
    }
    timed_end(h, launches);
    if (planes_resident(h)) {  // the state stays in the plane buffer the last record names
        int32_t c = 0;
        CK(cudaMemcpy(&c, h->d_cur.p, sizeof(int32_t), cudaMemcpyDeviceToHost));
        h->cur[0] = c >= 2 ? c - 2 : h->cur[0];
        h->planes_live = true;
    }
    CK(cudaGetLastError());
    std::vector<int32_t> st(h->nrep);
    CK(cudaMemcpy(h->mcs.data(), h->d_mcs.p, sizeof(int64_t) * h->nrep, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(st.data(), h->d_status.p, sizeof(int32_t) * h->nrep, cudaMemcpyDeviceToHost));
    if (status_out) std::memcpy(status_out, st.data(), sizeof(int32_t) * h->nrep);
}

}  // namespace

// ================================== C ABI ======================================================

extern "C" {

const char* escg_dev_last_error(void) { return g_last_error.c_str(); }

int escg_params_default(escg_params* out) {
    return guarded([&] {
        if (!out) config_error("null params");
        escg_params p{};
        p.length = 200;
        p.height = 200;
        p.mcs_limit = 100000;
        p.neighbourhood = 4;
        p.print_frequency = 200;
        p.mobility = 3e-05;
        p.species = 3;
        p.flux = 1;
        p.empty_prob = 0.0;
        p.num_randoms = 100000000;
        *out = p;
    });
}

int escg_validate(const escg_params* p, const double* dominance, int32_t species, int32_t kind) {
    return guarded([&] {
        if (!p) config_error("null params");
        validate_params(*p);
        validate_dominance(dominance, species, kind);
        if (species != p->species)
            config_error("species count (" + std::to_string(p->species) + ") does not match dominance size (" +
                         std::to_string(species) + ")");
    });
}

int escg_action_rates(double mobility, int64_t cells, double* out4) {
    return guarded([&] {
        if (mobility < 0.0) config_error("mobility must be non-negative");
        if (cells < 1) config_error("cell count must be positive");
        out4[0] = 1.0;
        out4[1] = 1.0;
        out4[2] = 2.0 * mobility * static_cast<double>(cells);
        out4[3] = out4[0] + out4[1] + out4[2];
    });
}

int escg_thresholds(double mobility, int64_t cells, const double* dominance, int32_t species, uint32_t* out_xmx,
                    uint32_t* out_T) {
    return guarded([&] {
        if (mobility < 0.0) config_error("mobility must be non-negative");
        if (cells < 1) config_error("cell count must be positive");
        Thresholds t = compute_thresholds(mobility, cells, dominance, species);
        out_xmx[0] = t.xm;
        out_xmx[1] = t.xi;
        if (out_T) std::memcpy(out_T, t.T.data(), sizeof(uint32_t) * t.T.size());
    });
}

int64_t escg_align_num_randoms(int64_t requested, int64_t cells) {
    int64_t out = -1;
    const int rc = guarded([&] { out = align_num_randoms_or_throw(requested, cells); });
    return rc == ESCG_OK ? out : -1;
}

}  // extern "C"

namespace {
struct BandSpec {
    int nbands = 1, band = 0, kmcs = 2;
    int ring = 0, ctas = 0;  // multi-part ring: this part's bands (0: one per SM, >= 8 rows each)
};

void create_impl(const escg_params* p, const double* dominance, int32_t species, int32_t kind, int32_t device,
                 int32_t n_replicas, const uint64_t* replica_seeds, int32_t kernel, escg_dev** out,
                 const BandSpec* bs);
}  // namespace

extern "C" {

int escg_dev_create(const escg_params* p, const double* dominance, int32_t species, int32_t kind, int32_t device,
                    int32_t n_replicas, const uint64_t* replica_seeds, int32_t kernel, escg_dev** out) {
    return guarded([&] { create_impl(p, dominance, species, kind, device, n_replicas, replica_seeds, kernel, out, nullptr); });
}

int escg_dev_create_band(const escg_params* p, const double* dominance, int32_t species, int32_t kind, int32_t device,
                         int32_t n_bands, int32_t band, int32_t kmcs, escg_dev** out) {
    return guarded([&] {
        BandSpec bs;
        bs.nbands = n_bands;
        bs.band = band;
        bs.kmcs = kmcs > 0 ? kmcs : 2;
        create_impl(p, dominance, species, kind, device, 1, nullptr, ESCG_KERNEL_BLOCK, out, &bs);
    });
}

int escg_dev_create_ring_part(const escg_params* p, const double* dominance, int32_t species, int32_t kind,
                              int32_t device, int32_t n_parts, int32_t part, int32_t n_ctas, escg_dev** out) {
    return guarded([&] {
        BandSpec bs;
        bs.nbands = n_parts;
        bs.band = part;
        bs.kmcs = 1;
        bs.ring = 1;
        bs.ctas = n_ctas;
        create_impl(p, dominance, species, kind, device, 1, nullptr, ESCG_KERNEL_RING, out, &bs);
    });
}

}  // extern "C"

namespace {
void create_impl(const escg_params* p, const double* dominance, int32_t species, int32_t kind, int32_t device,
                 int32_t n_replicas, const uint64_t* replica_seeds, int32_t kernel, escg_dev** out,
                 const BandSpec* bs) {
    {
        if (!p || !out) config_error("null argument");
        *out = nullptr;
        validate_params(*p);
        validate_dominance(dominance, species, kind);
        if (species != p->species)
            config_error("species count (" + std::to_string(p->species) + ") does not match dominance size (" +
                         std::to_string(species) + ")");
        if (n_replicas < 1) config_error("replica count must be positive");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1)
            engine_error("no CUDA device available (the ESCG engine has no CPU fallback)");
        if (device < 0 || device >= ndev) config_error("CUDA device index out of range");
        CK(cudaSetDevice(device));
        auto h = std::make_unique<escg_dev>();
        h->p = *p;
        h->S = species;
        h->S1 = species + 1;
        h->kind = kind;
        h->arity = p->neighbourhood;
        h->flux = p->flux ? 1 : 0;
        h->H = p->height;
        h->L = p->length;
        h->N = static_cast<int64_t>(h->H) * h->L;
        h->device = device;
        h->nrep = n_replicas;
        // no seed: non-reproducible like the reference (std::random_device, engine.cpp:210)
        const uint64_t base_seed =
            p->has_seed ? p->seed : ((static_cast<uint64_t>(std::random_device{}()) << 32) | std::random_device{}());
        h->seeds.resize(n_replicas);
        for (int r = 0; r < n_replicas; ++r) h->seeds[r] = replica_seeds ? replica_seeds[r] : base_seed + r;
        h->th = compute_thresholds(p->mobility, h->N, dominance, species);
        h->x_empty = empty_threshold(p->empty_prob);
        h->mcs.assign(n_replicas, 0);
        h->cur.assign(n_replicas, 0);
        h->Hg = h->H;
        h->rows_begin = 0;
        h->rows_count = h->H;
        if (bs) {
            // band `band` of `nbands` row bands (multiples of 4 rows) plus halo rows on both sides
            if (bs->nbands < 2) config_error("a band engine needs at least 2 bands");
            if (bs->band < 0 || bs->band >= bs->nbands) config_error("band index out of range");
            if (bs->kmcs < 1 || bs->kmcs > escgd::kMaxBlockMcs) config_error("band chunk (kmcs) must be in [1, 4]");
            if (bs->ring && bs->nbands > escgd::kMaxRingParts)
                config_error("a multi-part ring has at most " + std::to_string(escgd::kMaxRingParts) + " parts");
            if (!(h->flux && h->H % 4 == 0 && h->L % 4 == 0)) config_error("band sharding needs a periodic lattice with L, H divisible by 4");
            if (n_replicas != 1) config_error("band engines hold one lattice");
            const int u = h->H / 4;
            h->nbands = bs->nbands;
            h->band = bs->band;
            h->band_start = static_cast<int>(static_cast<int64_t>(u) * bs->band / bs->nbands) * 4;
            h->band_rows = static_cast<int>(static_cast<int64_t>(u) * (bs->band + 1) / bs->nbands) * 4 - h->band_start;
            // a ring part keeps 2 halo rows per side (a slab reaches 1 row above and 2 below its band)
            h->halo = bs->ring ? 2 : escgd::margin_rows(bs->kmcs);
            if (bs->ring && h->band_rows < 8)
                config_error("ring part too thin (" + std::to_string(h->band_rows) + " rows < 8): use fewer parts");
            if (h->band_rows < h->halo)
                config_error("band too thin for the halo (" + std::to_string(h->band_rows) + " rows < " +
                             std::to_string(h->halo) + "): use fewer bands or a smaller chunk");
            h->H = h->band_rows + 2 * h->halo;
            h->N = static_cast<int64_t>(h->H) * h->L;
            h->row0 = ((h->band_start - h->halo) % h->Hg + h->Hg) % h->Hg;
            h->wrap_rows = 0;
            h->rows_begin = h->halo;
            h->rows_count = h->band_rows;
            h->kmcs = bs->kmcs;
        }

        cudaDeviceProp prop{};
        CK(cudaGetDeviceProperties(&prop, device));
        const int smem_cap = escgd::max_smem_optin(device);
        int tpitch = 0;
        const int tbytes = escgd::tile_smem_bytes(h->H, h->L, species, &tpitch);
        const bool periodic4 = h->flux && (h->H % 4 == 0) && (h->L % 4 == 0);
        if (h->flux && (h->H < 4 || h->L < 4))
            config_error("device engine: periodic lattices need L, H >= 4 (2x2 tiles, footprints may not wrap)");
        // tile-kernel CTA size: ~2.5 items (tile pairs) per thread and phase, so small lattices get
        // small CTAs and more replicas share an SM (measured: L=64 → 64 threads, L=100 → 128, L >= 200 → 512)
        int tile_threads;
        {
            const int64_t items = ((h->H + 3) / 4) * (int64_t)((h->L + 7) / 8);
            int64_t tt = (items * 2 / 5) / 32 * 32;
            tt = tt > 448 ? 512 : std::max<int64_t>(64, tt);
            const int cap = escgd::tile_one_per_sm(tbytes) ? escgd::kTileThreadsOne : escgd::kTileThreadsTwo;
            tile_threads = static_cast<int>(std::min<int64_t>(tt, cap));
            if (const char* tv = std::getenv("ESCG_TILE_THREADS"))
                tile_threads = std::max(32, std::min(cap, (std::atoi(tv) + 31) / 32 * 32));
        }
        if (kernel < ESCG_KERNEL_AUTO || kernel > ESCG_KERNEL_RING) config_error("unknown kernel selection");
        int choice = kernel == ESCG_KERNEL_RING ? ESCG_KERNEL_BLOCK : kernel;
        if (choice == ESCG_KERNEL_AUTO) {
            // one CTA per replica (tile) wins only when the replicas fill the device: at least one
            // per SM and a quarter of the tile kernel's concurrent CTAs; fewer lattices run faster
            // spread over all SMs by the block kernel (measured on B200: one L=200 lattice 5.2e9 vs
            // 1.5e9 attempts/s; 148 replicas of L=200 2.2e11 tile vs 1.7e11 block)
            choice = ESCG_KERNEL_BLOCK;
            if (tbytes <= smem_cap && !bs) {
                const int slots = escgd::tile_capacity(h->arity, h->flux, h->H, h->L, tile_threads, tbytes, device);
                if (n_replicas >= prop.multiProcessorCount && 4 * static_cast<int64_t>(n_replicas) >= slots)
                    choice = ESCG_KERNEL_TILE;
            }
        }
        if (choice == ESCG_KERNEL_TILE && tbytes > smem_cap)
            config_error("lattice too large for the shared-memory tile kernel");
        if (choice == ESCG_KERNEL_BLOCK && h->flux && !periodic4) {
            // seams on the block kernel: 2 or 3 colours per axis
            h->seam_np = (h->H % 4 == 0 ? 2 : 3) * (h->L % 4 == 0 ? 2 : 3);
        }
        h->kernel = choice;
        // NARROW (16-bit attempt words, one draw per tile pair) when migrations dominate so much that
        // at most 1/300 of attempts leave the coarse fast path (measured on B200: L=1000, M=1e-4 has
        // 1/100 slow and runs 24% faster WIDE; L=2000 ≈ 1/370 is even; L=3200 ≈ 1/800 is 17% faster
        // NARROW); needs periodic wrap with L, H ≡ 0 (mod 4) and L % 8 == 0.
        {
            const int LB = h->arity == 8 ? 5 : 4, CB = 16 - LB;
            const uint64_t fast_coarse = h->th.xm >> (32 - CB);
            h->narrow = (periodic4 && h->L % 8 == 0 && fast_coarse * 300 >= 299ull * (1ull << CB)) ? 1 : 0;
            if (const char* f = std::getenv("ESCG_DRAW_FORMAT")) {
                if (std::strcmp(f, "wide") == 0) h->narrow = 0;
                if (std::strcmp(f, "narrow") == 0 && periodic4 && h->L % 8 == 0) h->narrow = 1;
            }
        }
        // SLICED (bit-sliced block kernel, slice.cu): periodic von Neumann lattices with L % 128 == 0,
        // S <= 7 (row-band engines too), when at least 6 leading bits of X_mig are ones: K (even, <= 16,
        // <= those bits) action planes make every word with a zero among its top K bits a certain
        // migration.  Chosen by default from 8 leading ones (P(migration) >= 0.996).
        {
            int lead = 0;
            while (lead < 32 && ((h->th.xm >> (31 - lead)) & 1u)) ++lead;
            const bool ok = choice == ESCG_KERNEL_BLOCK && periodic4 && h->arity == 4 && h->L % 128 == 0 &&
                            h->S <= 7 && lead >= 6;
            bool use = ok && lead >= 8;
            if (const char* f = std::getenv("ESCG_DRAW_FORMAT")) use = ok && std::strcmp(f, "sliced") == 0;
            if (kernel == ESCG_KERNEL_RING) {
                if (!ok) config_error("the ring kernel needs the bit-sliced draw format (periodic von Neumann, L % 128 == 0, S <= 7, P(migration) >= 0.98)");
                use = true;
            }
            if (use) {
                h->narrow = 2;
                h->K = std::min(lead, escgd::kSliceMaxK) & ~1;
                if (const char* kv = std::getenv("ESCG_SLICE_K")) {  // experiments: fewer action planes
                    const int kf = std::atoi(kv) & ~1;
                    if (kf >= 6 && kf <= h->K) h->K = kf;
                }
                h->npl = h->S <= 3 ? 2 : 3;
                // one lane per item: measured faster than a lane pair at L=3200 (4.8e11 vs 4.3e11) and
                // even at L=16384 (8.8e11 vs 9.0e11); the pair stays selectable (ESCG_SLICE_LPI=2)
                h->lpi = 1;
                if (const char* lv = std::getenv("ESCG_SLICE_LPI")) h->lpi = (h->npl == 2 && std::atoi(lv) == 2) ? 2 : 1;
                if (const char* qv = std::getenv("ESCG_SLICE_QCAP")) h->qcap = std::atoi(qv);
                // SLICED3 (one draw word per attempt for the undecided masks instead of K) on the
                // overlapped-tile kernel; the ring kernel keeps SLICED (set below once it is chosen)
                h->sliced3 = true;
            }
        }
        CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
        h->stream = h->own_stream;
        CK(cudaEventCreate(&h->ev0));
        CK(cudaEventCreate(&h->ev1));
        CK(cudaEventCreateWithFlags(&h->ev_poll, cudaEventDisableTiming));
        CK(cudaMallocHost(&h->h_status, sizeof(int32_t) * n_replicas));
        h->lat[0].alloc(static_cast<size_t>(h->N) * n_replicas);
        if (choice == ESCG_KERNEL_TILE) {
            h->P = tpitch;
            h->smem = tbytes;
            h->threads = tile_threads;
        } else {
            h->lat[1].alloc(static_cast<size_t>(h->N) * n_replicas);
            // 640 threads per CTA at up to 96 registers (the kernel's launch bound): fewer warps, no
            // spills — faster than 1024 x 64 registers and than 2 x 512 per SM at every size measured
            h->threads = escgd::kBlockThreads;
            if (const char* tv = std::getenv("ESCG_BLOCK_THREADS")) {  // experiments: fewer threads
                const int t = std::atoi(tv);
                if (t >= 256 && t <= escgd::kBlockThreads && t % 32 == 0) h->threads = t;
            }
            int kmax = escgd::kMaxBlockMcs;
            if (const char* kv = std::getenv("ESCG_BLOCK_MCS")) kmax = std::max(1, std::min(kmax, std::atoi(kv)));
            if (bs) kmax = bs->kmcs;  // chunks may not outgrow the band's halo
            if (h->narrow == 2) {
                if (!(bs && bs->ring))
                    plan_slices(h.get(), prop.multiProcessorCount, std::min(smem_cap, 200 * 1024), kmax, bs != nullptr);
                const size_t words = static_cast<size_t>(h->H) * h->npl * (h->L / 128) * 4 * n_replicas;
                h->pl[0].alloc(words);
                h->pl[1].alloc(words);
            } else {
                plan_blocks(h.get(), prop.multiProcessorCount, std::min(smem_cap, 200 * 1024), kmax, bs != nullptr);
            }
            h->d_cur.alloc(n_replicas);
            // persistent cooperative mode: every CTA co-resident, 16-aligned columns (TMA rows and
            // vector stores) and a window that wraps at most once
            // opt-in (ESCG_PERSISTENT=1): bit-identical results, one launch per run, but measured
            // ~4% slower than one launch per chunk at L=3200 (grid.sync vs kernel boundary)
            const bool env_off = !(std::getenv("ESCG_PERSISTENT") && std::string(std::getenv("ESCG_PERSISTENT")) == "1");
            const bool geom_ok = h->L % 16 == 0 && h->bw_max % 16 == 0 &&
                                 h->bh_max + 2 * escgd::margin_rows(h->kmcs) <= h->H &&
                                 h->bw_max + 2 * escgd::margin_cols(h->kmcs) <= h->L;
            if (!env_off && geom_ok && h->wrap_rows && h->flux && h->narrow != 2) {
                const int cap = escgd::block_persistent_capacity(h->arity, h->threads, h->smem, device);
                h->persist = h->nby * h->nbx * n_replicas <= cap;
            }
            if (h->persist) h->d_acc3.alloc(static_cast<size_t>(3) * n_replicas * h->S1);
            // ring kernel (ring.cu): single periodic bit-sliced lattices whose rows fit one warp
            // (L/128 <= 32 groups), one band of >= 8 rows per SM.  AUTO takes it from L >= 1024
            // (8 busy lanes per warp); ESCG_KERNEL_RING forces it (tests: any L/128 <= 32).
            if (h->narrow == 2 && !bs && n_replicas == 1 &&
                (kernel == ESCG_KERNEL_RING ||
                 (kernel == ESCG_KERNEL_AUTO && !(std::getenv("ESCG_RING") && std::getenv("ESCG_RING")[0] == '0')))) {
                const int GL = h->L / 128;
                int nb = std::min(prop.multiProcessorCount, h->H / 8);
                if (const char* nv = std::getenv("ESCG_RING_NB")) nb = std::max(2, std::min(nb, std::atoi(nv)));
                int coop = 0;
                CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
                const int rsmem = nb >= 2 ? escgd::ring_smem_bytes(h->H, h->L, h->npl, nb) : 0;
                const bool ok = coop && nb >= 2 && GL <= 32 && (kernel == ESCG_KERNEL_RING || GL >= 8) &&
                                rsmem <= std::min(smem_cap, 200 * 1024) &&
                                nb <= escgd::ring_capacity(h->npl, rsmem, device);
                if (ok) {
                    h->ring = true;
                    // measured on B200 at L=3200: SLICED 6.5e11 vs SLICED3 6.0e11 attempts/s on the ring
                    // (its phase is bound by the boundary slabs, whose draws producer warps make ahead),
                    // while SLICED3 lifts the overlapped-tile kernel at L=16384 from 8.6e11 to 1.08e12
                    h->sliced3 = false;
                    h->ring_nb = nb;
                    h->ring_smem = rsmem;
                    h->ring_mbs = 2 + 3 * h->npl * GL * 4;
                    h->d_mbox.alloc(static_cast<size_t>(nb) * 4 * h->ring_mbs);
                    h->d_decided.alloc(1);
                } else if (kernel == ESCG_KERNEL_RING) {
                    config_error("lattice not eligible for the ring kernel (L/128 <= 32, H >= 16, co-resident bands)");
                }
            }
            if (bs && bs->ring) {
                // one part of a multi-part ring: bands of >= 8 rows of this part, co-resident (the
                // group emulation on one device checks the sum of its parts at launch)
                const int GL = h->L / 128;
                int nb = bs->ctas > 0 ? bs->ctas : prop.multiProcessorCount;
                nb = std::min(nb, h->band_rows / 8);
                int coop = 0;
                CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
                const int rsmem = nb >= 1 ? escgd::ring_smem_bytes(h->band_rows, h->L, h->npl, nb) : 0;
                if (!(h->narrow == 2 && coop && nb >= 1 && GL <= 32 && rsmem <= std::min(smem_cap, 200 * 1024) &&
                      nb <= escgd::ring_capacity(h->npl, rsmem, device)))
                    config_error("lattice not eligible for a multi-part ring (bit-sliced, L/128 <= 32, parts of >= 8 rows)");
                h->ring = true;
                h->ring_part = true;
                h->sliced3 = false;
                h->ring_nb = nb;
                h->ring_smem = rsmem;
                h->ring_mbs = 2 + 3 * h->npl * GL * 4;
                const size_t local = static_cast<size_t>(nb) * 4 * h->ring_mbs;
                h->d_mbox.alloc(local + escgd::kRingInboxWords(h->ring_mbs));
                CK(cudaMemset(h->d_mbox.p, 0, sizeof(unsigned long long) * h->d_mbox.n));
                h->rpart.pl[0] = h->pl[0].p;
                h->rpart.pl[1] = h->pl[1].p;
                h->rpart.mbox = h->d_mbox.p;
                h->rpart.inbox = h->d_mbox.p + local;
                h->rpart.r0 = h->band_start;
                h->rpart.rows = h->band_rows;
                h->rpart.nb = nb;
            }
            h->d_acc.alloc(static_cast<size_t>(h->S1) * n_replicas);
            h->d_ticket.alloc(n_replicas);
        }
        if (h->narrow == 2) {  // explicit choice of the sliced draw format (tests, experiments)
            if (const char* dv = std::getenv("ESCG_SLICE_DRAWS")) h->sliced3 = std::atoi(dv) != 2;
        }
        if (h->sliced3) {
            std::vector<uint32_t> t3(kSlice3Words);
            slice3_table(h->K, t3.data());
            h->d_T3.alloc(kSlice3Words);
            CK(cudaMemcpy(h->d_T3.p, t3.data(), sizeof(uint32_t) * kSlice3Words, cudaMemcpyHostToDevice));
        }
        h->d_seeds.alloc(n_replicas);
        h->d_last.alloc(static_cast<size_t>(h->S1) * n_replicas);
        h->d_T.alloc(h->th.T.size());
        h->d_mcs.alloc(n_replicas);
        h->d_nrec.alloc(n_replicas);
        h->d_status.alloc(n_replicas);
        h->d_bad.alloc(1);
        CK(cudaMemcpy(h->d_seeds.p, h->seeds.data(), sizeof(uint64_t) * n_replicas, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(h->d_T.p, h->th.T.data(), sizeof(uint32_t) * h->th.T.size(), cudaMemcpyHostToDevice));
        CK(cudaMemset(h->lat[0].p, 0, static_cast<size_t>(h->N) * n_replicas));
        CK(cudaMemset(h->d_status.p, 0xFF, sizeof(int32_t) * n_replicas));
        CK(cudaMemset(h->d_nrec.p, 0, sizeof(int64_t) * n_replicas));
        CK(cudaMemset(h->d_last.p, 0, sizeof(uint64_t) * h->S1 * n_replicas));
        *out = h.release();
    }
}
}  // namespace

extern "C" {

int escg_dev_destroy(escg_dev* h) {
    return guarded([&] {
        if (!h) return;
        cudaSetDevice(h->device);
        delete h;
    });
}

int escg_dev_init_lattice(escg_dev* h) {
    return guarded([&] {
        if (!h) config_error("null handle");
        CK(cudaSetDevice(h->device));
        escgd::InitArgs a{};
        a.lat = h->lat[0].p;
        a.seeds = h->d_seeds.p;
        a.n = h->N;
        a.L = h->L;
        a.Hg = h->Hg;
        a.row0 = h->row0;
        a.nrep = h->nrep;
        a.S = h->S;
        a.x_empty = h->x_empty;
        a.all_empty = h->p.empty_prob >= 1.0 ? 1 : 0;
        CK(escgd::launch_init(a, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        std::fill(h->mcs.begin(), h->mcs.end(), 0);
        std::fill(h->cur.begin(), h->cur.end(), 0);
        h->planes_live = false;
        ring_part_fresh(h);
    });
}

int escg_dev_set_lattice(escg_dev* h, int32_t replica, const int32_t* cells, int64_t mcs) {
    return guarded([&] {
        if (!h || !cells) config_error("null argument");
        check_replica(h, replica);
        if (mcs < 0) config_error("mcs must be non-negative");
        CK(cudaSetDevice(h->device));
        const int64_t n = owned_cells(h);
        if (h->d_i32.n < static_cast<size_t>(n)) h->d_i32.alloc(n);
        CK(cudaMemcpyAsync(h->d_i32.p, cells, sizeof(int32_t) * n, cudaMemcpyHostToDevice, h->stream));
        CK(cudaMemsetAsync(h->d_bad.p, 0, sizeof(int), h->stream));
        CK(escgd::launch_i32_to_u8(h->d_i32.p, owned_lat(h, replica), n, h->S, h->d_bad.p, h->stream));
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, h->d_bad.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
        if (bad) throw Error(ESCG_EENGINE, "corrupt lattice value (outside [0, S])");
        h->mcs[replica] = mcs;
        h->planes_live = false;
        ring_part_fresh(h);
    });
}

int escg_dev_get_lattice(escg_dev* h, int32_t replica, int32_t* out, int64_t* mcs_out) {
    return guarded([&] {
        if (!h) config_error("null handle");
        check_replica(h, replica);
        CK(cudaSetDevice(h->device));
        band_sync_bytes(h);
        ring_part_check(h);
        if (out) {
            const int64_t n = owned_cells(h);
            if (h->d_i32.n < static_cast<size_t>(n)) h->d_i32.alloc(n);
            CK(escgd::launch_u8_to_i32(owned_lat(h, replica), h->d_i32.p, n, h->stream));
            CK(cudaMemcpyAsync(out, h->d_i32.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, h->stream));
            CK(cudaStreamSynchronize(h->stream));
        }
        if (mcs_out) *mcs_out = h->mcs[replica];
    });
}

int escg_dev_counts(escg_dev* h, int32_t replica, uint64_t* out) {
    return guarded([&] {
        if (!h || !out) config_error("null argument");
        check_replica(h, replica);
        CK(cudaSetDevice(h->device));
        band_sync_bytes(h);
        ring_part_check(h);
        DevBuf<unsigned long long> tmp;
        tmp.alloc(h->S1);
        CK(escgd::launch_count(owned_lat(h, replica), owned_cells(h), 1, h->S, tmp.p, h->stream));
        CK(cudaMemcpyAsync(out, tmp.p, sizeof(uint64_t) * h->S1, cudaMemcpyDeviceToHost, h->stream));
        CK(cudaStreamSynchronize(h->stream));
    });
}

int escg_dev_advance(escg_dev* h, int64_t n_mcs) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (h->ring_part) {  // this process's part of a multi-part ring (one rank per GPU)
            ring_parts_advance(&h, 1, n_mcs, false);
            return;
        }
        if (h->nbands > 1) config_error("band engines advance through escg_group_advance");
        if (n_mcs < 0) config_error("mcs count must be non-negative");
        CK(cudaSetDevice(h->device));
        normalize_buffers(h);
        int64_t launches = 0;
        if (h->kernel == ESCG_KERNEL_TILE) {
            upload_mcs(h);
            escgd::TileArgs a{};
            a.lat = h->lat[0].p;
            a.seeds = h->d_seeds.p;
            a.rule = rule_args(h);
            a.run = run_args(h, 0, 1, 0, 0, false);
            a.H = h->H;
            a.L = h->L;
            a.S = h->S;
            a.P = h->P;
            a.arity = h->arity;
            a.flux = h->flux;
            a.narrow = h->narrow;
            a.record = 0;
            a.smem_bytes = h->smem;
            a.one_per_sm = escgd::tile_one_per_sm(h->smem) ? 1 : 0;
            // per-replica limit: all replicas advance by n_mcs from their own MCS; the kernel
            // reads mcs[r] and runs to mcs_limit, so stage limit = mcs + n per replica by
            // shifting: launch once per distinct starting MCS.
            std::vector<int64_t> starts(h->mcs);
            std::sort(starts.begin(), starts.end());
            starts.erase(std::unique(starts.begin(), starts.end()), starts.end());
            if (starts.size() != 1) config_error("advance requires all replicas at the same MCS");
            a.run.mcs_limit = starts[0] + n_mcs;
            timed_begin(h);
            CK(escgd::launch_tile(a, h->nrep, h->threads, h->stream));
            launches = 1;
            timed_end(h, launches);
            for (auto& m : h->mcs) m += n_mcs;
        } else if (h->persist) {
            const escgd::RunArgs run = run_args(h, 0, 1, 0, 0, false);
            CK(cudaMemsetAsync(h->d_status.p, 0xFF, sizeof(int32_t) * h->nrep, h->stream));
            upload_mcs(h);
            escgd::PersistArgs pa = persist_args(h, run);
            pa.mcs0 = h->mcs[0];
            pa.mcs_end = h->mcs[0] + n_mcs;
            pa.record = 0;
            timed_begin(h);
            CK(escgd::launch_block_persistent(pa, h->nrep, h->threads, h->stream));
            launches = 1;
            timed_end(h, launches);
            std::vector<int32_t> cur(h->nrep);
            CK(cudaMemcpy(cur.data(), h->d_cur.p, sizeof(int32_t) * h->nrep, cudaMemcpyDeviceToHost));
            for (int r = 0; r < h->nrep; ++r) {
                h->mcs[r] += n_mcs;
                h->cur[r] = cur[r];
            }
        } else {
            const escgd::RunArgs run = run_args(h, 0, 1, 0, 0, false);
            CK(cudaMemsetAsync(h->d_status.p, 0xFF, sizeof(int32_t) * h->nrep, h->stream));
            const int64_t t0 = h->mcs[0];
            int64_t launch_no = 0;
            timed_begin(h);
            if (h->ring && n_mcs > 0) {
                CK(escgd::launch_to_planes(h->lat[0].p, h->pl[0].p, h->H, h->L, h->npl, h->nrep, h->stream));
                enqueue_ring(h, t0, t0 + n_mcs, 0, run);  // final lattice in plane buffer 1
                CK(escgd::launch_from_planes(h->pl[0].p, h->pl[1].p, nullptr, 1, h->lat[0].p, h->H, h->L, h->npl,
                                             h->nrep, h->stream));
                launches = 3;
            } else if (h->narrow == 2 && n_mcs > 0) {
                const bool live = h->planes_live;
                launch_no = live ? h->cur[0] : 0;
                if (!live) {
                    CK(escgd::launch_to_planes(h->lat[0].p, h->pl[0].p, h->H, h->L, h->npl, h->nrep, h->stream));
                    ++launches;
                }
                launches += enqueue_block_steps(h, t0, n_mcs, false, run, launch_no);
                if (planes_resident(h)) {
                    h->planes_live = true;  // the state stays in plane buffer launch_no & 1
                } else {
                    CK(escgd::launch_from_planes(h->pl[0].p, h->pl[1].p, nullptr, static_cast<int>(launch_no & 1),
                                                 h->lat[0].p, h->H, h->L, h->npl, h->nrep, h->stream));
                    ++launches;
                    launch_no = 0;  // the lattice is back in byte buffer 0
                }
            } else if (h->narrow != 2) {
                launches = enqueue_block_steps(h, t0, n_mcs, false, run, launch_no);
            }
            timed_end(h, launches);
            for (int r = 0; r < h->nrep; ++r) {
                h->mcs[r] += n_mcs;
                if (n_mcs > 0 || h->narrow != 2) h->cur[r] = static_cast<int>(launch_no & 1);
            }
        }
        CK(cudaGetLastError());
    });
}

int escg_dev_run(escg_dev* h, int64_t mcs_limit, int64_t interval, uint32_t stop_flags, int32_t tracked_species,
                 int32_t record_trace, int32_t* status_out) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (h->ring_part) config_error("ring parts advance through escg_dev_advance / escg_ring_group_advance");
        if (h->nbands > 1) config_error("band engines advance through escg_group_advance");
        CK(cudaSetDevice(h->device));
        const std::vector<int64_t> start(h->mcs);
        run_impl(h, mcs_limit, interval, stop_flags, tracked_species, record_trace != 0, status_out);
        (void)start;
        if (planes_resident(h))
            ;  // the state stays in plane buffer cur[0] (run_impl)
        else if (h->kernel == ESCG_KERNEL_BLOCK && h->narrow == 2)
            std::fill(h->cur.begin(), h->cur.end(), 0);  // converted back into byte buffer 0
        else if (h->kernel == ESCG_KERNEL_BLOCK)
            CK(cudaMemcpy(h->cur.data(), h->d_cur.p, sizeof(int32_t) * h->nrep, cudaMemcpyDeviceToHost));
    });
}

int escg_dev_read_trace(escg_dev* h, int32_t replica, int64_t* steps, uint64_t* counts, int64_t cap, int64_t* n_out) {
    return guarded([&] {
        if (!h) config_error("null handle");
        check_replica(h, replica);
        CK(cudaSetDevice(h->device));
        int64_t n = 0;
        CK(cudaMemcpy(&n, h->d_nrec.p + replica, sizeof(int64_t), cudaMemcpyDeviceToHost));
        if (n_out) *n_out = n;
        if (!h->traced) return;
        const int64_t m = std::min({n, cap, h->trace_cap});
        if (m <= 0) return;
        if (steps)
            CK(cudaMemcpy(steps, h->d_tsteps.p + static_cast<size_t>(replica) * h->trace_cap, sizeof(int64_t) * m,
                          cudaMemcpyDeviceToHost));
        if (counts)
            CK(cudaMemcpy(counts, h->d_tcounts.p + static_cast<size_t>(replica) * h->trace_cap * h->S1,
                          sizeof(uint64_t) * m * h->S1, cudaMemcpyDeviceToHost));
    });
}

int escg_dev_replica_result(escg_dev* h, int32_t replica, int64_t* mcs, int32_t* status, uint64_t* last_counts) {
    return guarded([&] {
        if (!h) config_error("null handle");
        check_replica(h, replica);
        CK(cudaSetDevice(h->device));
        if (mcs) *mcs = h->mcs[replica];
        if (status) CK(cudaMemcpy(status, h->d_status.p + replica, sizeof(int32_t), cudaMemcpyDeviceToHost));
        if (last_counts)
            CK(cudaMemcpy(last_counts, h->d_last.p + static_cast<size_t>(replica) * h->S1, sizeof(uint64_t) * h->S1,
                          cudaMemcpyDeviceToHost));
    });
}

int escg_dev_replay(escg_dev* h, const uint32_t* w_cell, const uint32_t* w_dir, const uint32_t* w_act, int64_t n) {
    return guarded([&] {
        if (!h || !w_cell || !w_dir || !w_act) config_error("null argument");
        if (n < 0) config_error("attempt count must be non-negative");
        CK(cudaSetDevice(h->device));
        band_sync_bytes(h);
        normalize_buffers(h);
        DevBuf<uint32_t> wc, wd, wa;
        wc.alloc(std::max<int64_t>(n, 1));
        wd.alloc(std::max<int64_t>(n, 1));
        wa.alloc(std::max<int64_t>(n, 1));
        CK(cudaMemcpy(wc.p, w_cell, sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(wd.p, w_dir, sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(wa.p, w_act, sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
        escgd::ReplayArgs a{};
        a.lat = replica_lat(h, 0);
        a.wc = wc.p;
        a.wd = wd.p;
        a.wa = wa.p;
        a.n_attempts = n;
        a.rule = rule_args(h);
        a.H = h->H;
        a.L = h->L;
        a.S = h->S;
        a.arity = h->arity;
        a.flux = h->flux;
        timed_begin(h);
        CK(escgd::launch_replay(a, h->stream));
        timed_end(h, 1);
    });
}

int escg_dev_last_timing(escg_dev* h, double* ms, int64_t* launches) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (ms) *ms = h->last_ms;
        if (launches) *launches = h->last_launches;
    });
}

int escg_dev_describe(escg_dev* h, int32_t* kernel, int32_t* grid_ctas, int32_t* threads, int32_t* smem_bytes) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (kernel) *kernel = h->ring ? ESCG_KERNEL_RING : h->kernel;
        if (grid_ctas) *grid_ctas = h->ring ? h->ring_nb : (h->kernel == ESCG_KERNEL_TILE ? h->nrep : h->nby * h->nbx * h->nrep);
        if (threads) *threads = h->ring ? escgd::kRingThreads : h->threads;
        if (smem_bytes) *smem_bytes = h->ring ? h->ring_smem : h->smem;
    });
}

int escg_dev_block_mode(escg_dev* h, int32_t* kmcs, int32_t* persistent) {
    return guarded([&] {
        if (!h) config_error("null argument");
        if (kmcs) *kmcs = h->ring ? 0 : (h->kernel == ESCG_KERNEL_BLOCK ? h->kmcs : 1);
        if (persistent) *persistent = (h->kernel == ESCG_KERNEL_BLOCK && (h->persist || h->ring)) ? 1 : 0;
    });
}

int escg_dev_band_info(escg_dev* h, int32_t* band_start, int32_t* band_rows, int32_t* halo, int32_t* kmcs) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (band_start) *band_start = h->nbands > 1 ? h->band_start : 0;
        if (band_rows) *band_rows = h->nbands > 1 ? h->band_rows : h->H;
        if (halo) *halo = h->nbands > 1 ? h->halo : 0;
        if (kmcs) *kmcs = h->kernel == ESCG_KERNEL_BLOCK ? h->kmcs : 1;
    });
}

// One group of band engines (one band each, any devices): chunks of k MCS; before each chunk every
// band pulls its halo rows from its two ring neighbours' current buffers (cudaMemcpyPeerAsync), then
// runs the block kernel on its band.  Streams are ordered with events, so bands on different GPUs
// overlap; on one GPU the group is the bit-exact single-process reference of the sharded run.
int escg_group_advance(escg_dev** bands, int32_t n, int64_t n_mcs) {
    return guarded([&] {
        if (!bands || n < 2) config_error("a band group needs at least 2 bands");
        if (n_mcs < 0) config_error("mcs count must be non-negative");
        for (int g = 0; g < n; ++g) {
            escg_dev* h = bands[g];
            if (!h || h->nbands != n || h->band != g) config_error("group must list bands 0..n-1 of one lattice");
            if (h->ring_part) config_error("ring parts advance through escg_ring_group_advance");
            if (h->mcs[0] != bands[0]->mcs[0] || h->cur[0] != bands[0]->cur[0] || h->kmcs != bands[0]->kmcs)
                config_error("bands are out of step");
            if (h->narrow != bands[0]->narrow || h->K != bands[0]->K || h->npl != bands[0]->npl)
                config_error("bands must share one draw format");
        }
        // peer access between ring neighbours on different GPUs (NVLink P2P copies)
        for (int g = 0; g < n; ++g) {
            for (int nb : {(g + n - 1) % n, (g + 1) % n}) {
                const int d0 = bands[g]->device, d1 = bands[nb]->device;
                int can = 0;
                if (d0 != d1 && cudaDeviceCanAccessPeer(&can, d0, d1) == cudaSuccess && can) {
                    CK(cudaSetDevice(d0));
                    const cudaError_t pe = cudaDeviceEnablePeerAccess(d1, 0);
                    if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
                    cudaGetLastError();  // clear "already enabled"
                }
            }
        }
        // per-band ordering events, destroyed on every exit path
        struct Events {
            std::vector<cudaEvent_t> k, x;
            std::vector<int> dev;
            ~Events() {
                for (size_t g = 0; g < k.size(); ++g) {
                    cudaSetDevice(dev[g]);
                    if (k[g]) cudaEventDestroy(k[g]);
                    if (x[g]) cudaEventDestroy(x[g]);
                }
            }
        } ev;
        ev.k.assign(n, nullptr);
        ev.x.assign(n, nullptr);
        ev.dev.assign(n, 0);
        std::vector<cudaEvent_t>& ev_k = ev.k;
        std::vector<cudaEvent_t>& ev_x = ev.x;
        for (int g = 0; g < n; ++g) {
            ev.dev[g] = bands[g]->device;
            CK(cudaSetDevice(bands[g]->device));
            CK(cudaEventCreateWithFlags(&ev_k[g], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_x[g], cudaEventDisableTiming));
        }
        const int64_t t0 = bands[0]->mcs[0];
        int64_t launch_no = 0;
        int par = bands[0]->cur[0];
        const int k = bands[0]->kmcs;
        // bit-sliced bands stay in plane form for the whole call: halos move as plane rows
        const bool sliced = bands[0]->narrow == 2 && n_mcs > 0;
        for (int g = 0; g < n; ++g) {
            escg_dev* h = bands[g];
            CK(cudaSetDevice(h->device));
            if (sliced) band_sync_planes(h);
            CK(cudaEventRecord(ev_k[g], h->stream));
        }
        for (int64_t done = 0; done < n_mcs;) {
            const int chunk = static_cast<int>(std::min<int64_t>(k, n_mcs - done));
            // halo exchange into buffer `par` (reads the neighbours' band rows of buffer `par`)
            for (int g = 0; g < n; ++g) {
                escg_dev* h = bands[g];
                escg_dev* up = bands[(g + n - 1) % n];
                escg_dev* dn = bands[(g + 1) % n];
                CK(cudaSetDevice(h->device));
                CK(cudaStreamWaitEvent(h->stream, ev_k[(g + n - 1) % n], 0));
                CK(cudaStreamWaitEvent(h->stream, ev_k[(g + 1) % n], 0));
                // a row: L bytes, or NPL planes x L/128 groups x 4 words when bit-sliced
                const size_t rowb = sliced ? static_cast<size_t>(h->npl) * (h->L / 128) * 16 : static_cast<size_t>(h->L);
                const size_t hb = static_cast<size_t>(h->halo) * rowb;
                auto buf = [&](escg_dev* e) {
                    return sliced ? reinterpret_cast<uint8_t*>(e->pl[par].p) : e->lat[par].p;
                };
                uint8_t* mine = buf(h);
                // top halo ← the last `halo` rows of the band above; bottom halo ← the first rows below
                CK(cudaMemcpyPeerAsync(mine, h->device,
                                       buf(up) + static_cast<size_t>(up->halo + up->band_rows - h->halo) * rowb,
                                       up->device, hb, h->stream));
                CK(cudaMemcpyPeerAsync(mine + static_cast<size_t>(h->halo + h->band_rows) * rowb, h->device,
                                       buf(dn) + static_cast<size_t>(dn->halo) * rowb, dn->device, hb, h->stream));
                CK(cudaEventRecord(ev_x[g], h->stream));
            }
            // chunk: src = buffer par, dst = 1 - par.  A band's kernel overwrites buffer 1-par, which
            // its neighbours read during the previous exchange: wait for their exchange events.
            for (int g = 0; g < n; ++g) {
                escg_dev* h = bands[g];
                CK(cudaSetDevice(h->device));
                CK(cudaStreamWaitEvent(h->stream, ev_x[(g + n - 1) % n], 0));
                CK(cudaStreamWaitEvent(h->stream, ev_x[(g + 1) % n], 0));
                const escgd::RunArgs run = run_args(h, 0, 1, 0, 0, false);
                escgd::BlockArgs a{};
                a.seeds = h->d_seeds.p;
                a.rule = rule_args(h);
                a.run = run;
                a.H = h->H;
                a.L = h->L;
                a.S = h->S;
                a.P = h->P;
                a.arity = h->arity;
                a.narrow = h->narrow;
                a.Hg = h->Hg;
                a.row0 = h->row0;
                a.wrap_rows = h->wrap_rows;
                a.reflect = h->flux ? 0 : 1;
        a.seam_np = h->seam_np;
        a.phase_table = h->phase_table;
                a.nby = h->nby;
                a.nbx = h->nbx;
                a.row_split = h->d_rows.p;
                a.col_split = h->d_cols.p;
                a.acc = h->d_acc.p;
                a.ticket = h->d_ticket.p;
                a.smem_bytes = h->smem;
                a.step = 1;
                a.count = 0;
                a.src = h->lat[par].p;
                a.dst = h->lat[1 - par].p;
                a.psrc = h->pl[par].p;
                a.pdst = h->pl[1 - par].p;
                a.K = h->K;
                a.npl = h->npl;
                a.lpi = h->lpi;
                a.qcap = h->qcap;
                a.T3 = h->sliced3 ? h->d_T3.p : nullptr;
                a.dst_index = 1 - par;
                a.mcs = t0 + done;
                a.nmcs = chunk;
                CK(cudaMemsetAsync(h->d_status.p, 0xFF, sizeof(int32_t), h->stream));
                if (sliced)
                    CK(escgd::launch_slice(a, 1, h->stream));
                else
                    CK(escgd::launch_block(a, 1, h->threads, h->stream));
                CK(cudaEventRecord(ev_k[g], h->stream));
            }
            par ^= 1;
            done += chunk;
            ++launch_no;
        }
        for (int g = 0; g < n; ++g) {
            CK(cudaSetDevice(bands[g]->device));
            if (sliced) {
                bands[g]->cur[0] = par;
                band_sync_bytes(bands[g]);
            }
            CK(cudaStreamSynchronize(bands[g]->stream));
            bands[g]->mcs[0] += n_mcs;
            bands[g]->cur[0] = par;
            bands[g]->last_launches = launch_no;
        }
    });
}

int escg_dev_ring_part_export(escg_dev* h, void** planes0, void** planes1, void** inbox, int32_t* rows, void* ipc,
                              int64_t* inbox_offset) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (!h->ring_part) config_error("not a ring part");
        CK(cudaSetDevice(h->device));
        if (planes0) *planes0 = h->rpart.pl[0];
        if (planes1) *planes1 = h->rpart.pl[1];
        if (inbox) *inbox = h->rpart.inbox;
        if (rows) *rows = h->rpart.rows;
        if (inbox_offset) *inbox_offset = static_cast<int64_t>(reinterpret_cast<char*>(h->rpart.inbox) -
                                                               reinterpret_cast<char*>(h->d_mbox.p));
        if (ipc) {  // CUDA IPC handles of the three allocations (planes 0, planes 1, mailboxes)
            static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
            cudaIpcMemHandle_t m[3];
            CK(cudaIpcGetMemHandle(&m[0], h->pl[0].p));
            CK(cudaIpcGetMemHandle(&m[1], h->pl[1].p));
            CK(cudaIpcGetMemHandle(&m[2], h->d_mbox.p));
            std::memcpy(ipc, m, sizeof(m));
        }
    });
}

int escg_dev_ring_part_connect(escg_dev* h, void* up_planes0, void* up_planes1, void* up_inbox, int32_t up_rows,
                               void* dn_planes0, void* dn_planes1, void* dn_inbox, int32_t dn_rows) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (!h->ring_part) config_error("not a ring part");
        if (!up_planes0 || !up_planes1 || !up_inbox || !dn_planes0 || !dn_planes1 || !dn_inbox)
            config_error("null neighbour pointer");
        if (up_rows < 8 || dn_rows < 8) config_error("neighbour part too thin");
        h->rpart.up_pl[0] = static_cast<uint32_t*>(up_planes0);
        h->rpart.up_pl[1] = static_cast<uint32_t*>(up_planes1);
        h->rpart.up_inbox = static_cast<unsigned long long*>(up_inbox);
        h->rpart.up_rows = up_rows;
        h->rpart.dn_pl[0] = static_cast<uint32_t*>(dn_planes0);
        h->rpart.dn_pl[1] = static_cast<uint32_t*>(dn_planes1);
        h->rpart.dn_inbox = static_cast<unsigned long long*>(dn_inbox);
        h->ring_connected = true;
    });
}

int escg_ipc_open(int32_t device, const void* handle, void** ptr) {
    return guarded([&] {
        if (!handle || !ptr) config_error("null argument");
        CK(cudaSetDevice(device));
        cudaIpcMemHandle_t m;
        std::memcpy(&m, handle, sizeof(m));
        CK(cudaIpcOpenMemHandle(ptr, m, cudaIpcMemLazyEnablePeerAccess));
    });
}

int escg_ipc_close(int32_t device, void* ptr) {
    return guarded([&] {
        if (!ptr) config_error("null argument");
        CK(cudaSetDevice(device));
        CK(cudaIpcCloseMemHandle(ptr));
    });
}

int escg_ring_group_advance(escg_dev** parts, int32_t n, int64_t n_mcs) {
    return guarded([&] {
        if (!parts || n < 2) config_error("a ring group needs at least 2 parts");
        for (int g = 0; g < n; ++g)
            if (!parts[g] || !parts[g]->ring_part || parts[g]->nbands != n || parts[g]->band != g)
                config_error("group must list parts 0..n-1 of one ring");
        bool one = true;
        for (int g = 0; g < n; ++g) one = one && parts[g]->device == parts[0]->device;
        if (!one) {  // parts on several GPUs of this process: peer access between ring neighbours
            for (int g = 0; g < n; ++g)
                for (int nb : {(g + n - 1) % n, (g + 1) % n}) {
                    const int d0 = parts[g]->device, d1 = parts[nb]->device;
                    int can = 0;
                    if (d0 == d1) continue;
                    CK(cudaDeviceCanAccessPeer(&can, d0, d1));
                    if (!can) config_error("ring parts on GPUs without peer access");
                    CK(cudaSetDevice(d0));
                    const cudaError_t pe = cudaDeviceEnablePeerAccess(d1, 0);
                    if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) CK(pe);
                    cudaGetLastError();
                }
        }
        ring_parts_advance(parts, n, n_mcs, one);
    });
}

int escg_dev_band_rows(escg_dev* h, uint8_t** recv_top, uint8_t** send_top, uint8_t** send_bot, uint8_t** recv_bot,
                       int64_t* bytes) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (h->nbands < 2 || h->ring_part) config_error("not a band engine");
        CK(cudaSetDevice(h->device));
        uint8_t* base = h->lat[h->cur[0]].p;
        size_t row = static_cast<size_t>(h->L);
        if (h->narrow == 2) {  // bit-sliced: halos move as plane rows (NPL x L/128 x 16 bytes)
            band_sync_planes(h);
            if (h->stream == h->own_stream) CK(cudaStreamSynchronize(h->stream));
            base = reinterpret_cast<uint8_t*>(h->pl[h->cur[0]].p);
            row = static_cast<size_t>(h->npl) * (h->L / 128) * 16;
        }
        if (recv_top) *recv_top = base;
        if (send_top) *send_top = base + static_cast<size_t>(h->halo) * row;
        if (send_bot) *send_bot = base + static_cast<size_t>(h->band_rows) * row;
        if (recv_bot) *recv_bot = base + static_cast<size_t>(h->halo + h->band_rows) * row;
        if (bytes) *bytes = static_cast<int64_t>(h->halo * row);
    });
}

int escg_dev_band_step(escg_dev* h, int32_t n_mcs) {
    return guarded([&] {
        if (!h) config_error("null handle");
        if (h->nbands < 2 || h->ring_part) config_error("not a band engine");
        if (n_mcs < 1 || n_mcs > h->kmcs)
            config_error("band step must run 1.." + std::to_string(h->kmcs) + " MCS (the halo depth)");
        CK(cudaSetDevice(h->device));
        const int par = h->cur[0];
        escgd::BlockArgs a{};
        a.seeds = h->d_seeds.p;
        a.rule = rule_args(h);
        a.run = run_args(h, 0, 1, 0, 0, false);
        a.H = h->H;
        a.L = h->L;
        a.S = h->S;
        a.P = h->P;
        a.arity = h->arity;
        a.narrow = h->narrow;
        a.Hg = h->Hg;
        a.row0 = h->row0;
        a.wrap_rows = h->wrap_rows;
        a.reflect = 0;
        a.seam_np = 0;
        a.nby = h->nby;
        a.nbx = h->nbx;
        a.row_split = h->d_rows.p;
        a.col_split = h->d_cols.p;
        a.acc = h->d_acc.p;
        a.ticket = h->d_ticket.p;
        a.smem_bytes = h->smem;
        a.step = 1;
        a.count = 0;
        a.src = h->lat[par].p;
        a.dst = h->lat[1 - par].p;
        a.psrc = h->pl[par].p;
        a.pdst = h->pl[1 - par].p;
        a.K = h->K;
        a.npl = h->npl;
        a.lpi = h->lpi;
        a.qcap = h->qcap;
        a.T3 = h->sliced3 ? h->d_T3.p : nullptr;
        a.dst_index = 1 - par;
        a.mcs = h->mcs[0];
        a.nmcs = n_mcs;
        CK(cudaMemsetAsync(h->d_status.p, 0xFF, sizeof(int32_t), h->stream));
        if (h->narrow == 2) {  // bit-sliced: the band stays in plane form between steps
            band_sync_planes(h);
            CK(escgd::launch_slice(a, 1, h->stream));
        } else {
            CK(escgd::launch_block(a, 1, h->threads, h->stream));
        }
        // on the engine's own stream the step completes before return; on a caller's stream it is
        // only enqueued, ordered after (and before) the caller's halo exchange on that stream
        if (h->stream == h->own_stream) CK(cudaStreamSynchronize(h->stream));
        CK(cudaGetLastError());
        h->cur[0] = 1 - par;
        h->mcs[0] += n_mcs;
        h->last_launches = 1;
    });
}

int escg_dev_set_stream(escg_dev* h, void* stream) {
    return guarded([&] {
        if (!h) config_error("null handle");
        CK(cudaSetDevice(h->device));
        CK(cudaStreamSynchronize(h->stream));  // work already enqueued on the previous stream
        h->stream = stream ? static_cast<cudaStream_t>(stream) : h->own_stream;
    });
}

int escg_dev_draw_format(escg_dev* h, int32_t* narrow) {
    return guarded([&] {
        if (!h || !narrow) config_error("null argument");
        *narrow = h->narrow == 2 ? ((h->sliced3 ? 3 : 2) | (h->K << 8)) : h->narrow;
    });
}

int escg_simulate(const escg_params* p, const double* dominance, int32_t species, int32_t kind, int32_t mode,
                  int32_t device, const int32_t* resume_cells, int64_t resume_mcs, uint32_t stop_flags,
                  int32_t tracked_species, int32_t* out_cells, int64_t* out_mcs, int64_t* steps, uint64_t* counts,
                  int64_t cap, int64_t* n_records, int32_t* status) {
    return guarded([&] {
        if (!p) config_error("null params");
        validate_params(*p);
        escg_params pp = *p;  // a missing seed is drawn per call (engine.cpp:210 random_device)
        if (!pp.has_seed) {
            pp.has_seed = 1;
            pp.seed = (static_cast<uint64_t>(std::random_device{}()) << 32) | std::random_device{}();
        }
        p = &pp;
        const int64_t N = static_cast<int64_t>(p->length) * p->height;
        int64_t interval = 1;
        if (mode == ESCG_MODE_MAX_STEP) interval = align_num_randoms_or_throw(p->num_randoms, N) / N;
        else if (mode == ESCG_MODE_PARALLEL_MCS) align_num_randoms_or_throw(p->num_randoms, N);  // engine.cpp:142
        else if (mode != ESCG_MODE_SERIAL) config_error("unknown engine mode");
        validate_dominance(dominance, species, kind);  // before the model is copied into the key
        // Engines are cached per thread by shape/model so repeated calls reuse device buffers.  The key
        // is compared field by field (no memcmp over padding) and includes the environment knobs that
        // shape an engine at creation (draw format, planner experiments); the seed is not part of it —
        // a new seed only rewrites the replica seed of the cached engine.
        struct Cache {
            escg_dev* h = nullptr;
            std::vector<double> dom;
            int length = 0, height = 0, neighbourhood = 0, species = 0, flux = 0, kind = -1, device = -1;
            double mobility = 0.0, empty_prob = 0.0;
            std::string env;
            ~Cache() {
                if (h) escg_dev_destroy(h);
            }
        };
        thread_local Cache cache;
        std::vector<double> dom(dominance, dominance + static_cast<size_t>(species) * species);
        std::string env;
        for (const char* k : {"ESCG_DRAW_FORMAT", "ESCG_SLICE_K", "ESCG_SLICE_LPI", "ESCG_SLICE_QCAP", "ESCG_SLICE_SPLIT",
                              "ESCG_SLICE_OVERHEAD", "ESCG_BLOCK_MCS", "ESCG_BLOCK_K", "ESCG_BLOCK_THREADS",
                              "ESCG_PERSISTENT", "ESCG_PHASE_TABLE", "ESCG_TILE_THREADS", "ESCG_WIDE_RULE", "ESCG_RING",
                              "ESCG_RING_NB", "ESCG_SLICE_DRAWS"}) {
            const char* v = std::getenv(k);
            env += std::string(k) + "=" + (v ? v : "") + ";";
        }
        const bool same = cache.h && cache.kind == kind && cache.device == device && cache.dom == dom &&
                          cache.length == p->length && cache.height == p->height &&
                          cache.neighbourhood == p->neighbourhood && cache.species == p->species &&
                          cache.flux == p->flux && cache.mobility == p->mobility &&
                          cache.empty_prob == p->empty_prob && cache.env == env;
        if (!same) {
            if (cache.h) escg_dev_destroy(cache.h);
            cache.h = nullptr;
            escg_dev* h = nullptr;
            const int rc = escg_dev_create(p, dominance, species, kind, device, 1, nullptr, ESCG_KERNEL_AUTO, &h);
            if (rc != ESCG_OK) throw Error(rc, g_last_error);
            cache.h = h;
            cache.dom = dom;
            cache.length = p->length;
            cache.height = p->height;
            cache.neighbourhood = p->neighbourhood;
            cache.species = p->species;
            cache.flux = p->flux;
            cache.mobility = p->mobility;
            cache.empty_prob = p->empty_prob;
            cache.kind = kind;
            cache.device = device;
            cache.env = env;
        } else if (cache.h->seeds[0] != p->seed) {
            cache.h->seeds[0] = p->seed;
            CK(cudaSetDevice(cache.h->device));
            CK(cudaMemcpy(cache.h->d_seeds.p, cache.h->seeds.data(), sizeof(uint64_t), cudaMemcpyHostToDevice));
        }
        escg_dev* h = cache.h;
        h->p = *p;
        int rc;
        if (resume_cells)
            rc = escg_dev_set_lattice(h, 0, resume_cells, resume_mcs);
        else
            rc = escg_dev_init_lattice(h);
        if (rc != ESCG_OK) throw Error(rc, g_last_error);
        const uint32_t flags = stop_flags | ESCG_STOP_STASIS | (tracked_species >= 1 ? ESCG_STOP_TRACKED : 0u);
        int32_t st = 0;
        rc = escg_dev_run(h, p->mcs_limit, interval, flags, tracked_species, (steps || counts) ? 1 : 0, &st);
        if (rc != ESCG_OK) throw Error(rc, g_last_error);
        int64_t n = 0;
        rc = escg_dev_read_trace(h, 0, steps, counts, cap, &n);
        if (rc != ESCG_OK) throw Error(rc, g_last_error);
        if (n_records) *n_records = n;
        rc = escg_dev_get_lattice(h, 0, out_cells, out_mcs);
        if (rc != ESCG_OK) throw Error(rc, g_last_error);
        if (status) *status = st;
    });
}

}  // extern "C"
