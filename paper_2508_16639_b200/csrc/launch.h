// launch.h — argument blocks and launchers shared by the host engine (engine.cpp) and the
// sm_100a kernels (kernels.cu).  No torch types; plain device pointers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace escgd {

// Margin of the overlapped-tile (block) kernel: a tile footprint reaches 3 cells past the tile
// origin, so validity shrinks by 3 cells per phase and 4 phases need 12 cells.
// With k MCS per launch (temporal blocking) the margin is 12k rows and 12k+4 columns rounded up to
// a multiple of 16 (window column 0 stays 16-aligned: TMA rows and NARROW tile pairs).
constexpr int kMaxBlockMcs = 4;
__host__ __device__ constexpr int margin_rows(int k) { return 12 * k; }
__host__ __device__ constexpr int margin_cols(int k) { return (12 * k + 4 + 15) & ~15; }
// Tile-kernel window: rows -2..H, cols -2..L (ghost frame of the periodic wrap), origin (2, 4).
constexpr int kTileR0 = 2;
constexpr int kTileC0 = 4;
constexpr int kMaxSpecies = 64;
constexpr int kMaxDevices = 64;
// Block-kernel CTA size = its launch bound: 640 threads → up to 96 registers per thread, no spills
// (measured faster than 1024 x 64 registers and 2 x 512 per SM).
constexpr int kBlockThreads = 640;
// Tile-kernel launch shapes (kernels.cu tile_kernel): two CTAs per SM when the lattice's shared
// memory allows it (<= 384 threads, <= 80 registers), else one (<= 512 threads, <= 128 registers).
constexpr int kTileThreadsTwo = 384, kTileThreadsOne = 512;
inline bool tile_one_per_sm(int smem_bytes) { return smem_bytes > (228 * 1024) / 2 - 1024 - 1024; }

struct RuleArgs {
    uint32_t xm, xi;       // X_mig, X_int
    const uint32_t* T;     // (S+1)^2 interaction thresholds (device)
    uint32_t fast;         // NARROW certain-migration bound on attempt bits: (xm >> (16+LB)) << LB
    uint32_t wide_bf;      // WIDE rule form: 1 branch-free (P(migration) < 0.97), 0 branchy
};

// Per-replica run bookkeeping (device arrays, length n_replicas unless noted).
struct RunArgs {
    int64_t* mcs;             // current MCS
    int32_t* status;          // ESCG_RUNNING (-1) or final RunStatus
    uint64_t* last_counts;    // [rep][S+1] last density record
    int64_t* n_rec;           // records written this run
    int64_t* trace_steps;     // [rep][cap] or nullptr
    uint64_t* trace_counts;   // [rep][cap][S+1] or nullptr
    int64_t trace_cap;
    int32_t* cur;             // block path: buffer (0/1) holding the lattice at the last record
    int64_t mcs_limit;
    int64_t interval;
    uint32_t stop_flags;
    int32_t tracked;
};

struct TileArgs {
    uint8_t* lat;  // [rep][H*L], row-major
    const uint64_t* seeds;
    RuleArgs rule;
    RunArgs run;
    int H, L, S, P;   // P = shared-memory pitch
    int arity, flux;
    int narrow;       // draw format
    int record;       // 1: record/check loop (escg_dev_run); 0: advance to run.mcs_limit
    int smem_bytes;
    int one_per_sm;   // launch shape (tile_one_per_sm(smem_bytes))
};

struct BlockArgs {
    const uint8_t* src;  // [rep][H*L]
    uint8_t* dst;
    const uint64_t* seeds;
    RuleArgs rule;
    RunArgs run;
    int H, L, S, P;      // P = window pitch; H = rows of the local buffer
    int arity;
    int narrow;
    int Hg;              // rows of the global lattice (tile ids / draws are global)
    int row0;            // global row of local row 0 (band engines: band start - halo, mod Hg)
    int wrap_rows;       // 1: the local buffer is the whole periodic lattice; 0: band with halo rows
    int reflect;         // 1: mirror-reflecting lattice (flux = false): clipped windows, reflect tiling
    int seam_np;         // > 0: periodic lattice with seams (L or H not divisible by 4): phases per MCS
    int phase_table;     // 1: per-launch phase-geometry table (few items per thread per phase)
    int nby, nbx;
    const int* row_split;  // nby+1 row boundaries (multiples of 4)
    const int* col_split;  // nbx+1
    int64_t mcs;           // first MCS executed by this launch
    int nmcs;              // MCS per launch (temporal blocking, margins margin_rows/cols(nmcs))
    int dst_index;         // buffer index of dst (recorded with the density record)
    int step;              // 1: execute MCS [mcs, mcs+nmcs) (src → dst); 0: count src only
    int count;             // 1: record densities of the result (at mcs+step)
    unsigned long long* acc;  // [rep][S+1] cross-CTA accumulators (zero between records)
    unsigned int* ticket;     // [rep]
    int smem_bytes;
    // bit-sliced path (narrow == 2, slice.cu): the lattice as NPL bit planes [rep][H][NPL][L/128][4]
    // u32 (word q of group g holds columns 128g + 4b + q in bit b); col_split then holds group
    // splits (block i covers columns [128 s_i + 64, 128 s_{i+1} + 64))
    const uint32_t* psrc;
    uint32_t* pdst;
    int K;    // SLICED action planes
    int npl;  // bit planes (species code bits)
    int lpi;  // lanes per bit-sliced item (1, or 2: draws and planes split over a lane pair)
    int qcap; // > 0: deferred-tile queue capacity override (tests of the in-place overflow path)
    const uint32_t* T3;  // SLICED3 tables (orc_slice3_table layout; slice_common.cuh slice3_masks), null: SLICED
};

// Persistent cooperative block kernel: the whole run/advance in one launch (all CTAs co-resident).
struct PersistArgs {
    BlockArgs b;              // geometry, rule, run bookkeeping, buffers (src = buffer 0 at start)
    uint8_t* buf[2];
    int64_t mcs0, mcs_end;    // advance: [mcs0, mcs_end); run: limit = b.run.mcs_limit
    int record;               // 1: record/check loop at b.run.interval; 0: advance only
    int kmcs;                 // MCS per chunk
    unsigned long long* acc3; // [3][rep][S+1] record accumulators (zeroed by the host)
};

struct InitArgs {
    uint8_t* lat;
    const uint64_t* seeds;
    int64_t n;          // cells per replica (local buffer)
    int L;              // row length
    int Hg;             // global rows; local row r is global row (row0 + r) mod Hg
    int row0;
    int nrep;
    int S;
    uint32_t x_empty;   // cell empty iff first word < x_empty (empty_prob test, lattice.hpp:59)
    int all_empty;      // empty_prob >= 1 (lattice.hpp:56-57)
};

struct ReplayArgs {
    uint8_t* lat;
    const uint32_t* wc;
    const uint32_t* wd;
    const uint32_t* wa;
    int64_t n_attempts;
    RuleArgs rule;
    int H, L, S, arity, flux;
};

cudaError_t launch_init(const InitArgs& a, cudaStream_t s);
cudaError_t launch_count(const uint8_t* lat, int64_t n, int nrep, int S, unsigned long long* out, cudaStream_t s);
cudaError_t launch_tile(const TileArgs& a, int nrep, int threads, cudaStream_t s);
cudaError_t launch_block(const BlockArgs& a, int nrep, int threads, cudaStream_t s);
cudaError_t launch_block_persistent(const PersistArgs& a, int nrep, int threads, cudaStream_t s);
int block_persistent_capacity(int arity, int threads, int smem_bytes, int device);
int tile_capacity(int arity, int flux, int H, int L, int threads, int smem_bytes, int device);
int block_kernel_registers(int arity);
cudaError_t launch_replay(const ReplayArgs& a, cudaStream_t s);
// bit-sliced path (slice.cu)
// CTA size of the bit-sliced kernel: 256 threads (<= 255 registers) with one lane per item, 512
// (<= 128 registers) with a lane pair per item
#ifndef ESCG_SLICE_T2
#define ESCG_SLICE_T2 512
#endif
#ifndef ESCG_SLICE_T1  // experiments: CTA size of the one-lane kernel
#define ESCG_SLICE_T1 256
#endif
#ifndef ESCG_SLICE_MINB1  // experiments: CTAs per SM the one-lane kernel is compiled for
#define ESCG_SLICE_MINB1 1
#endif
__host__ __device__ constexpr int slice_threads(int lpi) { return lpi == 2 ? ESCG_SLICE_T2 : ESCG_SLICE_T1; }
__host__ __device__ constexpr int slice_min_blocks(int lpi) { return lpi == 2 ? 512 / ESCG_SLICE_T2 : ESCG_SLICE_MINB1; }
constexpr int kSliceMaxK = 16;
cudaError_t launch_slice(const BlockArgs& a, int nrep, cudaStream_t s);
int slice_row_words(int npl, int gw);  // shared-memory words per window row (padded)
int slice_kernel_registers(int npl, int lpi);
// u8 lattice <-> bit planes for every replica; from_planes picks plane buffer cur[r] - 2 when cur
// is given (replicas with cur[r] < 2 are skipped), else `buf`
cudaError_t launch_to_planes(const uint8_t* lat, uint32_t* pl, int H, int L, int npl, int nrep, cudaStream_t s);
cudaError_t launch_from_planes(const uint32_t* pl0, const uint32_t* pl1, const int32_t* cur, int buf, uint8_t* lat,
                               int H, int L, int npl, int nrep, cudaStream_t s);
// Persistent bit-sliced ring kernel (ring.cu): one co-resident CTA per row band of
// full-width rows; colour phases exchange boundary rows with the two neighbour bands through L2
// mailboxes (data words tagged with the phase), so no area is recomputed.
constexpr int kRingThreads = 256;
// One row range of a multi-part ring (csrc/ring.cu "parts"): its bands run on one device, the
// boundary bands exchange with the neighbouring parts through tagged words in the consumer part's
// inboxes (NVLink peer stores when the parts sit on different GPUs) and write the rows they finish
// in a neighbour's range into its plane buffers as well.
constexpr int kMaxRingParts = 8;
struct RingPart {
    uint32_t* pl[2];                // plane buffers, rows [r0 - 2, r0 + rows + 2) (local row = gy - r0 + 2)
    uint32_t* up_pl[2];             // the part above's (peer memory)
    uint32_t* dn_pl[2];             // the part below's
    unsigned long long* mbox;       // local band mailboxes [nb][dir][parity][mbs]
    unsigned long long* inbox;      // [set][side: 0 from above, 1 from below][parity][mbs], flags [set][side]
    unsigned long long* up_inbox;   // the part above's inboxes (this part's band 0 publishes there)
    unsigned long long* dn_inbox;   // the part below's (this part's last band publishes there)
    int r0, rows, up_rows, nb, cta0;
};

struct RingArgs {
    const uint32_t* pin;      // input planes [H][NPL][L/128][4]
    uint32_t* pbuf[2];        // snapshots: record k of the launch -> pbuf[k & 1]; advance -> pbuf[1]
    const uint64_t* seeds;
    RuleArgs rule;
    RunArgs run;              // replica 0; run.interval = record cadence
    int H, L, S, npl, K;
    int64_t mcs0, mcs_end;    // MCS [mcs0, mcs_end)
    int record;               // 1: density records at mcs0 + k*interval and at mcs_end; 0: advance
    unsigned long long* mbox; // [nb][dir][parity][mbs] tagged words (zeroed before every launch)
    int mbs;                  // words per mailbox: 2 header + 3 rows x NPL x L/128 x 4
    unsigned int* decided;    // records decided in this launch (zeroed before the launch)
    unsigned long long* acc;  // [S+1] record accumulators (zero between records)
    unsigned int* ticket;
    int smem_bytes;
    int qcap;                 // > 0: per-warp deferred-tile queue capacity override (tests)
    const uint32_t* T3;       // SLICED3 tables (orc_slice3_table layout), null: SLICED
    // multi-part ring (nparts > 0; advance only): parts [0, nparts) of this launch, CTAs by cta0
    int nparts;
    int cur;                  // plane buffer holding the state (the final phase writes cur ^ 1)
    int xset;                 // inbox set of this launch (launch epoch & 1)
    uint32_t epoch;           // launch epoch (identical on every part)
    int wait_snap;            // 1: the previous launch's boundary rows arrive from the neighbours
    unsigned long long timeout_ns;  // a wait for a neighbour part gives up after this long
    RingPart part[kMaxRingParts];
};
constexpr int kRingInboxWords(int mbs) { return 8 * mbs + 4; }  // 2 sets x 2 sides x 2 parities + flags
// a multi-part ring whose neighbour stops answering (a rank that died, a launch that never came)
// gives up after this long, with this status (every waiting part times out in turn): the host
// raises instead of hanging
constexpr unsigned long long kRingPartTimeoutNs = 20ull * 1000 * 1000 * 1000;  // default (ESCG_RING_TIMEOUT_S)
constexpr int kStatusRingTimeout = 0x5254;
cudaError_t launch_ring(const RingArgs& a, int nb, cudaStream_t s);
int ring_smem_bytes(int H, int L, int npl, int nb);
int ring_capacity(int npl, int smem_bytes, int device);  // co-resident CTAs (cooperative launch)
cudaError_t launch_u8_to_i32(const uint8_t* src, int32_t* dst, int64_t n, cudaStream_t s);
cudaError_t launch_i32_to_u8(const int32_t* src, uint8_t* dst, int64_t n, int S, int* bad, cudaStream_t s);
int tile_smem_bytes(int H, int L, int S, int* pitch);
int max_smem_optin(int device);

}  // namespace escgd
