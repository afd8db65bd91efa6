/*
 * escg_dev.h — C ABI of the B200-native ESCG Monte Carlo engine (libescg_b200.so).
 *
 * The reference exposes its hot path only as C++ (`escg::simulate`, engine.hpp:169-171, and the
 * `run_*` loops, engine.hpp:149-159); it has no C ABI, plugin registry or FFI.  These entry points
 * are what an FFI for that path binds: plain pointers and sizes, int return codes instead of the
 * reference's exceptions (errors.hpp:9-26 → codes below), one thread-local error message.
 *
 * Threading: a handle is single-threaded (one host thread); distinct handles are independent.
 * Ownership: the library copies every input; output buffers are caller-owned.
 */
#ifndef ESCG_DEV_H
#define ESCG_DEV_H

#include <stdint.h>

#if defined(__GNUC__)
#define ESCG_API __attribute__((visibility("default")))
#else
#define ESCG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes — mirror of errors.hpp:9-26 mapped as SPEC.md:502 maps them to exit codes. */
#define ESCG_OK 0
#define ESCG_ECONFIG 2 /* escg::ConfigError  */
#define ESCG_EIO 3     /* escg::IoError      */
#define ESCG_EFORMAT 4 /* escg::FormatError  */
#define ESCG_EENGINE 5 /* escg::EngineError, CUDA failure, missing device */

/* RunStatus (engine.hpp:20); ESCG_RUNNING only appears in per-replica status arrays mid-run. */
#define ESCG_COMPLETED 0
#define ESCG_STASIS 1
#define ESCG_STOPPED 2
#define ESCG_RUNNING (-1)

/* DominanceModel::Kind (dominance.hpp:16) */
#define ESCG_DOM_BINARY 0
#define ESCG_DOM_RATED 1

/* EngineMode (engine.hpp:18): the record cadence the device engine reproduces.
 * SERIAL / PARALLEL_MCS record every MCS; MAX_STEP records every align(num_randoms, N)/N MCS
 * (engine.cpp:165-192).  The device update itself is always the coloured kernel. */
#define ESCG_MODE_SERIAL 0
#define ESCG_MODE_PARALLEL_MCS 1
#define ESCG_MODE_MAX_STEP 2

/* Kernel selection (escg_dev_create `kernel` argument). */
#define ESCG_KERNEL_AUTO 0
#define ESCG_KERNEL_TILE 1  /* whole lattice resident in one CTA's shared memory, persistent  */
#define ESCG_KERNEL_BLOCK 2 /* overlapped-tile kernel over an HBM/L2-resident lattice          */
#define ESCG_KERNEL_RING 3  /* persistent bit-sliced row bands (one CTA per SM, L2 boundary mail):
                               AUTO picks it for single periodic lattices with 1024 <= L <= 4096,
                               L % 128 == 0 at high mobility (the L=3200 bench) */

/* POD mirror of escg::SimParams (params.hpp:18-49); defaults via escg_params_default(). */
typedef struct escg_params {
    int32_t length;          /* L, columns                     params.hpp:19 */
    int32_t height;          /* H, rows                        params.hpp:20 */
    int64_t mcs_limit;       /*                                params.hpp:21 */
    int32_t neighbourhood;   /* 4 (VonNeumann4) or 8 (Moore8)  params.hpp:22 */
    int32_t print_frequency; /*                                params.hpp:23 */
    double mobility;         /* M                              params.hpp:24 */
    int32_t species;         /* S in [1, 64]                   params.hpp:25 */
    int32_t flux;            /* 1 periodic, 0 mirror reflect   params.hpp:26 */
    double empty_prob;       /*                                params.hpp:27 */
    int32_t save;            /*                                params.hpp:28 */
    int32_t dominance_import;
    int32_t resume;
    int64_t num_randoms;     /*                                params.hpp:31 */
    int32_t max_step;        /*                                params.hpp:32 */
    int32_t has_seed;        /* std::optional<uint64_t> seed   params.hpp:33 */
    uint64_t seed;
} escg_params;

/* Stop predicates evaluated on device at every density record (record_and_check order,
 * engine.cpp:47-57): tracked-species extinction (the experiments harness's on_record,
 * experiments.cpp:107-113) → STOPPED; mcs >= limit → COMPLETED; |alive| <= 1 → STASIS. */
#define ESCG_STOP_TRACKED 1u
#define ESCG_STOP_STASIS 2u

typedef struct escg_dev escg_dev;

/* Thread-local message of the last failing call on this thread ("" if none). */
ESCG_API const char* escg_dev_last_error(void);

/* SimParams defaults (params.hpp:19-33; Table 3.1/3.2). */
ESCG_API int escg_params_default(escg_params* out);

/* SimParams::validate (params.hpp:37-48) + DominanceModel::validate (dominance.cpp:8-21). */
ESCG_API int escg_validate(const escg_params* p, const double* dominance, int32_t species, int32_t kind);

/* ε = 2MN, μ = σ = 1 (params.hpp:61-70): out = {mu, sigma, epsilon, total}. */
ESCG_API int escg_action_rates(double mobility, int64_t cells, double* out4);

/* Integer action thresholds equivalent to the reference's double bucketing:
 * out_xmx = {X_mig, X_int}; out_T = (S+1)*(S+1) interaction thresholds, T[a*(S+1)+b]. */
ESCG_API int escg_thresholds(double mobility, int64_t cells, const double* dominance, int32_t species, uint32_t* out_xmx,
                    uint32_t* out_T);

/* align_num_randoms (random_batch.hpp:32-38); returns -1 and sets the error on ConfigError. */
ESCG_API int64_t escg_align_num_randoms(int64_t requested, int64_t cells);

/* Create an engine for `n_replicas` independent lattices of params' shape on CUDA `device`.
 * replica_seeds may be NULL: replica r then uses seed + r (experiments.cpp:26 trial_seed).
 * dominance: S*S doubles, row = attacker-1 (dominance.hpp:20). */
ESCG_API int escg_dev_create(const escg_params* p, const double* dominance, int32_t species, int32_t kind, int32_t device,
                    int32_t n_replicas, const uint64_t* replica_seeds, int32_t kernel, escg_dev** out);
ESCG_API int escg_dev_destroy(escg_dev* h);

/* Device init_lattice (lattice.hpp:53-66 transform on Philox draws) for every replica; mcs := 0. */
ESCG_API int escg_dev_init_lattice(escg_dev* h);
/* Upload one replica's int32 lattice (range-checked, Lattice = row-major, lattice.hpp:14-27). */
ESCG_API int escg_dev_set_lattice(escg_dev* h, int32_t replica, const int32_t* cells, int64_t mcs);
/* Export one replica's lattice as int32 and its current MCS. */
ESCG_API int escg_dev_get_lattice(escg_dev* h, int32_t replica, int32_t* out, int64_t* mcs_out);
/* Species counts of the current lattice (densities(), engine.cpp:70-94); out = S+1 u64. */
ESCG_API int escg_dev_counts(escg_dev* h, int32_t replica, uint64_t* out);

/* Advance every replica by n_mcs Monte Carlo steps without density records. */
ESCG_API int escg_dev_advance(escg_dev* h, int64_t n_mcs);

/* The record/check/advance loop of run_parallel_mcs / run_max_step (engine.cpp:135-192) on
 * device: record at the current MCS, check stop predicates, advance min(interval, limit-mcs),
 * repeat.  Runs every replica to its own status; status_out[n_replicas] (may be NULL).
 * Density records are kept on device when record_trace != 0 (read with escg_dev_read_trace);
 * the last record of each replica is always kept. */
ESCG_API int escg_dev_run(escg_dev* h, int64_t mcs_limit, int64_t interval, uint32_t stop_flags, int32_t tracked_species,
                 int32_t record_trace, int32_t* status_out);

/* Density trace of one replica from the last escg_dev_run: steps[cap], counts[cap*(S+1)]. */
ESCG_API int escg_dev_read_trace(escg_dev* h, int32_t replica, int64_t* steps, uint64_t* counts, int64_t cap,
                        int64_t* n_out);
/* Per-replica summary of the last run: mcs at stop, status, last record counts [(S+1)]. */
ESCG_API int escg_dev_replica_result(escg_dev* h, int32_t replica, int64_t* mcs, int32_t* status, uint64_t* last_counts);

/* TEST PATH — bit-exact serial replay of injected reference draws (engine.cpp:104-110):
 * cell = w_cell % N, dir = w_dir % arity, action word = w_act, applied in order by one device
 * thread with the production rule on replica 0. */
ESCG_API int escg_dev_replay(escg_dev* h, const uint32_t* w_cell, const uint32_t* w_dir, const uint32_t* w_act, int64_t n);

/* Device time (ms) of the work enqueued by the last advance/run/replay call, CUDA events on the
 * engine's stream; and the number of kernels that call launched. */
ESCG_API int escg_dev_last_timing(escg_dev* h, double* ms, int64_t* launches);

/* Kernel actually selected (ESCG_KERNEL_TILE / _BLOCK / _RING) and its launch geometry. */
ESCG_API int escg_dev_describe(escg_dev* h, int32_t* kernel, int32_t* grid_ctas, int32_t* threads, int32_t* smem_bytes);

/* Draw format chosen for this engine: 0 WIDE (32-bit attempt words), 1 NARROW (16-bit words, one
 * draw per tile pair), 2 | K << 8 SLICED (bit-plane draws shared by 32 tiles, K action planes; the
 * bit-sliced block kernel) — DESIGN.md §RNG; the oracle needs it to replay the schedule. */
ESCG_API int escg_dev_draw_format(escg_dev* h, int32_t* narrow);

/* Block kernel mode: MCS per chunk (temporal blocking; 1 for the tile kernel; 0 for the ring kernel,
 * whose launch covers the whole advance/run) and whether a run executes as one persistent
 * cooperative launch (1) or one launch per chunk (0). */
ESCG_API int escg_dev_block_mode(escg_dev* h, int32_t* kmcs, int32_t* persistent);

/* Row-band sharding of one lattice.  Band `band` of `n_bands` (rows split at
 * multiples of 4) with halo = 12*kmcs rows on each side; draws use global coordinates, so a band
 * group reproduces the single-lattice run bit-for-bit.  set/get/counts address the band rows. */
ESCG_API int escg_dev_create_band(const escg_params* p, const double* dominance, int32_t species, int32_t kind,
                                  int32_t device, int32_t n_bands, int32_t band, int32_t kmcs, escg_dev** out);
ESCG_API int escg_dev_band_info(escg_dev* h, int32_t* band_start, int32_t* band_rows, int32_t* halo, int32_t* kmcs);
/* Advance a whole band group (bands[g] = band g; any mix of devices) by n_mcs: per chunk, halo
 * exchange by peer copies between ring neighbours, then the block kernel on every band. */
ESCG_API int escg_group_advance(escg_dev** bands, int32_t n, int64_t n_mcs);
/* Primitives of a multi-process band group (one rank per GPU, halos moved by the caller, e.g. NCCL
 * send/recv): device pointers into the band's current buffer — the top halo rows, the first
 * `halo` band rows (sent up), the last `halo` band rows (sent down), the bottom halo rows — and the
 * byte count of each: halo * L for u8 rows, halo * NPL * L/128 * 16 when the band runs the
 * bit-sliced kernel (draw format 2: the band stays in bit-plane rows between steps, and
 * get/counts convert back on demand).  Valid until the next escg_dev_band_step. */
ESCG_API int escg_dev_band_rows(escg_dev* h, uint8_t** recv_top, uint8_t** send_top, uint8_t** send_bot,
                                uint8_t** recv_bot, int64_t* bytes);
/* One chunk (1 <= n_mcs <= kmcs) of MCS on this band alone; the halos must hold the neighbours'
 * current rows.  Synchronous. */
ESCG_API int escg_dev_band_step(escg_dev* h, int32_t n_mcs);

/* Issue the engine's work on a caller's CUDA stream (a cudaStream_t; NULL: the engine's own stream).
 * On a caller's stream escg_dev_band_rows / escg_dev_band_step do not synchronise the host: a band
 * step is enqueued after, and before, the caller's halo exchange on that stream (device-ordered
 * stepping, bands.DistributedBand).  Replaces the host synchronisation per chunk of SURVEY §8e's
 * exchange loop; the reference's counterpart is the refill/step overlap of engine.cpp:142-162. */
ESCG_API int escg_dev_set_stream(escg_dev* h, void* stream);

/* Multi-part ring (the reference's row split of engine.cpp:119-131 across GPUs): part
 * `part` of `n_parts` (2..8; rows split at multiples of 4, >= 8 rows each) of one bit-sliced
 * lattice runs the persistent ring kernel over n_ctas bands of its rows (0: one per SM).  Its
 * boundary bands exchange rows with the neighbouring parts inside the kernel, every colour phase,
 * by system-scope tagged stores into the neighbour's inbox (NVLink peer memory on another GPU) —
 * no host step, no copy kernel.  State stays in bit planes; set/get/counts address the part's rows.
 * Wiring: escg_dev_ring_part_export gives the part's plane buffers, inbox and row count (and, if
 * `ipc` is not NULL, 3 x 64 bytes of cudaIpcMemHandle_t for planes 0, planes 1 and the mailbox
 * allocation, the inbox at *inbox_offset bytes into it); escg_dev_ring_part_connect takes the part
 * above's and below's (pointers valid on this part's device: same device, peer access, or
 * escg_ipc_open).  Then either escg_ring_group_advance over all parts from one process (one
 * device: ONE cooperative launch over every part — the single-GPU form of the multi-GPU kernel;
 * several devices: one launch per part, peer access enabled), or escg_dev_advance on each rank's
 * part (one process per GPU; the launches meet through their inbox words, the host does not wait).
 * set_lattice / init_lattice must be called on every part before the next advance of any. */
ESCG_API int escg_dev_create_ring_part(const escg_params* p, const double* dominance, int32_t species, int32_t kind,
                                       int32_t device, int32_t n_parts, int32_t part, int32_t n_ctas, escg_dev** out);
ESCG_API int escg_dev_ring_part_export(escg_dev* h, void** planes0, void** planes1, void** inbox, int32_t* rows,
                                       void* ipc, int64_t* inbox_offset);
ESCG_API int escg_dev_ring_part_connect(escg_dev* h, void* up_planes0, void* up_planes1, void* up_inbox,
                                        int32_t up_rows, void* dn_planes0, void* dn_planes1, void* dn_inbox,
                                        int32_t dn_rows);
ESCG_API int escg_ring_group_advance(escg_dev** parts, int32_t n, int64_t n_mcs);
/* CUDA IPC (one process per GPU): open a peer's 64-byte allocation handle on `device` / close it. */
ESCG_API int escg_ipc_open(int32_t device, const void* handle, void** ptr);
ESCG_API int escg_ipc_close(int32_t device, void* ptr);

/* One-call mirror of escg::simulate(params, model, mode, …) (engine.cpp:194-240) for a single
 * lattice: initialise on device (or resume from resume_cells at resume_mcs), run to completion
 * under `mode`'s record cadence with the device stop predicates, return the final int32 lattice,
 * the density trace and the status.  Host buffers in, host buffers out. */
ESCG_API int escg_simulate(const escg_params* p, const double* dominance, int32_t species, int32_t kind, int32_t mode,
                  int32_t device, const int32_t* resume_cells, int64_t resume_mcs, uint32_t stop_flags,
                  int32_t tracked_species, int32_t* out_cells, int64_t* out_mcs, int64_t* steps, uint64_t* counts,
                  int64_t cap, int64_t* n_records, int32_t* status);

#ifdef __cplusplus
}
#endif
#endif /* ESCG_DEV_H */
