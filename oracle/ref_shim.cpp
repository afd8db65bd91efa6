// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference engine.
//
//   *** TEST INFRASTRUCTURE ONLY ***  (oracle/_ref/libescg_ref.so)
//   Compiled by oracle/Makefile directly from /root/reference/proj/src/*.cpp and the reference
//   headers (no reference source is copied into this repository).  Used to pin the C restatement
//   (escg_oracle.c), to generate tests/golden/ fixtures, and as the timed CPU baseline
//   (bench.py --impl reference / cpu_baseline.kind == "reference").
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "escg/dominance.hpp"
#include "escg/engine.hpp"
#include "escg/errors.hpp"
#include "escg/experiments.hpp"
#include "escg/lattice.hpp"
#include "escg/mt19937.hpp"
#include "escg/params.hpp"
#include "escg/random_batch.hpp"
#include "escg/stats.hpp"
#include "escg/thread_pool.hpp"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

int code_of(const std::exception& e) {
    if (dynamic_cast<const escg::ConfigError*>(&e)) return 2;
    if (dynamic_cast<const escg::IoError*>(&e)) return 3;
    if (dynamic_cast<const escg::FormatError*>(&e)) return 4;
    return 5;
}

escg::DominanceModel model_of(const double* dom, int species, int rated) {
    escg::DominanceModel m;
    m.size = species;
    m.kind = rated ? escg::DominanceModel::Kind::Rated : escg::DominanceModel::Kind::Binary;
    m.entries.assign(dom, dom + static_cast<std::size_t>(species) * species);
    return m;
}

escg::SimParams params_of(int length, int height, int species, int arity, int flux, double mobility,
                          double empty_prob, std::int64_t mcs_limit, std::int64_t num_randoms, std::uint64_t seed) {
    escg::SimParams p;
    p.length = length;
    p.height = height;
    p.species = species;
    p.neighbourhood = arity == 8 ? escg::Neighbourhood::Moore8 : escg::Neighbourhood::VonNeumann4;
    p.flux = flux != 0;
    p.mobility = mobility;
    p.empty_prob = empty_prob;
    p.mcs_limit = mcs_limit;
    p.num_randoms = num_randoms;
    p.max_step = false;
    p.seed = seed;
    return p;
}

}  // namespace

// StreamSet(seed, count) stream k, n words after the burn-in (random_batch.hpp:44-53).
EXPORT int ref_stream_words(std::uint64_t seed, int count, int k, std::int64_t n, std::uint32_t* out) {
    try {
        escg::StreamSet streams(seed, count);
        auto& g = streams.stream(k);
        for (std::int64_t i = 0; i < n; ++i) out[i] = g.extract();
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Raw MT19937 (no seed mixing, no burn-in) for the SPEC KATs.
EXPORT void ref_mt_raw(std::uint32_t seed, std::int64_t n, std::uint32_t* out) {
    escg::Mt19937 g(seed);
    for (std::int64_t i = 0; i < n; ++i) out[i] = g.extract();
}

EXPORT std::uint32_t ref_seed_mix(std::uint32_t seed, std::uint32_t id) { return escg::seed_mix(seed, id); }

EXPORT std::int64_t ref_align_num_randoms(std::int64_t requested, std::int64_t cells) {
    try {
        return escg::align_num_randoms(requested, cells);
    } catch (const std::exception&) {
        return -1;
    }
}

EXPORT void ref_action_rates(double mobility, std::int64_t cells, double* out) {
    auto r = escg::action_rates(mobility, cells);
    out[0] = r.mu;
    out[1] = r.sigma;
    out[2] = r.epsilon;
    out[3] = r.total;
}

EXPORT std::int64_t ref_neighbor_index(std::int64_t i, int dir, int arity, int length, int height, int flux) {
    try {
        auto spec = escg::NeighborhoodSpec::of(arity == 8 ? escg::Neighbourhood::Moore8
                                                          : escg::Neighbourhood::VonNeumann4);
        return escg::neighbor_index(i, dir, spec, length, height, flux != 0);
    } catch (const std::exception&) {
        return -1;
    }
}

// init_lattice on StreamSet(seed,1) stream 0, exactly as simulate() does (engine.cpp:222).
EXPORT int ref_init_lattice(int length, int height, int species, double empty_prob, std::uint64_t seed,
                            std::int32_t* out) {
    try {
        auto p = params_of(length, height, species, 4, 1, 3e-5, empty_prob, 0, 100000000, seed);
        escg::StreamSet streams(seed, 1);
        auto lat = escg::init_lattice(p, streams.stream(0));
        std::memcpy(out, lat.cells.data(), sizeof(std::int32_t) * lat.cells.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// One elementary_step<PlainCellAccess> (engine.hpp:108-141) on a caller-owned int32 lattice.
EXPORT int ref_elementary_step(std::int32_t* cells, int length, int height, int species, int arity, int flux,
                               const double* dom, int rated, double mobility, std::int64_t cell, int dir,
                               float action) {
    try {
        escg::DominanceModel m = model_of(dom, species, rated);
        escg::StepContext ctx{&m,
                              escg::action_rates(mobility, static_cast<std::int64_t>(length) * height),
                              escg::NeighborhoodSpec::of(arity == 8 ? escg::Neighbourhood::Moore8
                                                                    : escg::Neighbourhood::VonNeumann4),
                              length,
                              height,
                              flux != 0};
        escg::PlainCellAccess grid{cells};
        escg::elementary_step(grid, ctx, escg::StepDraw{cell, dir, action});
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// simulate(params, model, mode) (engine.cpp:194-240).  mode: 0 Serial, 1 ParallelMcs, 2 MaxStep.
// tracked >= 1 installs the experiments-harness predicate (experiments.cpp:107-113).
// init_cells (optional) resumes from a given lattice at MCS 0 (engine.cpp:219-221).
// elapsed_s: wall time from the first on_record callback to return (SURVEY §8d window).
EXPORT int ref_simulate(int mode, int workers, int length, int height, int species, int arity, int flux,
                        const double* dom, int rated, double mobility, double empty_prob, std::int64_t mcs_limit,
                        std::int64_t num_randoms, std::uint64_t seed, int tracked, const std::int32_t* init_cells,
                        std::int32_t* out_cells, std::int64_t* steps, std::uint64_t* counts, std::int64_t cap,
                        std::int64_t* n_rec, int* status, double* elapsed_s) {
    try {
        auto p = params_of(length, height, species, arity, flux, mobility, empty_prob, mcs_limit, num_randoms, seed);
        p.max_step = mode == 2;
        escg::DominanceModel m = model_of(dom, species, rated);
        const escg::EngineMode em =
            mode == 0 ? escg::EngineMode::Serial : (mode == 1 ? escg::EngineMode::ParallelMcs : escg::EngineMode::MaxStep);
        std::unique_ptr<escg::ThreadPool> pool;
        if (mode != 0) pool = std::make_unique<escg::ThreadPool>(workers > 0 ? workers : 1);
        std::chrono::steady_clock::time_point t0;
        bool started = false;
        escg::RunHooks hooks;
        hooks.on_record = [&](const escg::RunState& st) {
            if (!started) {
                started = true;
                t0 = std::chrono::steady_clock::now();
            }
            if (tracked >= 1 && st.trace.counts.back()[tracked] == 0) return false;
            return true;
        };
        std::optional<escg::RunState> resume;
        std::unique_ptr<escg::StreamSet> streams;
        if (init_cells) {
            escg::RunState rs;
            rs.lattice = escg::Lattice(length, height);
            std::memcpy(rs.lattice.cells.data(), init_cells, sizeof(std::int32_t) * rs.lattice.cells.size());
            rs.current_mcs = 0;
            resume = std::move(rs);
        }
        auto res = escg::simulate(p, m, em, pool.get(), hooks, nullptr, std::move(resume));
        const auto t1 = std::chrono::steady_clock::now();
        if (elapsed_s) *elapsed_s = started ? std::chrono::duration<double>(t1 - t0).count() : 0.0;
        if (out_cells)
            std::memcpy(out_cells, res.state.lattice.cells.data(), sizeof(std::int32_t) * res.state.lattice.cells.size());
        const auto& tr = res.state.trace;
        *n_rec = static_cast<std::int64_t>(tr.steps.size());
        for (std::int64_t r = 0; r < *n_rec && r < cap; ++r) {
            if (steps) steps[r] = tr.steps[r];
            if (counts)
                for (int s = 0; s <= species; ++s) counts[r * (species + 1) + s] = tr.counts[r][s];
        }
        *status = static_cast<int>(res.status);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Dominance presets (dominance.cpp:23-42, experiments.cpp:53-76); out = S*S doubles.
EXPORT int ref_make_circulant(int species, const int* offsets, int n_offsets, double* out) {
    try {
        auto m = escg::make_circulant(species, std::vector<int>(offsets, offsets + n_offsets));
        std::memcpy(out, m.entries.data(), sizeof(double) * m.entries.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

EXPORT void ref_make_rpsls_ablated(double* out) {
    auto m = escg::make_rpsls_ablated();
    std::memcpy(out, m.entries.data(), sizeof(double) * m.entries.size());
}

EXPORT int ref_make_park8(double alpha, double beta, double gamma, double* out) {
    try {
        auto m = escg::make_park8(alpha, beta, gamma);
        std::memcpy(out, m.entries.data(), sizeof(double) * m.entries.size());
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

EXPORT int ref_validate_dominance(const double* dom, int species, int rated) {
    try {
        model_of(dom, species, rated).validate();
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Statistics used by the statistical-parity tests (stats.cpp).
EXPORT double ref_ks_two_sample_pvalue(const double* a, std::int64_t na, const double* b, std::int64_t nb) {
    return escg::ks_two_sample_pvalue(std::vector<double>(a, a + na), std::vector<double>(b, b + nb));
}

EXPORT double ref_chi_square_uniform_pvalue(const std::uint64_t* bins, std::int64_t n) {
    return escg::chi_square_uniform_pvalue(std::vector<std::uint64_t>(bins, bins + n));
}

// persistence.cpp:57-62 format_double (std::to_chars shortest round-trip), for the CSV formats.
#include "escg/persistence.hpp"
EXPORT int ref_format_double(double v, char* buf, int cap) {
    const std::string s = escg::format_double(v);
    if (static_cast<int>(s.size()) + 1 > cap) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return static_cast<int>(s.size());
}

// experiments.cpp:242-285 CSV writers on caller data (format pins for the device harness).
#include "escg/experiments.hpp"
EXPORT int ref_write_extinction_csv(const std::int64_t* times, const int* censored, int n, const char* path) {
    try {
        escg::ExtinctionStats st;
        for (int i = 0; i < n; ++i) {
            st.times.push_back(times[i]);
            st.censored.push_back(censored[i] != 0);
        }
        escg::write_extinction_csv(st, path);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

EXPORT int ref_write_coexistence_csv(int trials, int coexisting, double probability, double mobility, int length,
                                     std::int64_t mcs, const char* path) {
    try {
        escg::CoexistenceResult r;
        r.trials = trials;
        r.coexisting = coexisting;
        r.probability = probability;
        escg::write_coexistence_csv(r, mobility, length, mcs, path);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}

// Checkpoint round trip through the reference (persistence.cpp:322-351): load `src` (written by the
// device engine), save it again into `dst`.  Used out of process by ref_csv_tool.
EXPORT int ref_checkpoint_roundtrip(const char* src, const char* dst) {
    try {
        auto cp = escg::load_checkpoint(src);
        escg::save_checkpoint(dst, cp.params, cp.lattice, cp.dominance, cp.saved_mcs);
        return 0;
    } catch (const std::exception& e) {
        fprintf(stderr, "%s\n", e.what());
        return code_of(e);
    }
}

EXPORT int ref_output_dir_name(int length, int height, int n, double mobility, int flux, int species, char* buf,
                               int cap) {
    escg::SimParams p;
    p.length = length;
    p.height = height;
    p.neighbourhood = n == 8 ? escg::Neighbourhood::Moore8 : escg::Neighbourhood::VonNeumann4;
    p.mobility = mobility;
    p.flux = flux != 0;
    p.species = species;
    const std::string s = escg::output_dir_name(p);
    if (static_cast<int>(s.size()) + 1 > cap) return -1;
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

EXPORT int ref_write_densities(const std::int64_t* steps, const std::uint64_t* counts, int n, int species,
                               const char* path, int append) {
    try {
        escg::DensityTrace tr;
        for (int i = 0; i < n; ++i)
            tr.append(steps[i], std::vector<std::uint64_t>(counts + static_cast<size_t>(i) * (species + 1),
                                                          counts + static_cast<size_t>(i + 1) * (species + 1)));
        escg::export_densities(tr, path, append != 0);
        return 0;
    } catch (const std::exception& e) {
        return code_of(e);
    }
}
