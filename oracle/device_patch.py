"""Build the reference with the B200 engine plugged in, as a test binary.

    python oracle/device_patch.py [REFERENCE_PROJ] [OUT_BINARY]

Test infrastructure only.  Copies the unmodified reference sources to a scratch directory under
/tmp (never into this repository), applies the two-line EngineMode::Device seam that INTEGRATION.md
documents plus the `run_device` helper below, and links the reference's own `simulate()` against
libescg_b200.so.  The demo main (DEMO) calls escg::simulate(params, model, EngineMode::Device) and
prints the result; tests/test_gpu_parity.py::test_reference_simulate_dispatches_to_device_engine runs
it on the GPU box and checks it against this package's simulate() from the same initial lattice.
The binary lands in oracle/_ref/ (git-ignored, travels to the GPU box with the snapshot).
"""
import os
import shutil
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

# The helper INTEGRATION.md §1 shows, compiled for real (inside namespace escg, next to run_max_step).
RUN_DEVICE = r'''
// ---- EngineMode::Device (B200 engine, include/escg_dev.h; INTEGRATION.md §1) ------------------
RunStatus run_device(RunState& state, const SimParams& params, const RunHooks& hooks) {
    escg_params p{};
    escg_params_default(&p);
    p.length = params.length; p.height = params.height; p.mcs_limit = params.mcs_limit;
    p.neighbourhood = static_cast<int>(params.neighbourhood); p.print_frequency = params.print_frequency;
    p.mobility = params.mobility; p.species = params.species; p.flux = params.flux;
    p.empty_prob = params.empty_prob; p.num_randoms = params.num_randoms; p.max_step = params.max_step;
    p.has_seed = params.seed.has_value(); p.seed = params.seed.value_or(0);
    escg_dev* h = nullptr;
    if (escg_dev_create(&p, state.model.entries.data(), state.model.size,
                        state.model.kind == DominanceModel::Kind::Rated ? ESCG_DOM_RATED : ESCG_DOM_BINARY,
                        /*device*/ 0, /*replicas*/ 1, nullptr, ESCG_KERNEL_AUTO, &h) != ESCG_OK)
        throw EngineError(escg_dev_last_error());
    if (escg_dev_set_lattice(h, 0, state.lattice.cells.data(), state.current_mcs) != ESCG_OK)
        throw EngineError(escg_dev_last_error());
    const std::int64_t n = state.lattice.size();
    const std::int64_t interval = params.max_step ? align_num_randoms(params.num_randoms, n) / n : 1;
    RunStatus status;
    for (;;) {  // record_and_check (engine.cpp:47-57) with host hooks between device advances
        std::vector<std::uint64_t> c(params.species + 1);
        escg_dev_counts(h, 0, c.data());
        state.trace.append(state.current_mcs, c);
        if (hooks.on_record || hooks.on_save) escg_dev_get_lattice(h, 0, state.lattice.cells.data(), nullptr);
        if (hooks.console && state.current_mcs % params.print_frequency == 0) print_density_line(*hooks.console, state);
        if (params.save && hooks.on_save && is_save_mcs(state.current_mcs, params.mcs_limit)) hooks.on_save(state);
        if (hooks.on_record && !hooks.on_record(state)) { status = RunStatus::Stopped; break; }
        if (state.current_mcs >= params.mcs_limit) { status = RunStatus::Completed; break; }
        if (stasis(state.trace)) { status = RunStatus::Stasis; break; }
        const std::int64_t adv = std::min(interval, params.mcs_limit - state.current_mcs);
        escg_dev_advance(h, adv);
        state.current_mcs += adv;
    }
    escg_dev_get_lattice(h, 0, state.lattice.cells.data(), nullptr);
    escg_dev_destroy(h);
    return status;
}

'''

DEMO = r'''// Demo: the reference's own simulate() dispatching to EngineMode::Device.
#include <cstdio>
#include <cstdint>

#include "escg/engine.hpp"
#include "escg/experiments.hpp"
#include "escg/lattice.hpp"
#include "escg/random_batch.hpp"

static std::uint64_t fnv1a(const std::vector<std::int32_t>& v) {
    std::uint64_t h = 1469598103934665603ull;
    for (auto x : v) {
        for (int b = 0; b < 4; ++b) {
            h ^= static_cast<std::uint8_t>(static_cast<std::uint32_t>(x) >> (8 * b));
            h *= 1099511628211ull;
        }
    }
    return h;
}

int main(int argc, char** argv) {
    escg::SimParams p;
    p.length = argc > 1 ? std::atoi(argv[1]) : 64;
    p.height = argc > 2 ? std::atoi(argv[2]) : 48;
    p.mcs_limit = argc > 3 ? std::atoll(argv[3]) : 120;
    p.mobility = 1e-3;
    p.empty_prob = 0.1;
    p.seed = 77;
    p.print_frequency = 1000000;
    const auto model = escg::make_circulant(3, {1});
    escg::StreamSet streams(*p.seed, 1);
    const auto init = escg::init_lattice(p, streams.stream(0));
    escg::RunState start;
    start.lattice = init;
    auto r = escg::simulate(p, model, escg::EngineMode::Device, nullptr, {}, nullptr, start);
    std::uint64_t total = 0;
    for (auto c : r.state.trace.counts.back()) total += c;
    std::printf("status=%d mcs=%lld records=%zu total=%llu init_fnv=%016llx final_fnv=%016llx\n",
                static_cast<int>(r.status), static_cast<long long>(r.state.current_mcs), r.state.trace.counts.size(),
                static_cast<unsigned long long>(total), static_cast<unsigned long long>(fnv1a(init.cells)),
                static_cast<unsigned long long>(fnv1a(r.state.lattice.cells)));
    return 0;
}
'''


def patch(src_dir):
    hpp = os.path.join(src_dir, "include", "escg", "engine.hpp")
    s = open(hpp).read()
    old = "enum class EngineMode { Serial, ParallelMcs, MaxStep };"
    assert old in s, "engine.hpp: EngineMode enum not found"
    open(hpp, "w").write(s.replace(old, "enum class EngineMode { Serial, ParallelMcs, MaxStep, Device };"))
    cpp = os.path.join(src_dir, "src", "engine.cpp")
    s = open(cpp).read()
    anchor = "SimulationResult simulate(const SimParams& params, const DominanceModel& model, EngineMode mode,"
    assert anchor in s, "engine.cpp: simulate() not found"
    s = s.replace(anchor, RUN_DEVICE + anchor, 1)
    case = "        case EngineMode::MaxStep:\n            result.status = run_max_step(result.state, params, *streams, *pool, hooks);\n            break;\n"
    assert case in s, "engine.cpp: dispatch switch not found"
    s = s.replace(case, case + "        case EngineMode::Device:\n            result.status = run_device(result.state, params, hooks);\n            break;\n", 1)
    s = '#include "escg_dev.h"\n' + s
    open(cpp, "w").write(s)


def main():
    ref = sys.argv[1] if len(sys.argv) > 1 else "/root/reference/proj"
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(HERE, "_ref", "escg_device_demo")
    lib_dir = os.path.join(ROOT, "paper_2508_16639_b200")
    if not os.path.isdir(os.path.join(ref, "src")):
        print("reference sources absent: skipping the EngineMode::Device demo")
        return 0
    if not os.path.exists(os.path.join(lib_dir, "libescg_b200.so")):
        print("libescg_b200.so not built: skipping the EngineMode::Device demo")
        return 0
    with tempfile.TemporaryDirectory(prefix="escg_ref_device_") as tmp:
        shutil.copytree(os.path.join(ref, "include"), os.path.join(tmp, "include"))
        shutil.copytree(os.path.join(ref, "src"), os.path.join(tmp, "src"))
        patch(tmp)
        open(os.path.join(tmp, "demo.cpp"), "w").write(DEMO)
        srcs = [os.path.join(tmp, "src", f) for f in ("engine.cpp", "dominance.cpp", "experiments.cpp",
                                                       "persistence.cpp", "stats.cpp")]
        os.makedirs(os.path.dirname(out), exist_ok=True)
        cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(tmp, "include"), "-I", os.path.join(ROOT, "include"),
               *srcs, os.path.join(tmp, "demo.cpp"), "-L", lib_dir, "-lescg_b200",
               "-Wl,-rpath,$ORIGIN/../../paper_2508_16639_b200", "-lpthread", "-o", out]
        subprocess.run(cmd, check=True)
    print("built", out)
    return 0


if __name__ == "__main__":
    sys.exit(main())
