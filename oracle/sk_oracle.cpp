// oracle/sk_oracle.cpp -- C driver over the UNMODIFIED reference core.
//
// TEST INFRASTRUCTURE ONLY: the checker and the CPU baseline, never the
// product.  Compiled together with /root/reference/proj/src/*.cpp (read in
// place, never copied) and oracle/fft_shim.c by oracle/Makefile into
// oracle/_ref/libskref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's CPU legs load it.
//
// Every entry point drives the reference through its own public API:
//   create      -> create_default_params + Simulation ctor
//                  (proj/src/simulation.cpp:74-134, 297-346), files and
//                  forcing off, init "constant 0" (simulation.cpp:352-359),
//                  fixed dt (simulation.cpp:463-469), as run_bench does
//                  (proj/src/bench.cpp:51-85);
//   set_state   -> StateSet::spect_mut (proj/include/spectralkit/state.hpp)
//   step        -> Simulation::step_once (simulation.cpp:535-555)
//   run         -> Simulation::run (simulation.cpp:565-590)
//   tendency    -> Simulation::compute_tendency (simulation.cpp:478-480)
//   fft_*       -> plan_fft()->forward/inverse (proj/src/fft.cpp:92-137)
//   grid        -> SpectralGrid k_axis / dealias_mask (proj/src/grid.cpp:20-110)
//   create_files-> the same Simulation with output.enable_files on (its
//                  OutputManager writes params.txt, snapshots/*.fld and the
//                  spectra / budget records, proj/src/output.cpp:105-300)
//   restart     -> load_state_phys_file (proj/src/simulation.cpp:705-732)
// Errors are caught and mapped to the same status codes as include/skgpu.h.
#include <chrono>
#include <complex>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "spectralkit/errors.hpp"
#include "spectralkit/fft.hpp"
#include "spectralkit/grid.hpp"
#include "spectralkit/output.hpp"
#include "spectralkit/simulation.hpp"

using namespace spectralkit;

namespace {

thread_local std::string g_err;

enum {
    SKR_OK = 0,
    SKR_ECONFIG = 1,
    SKR_ESHAPE = 2,
    SKR_EDIVERGENCE = 3,
    SKR_EOTHER = 9,
};

struct RefSim {
    std::unique_ptr<Simulation> sim;
    long div_iteration = -1;
    int div_var = -1;
};

template <typename F>
int guard(F&& f, RefSim* rs = nullptr) {
    try {
        f();
        return SKR_OK;
    } catch (const DivergenceError& e) {
        g_err = e.what();
        if (rs) {
            rs->div_iteration = e.iteration;
            const auto& keys = rs->sim->info().keys_state_spect;
            for (std::size_t v = 0; v < keys.size(); ++v)
                if (keys[v] == e.field) rs->div_var = static_cast<int>(v);
        }
        return SKR_EDIVERGENCE;
    } catch (const ShapeError& e) {
        g_err = e.what();
        return SKR_ESHAPE;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return SKR_ECONFIG;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SKR_EOTHER;
    }
}

}  // namespace

extern "C" {

const char* skref_last_error(void) { return g_err.c_str(); }

void skref_set_workers(int n) { set_fft_workers(n); }

static int create_impl(RefSim** out, const char* solver, int dims, const int* n, double nu,
                       double fixed_dt, int scheme_rk2, double dealias_coef, int forcing,
                       double k_lo, double k_hi, double rate, long seed,
                       const char* root_dir = nullptr, double period_save = 0.0);

int skref_create(RefSim** out, const char* solver, int dims, const int* n, double nu,
                 double fixed_dt, int scheme_rk2, double dealias_coef) {
    return create_impl(out, solver, dims, n, nu, fixed_dt, scheme_rk2, dealias_coef, 0, 2.0, 4.0,
                       1.0, 1234);
}

// The same with forcing.enable = true and its band, rate and seed
// (create_default_params forcing.*, simulation.cpp:112-117).
int skref_create_forced(RefSim** out, const char* solver, int dims, const int* n, double nu,
                        double fixed_dt, int scheme_rk2, double dealias_coef, double k_lo,
                        double k_hi, double rate, long seed) {
    return create_impl(out, solver, dims, n, nu, fixed_dt, scheme_rk2, dealias_coef, 1, k_lo, k_hi,
                       rate, seed);
}

// Files on: the run directory goes under root_dir (output.root_dir), records
// and a snapshot every period_save of simulated time (output.period_save),
// plus at run start and end (OutputManager on_run_start / on_run_end).
int skref_create_files(RefSim** out, const char* solver, int dims, const int* n, double nu,
                       double fixed_dt, int scheme_rk2, double dealias_coef, const char* root_dir,
                       double period_save) {
    return create_impl(out, solver, dims, n, nu, fixed_dt, scheme_rk2, dealias_coef, 0, 2.0, 4.0,
                       1.0, 1234, root_dir, period_save);
}

// The run directory of a files-on simulation (OutputManager::dir, output.hpp:49).
int skref_output_dir(RefSim* rs, char* buf, long len) {
    return guard([&] {
        const std::string& d = rs->sim->output().dir();
        if (static_cast<long>(d.size()) + 1 > len) throw ConfigError("buffer too small");
        std::memcpy(buf, d.c_str(), d.size() + 1);
    });
}

// Restart from a run directory's snapshot (time < 0: the latest):
// load_state_phys_file checks the snapshot's digest against params.txt
// (simulation.cpp:705-732).
int skref_restart(RefSim** out, const char* dir, double time) {
    *out = nullptr;
    return guard([&] {
        ensure_builtin_solvers();
        auto rs = std::make_unique<RefSim>();
        rs->sim = load_state_phys_file(dir, time);
        rs->sim->set_quiet(true);
        *out = rs.release();
    });
}

double skref_last_injection(RefSim* rs) { return rs->sim->last_injection(); }

static int create_impl(RefSim** out, const char* solver, int dims, const int* n, double nu,
                       double fixed_dt, int scheme_rk2, double dealias_coef, int forcing,
                       double k_lo, double k_hi, double rate, long seed, const char* root_dir,
                       double period_save) {
    *out = nullptr;
    return guard([&] {
        ensure_builtin_solvers();
        ParamTree p = create_default_params(solver);
        static const char* ns[] = {"nx", "ny", "nz"};
        for (int d = 0; d < dims; ++d)
            p.set(std::string("oper.") + ns[d], static_cast<std::int64_t>(n[d]));
        if (dealias_coef > 0) p.set("oper.dealias_coef", dealias_coef);
        p.set("nu_2", nu);
        p.set("output.enable_files", root_dir != nullptr);
        if (root_dir) {
            p.set("output.root_dir", std::string(root_dir));
            p.set("output.period_save", period_save);
        }
        p.set("forcing.enable", forcing != 0);
        if (forcing) {
            p.set("forcing.k_lo", k_lo);
            p.set("forcing.k_hi", k_hi);
            p.set("forcing.rate", rate);
            p.set("forcing.seed", static_cast<std::int64_t>(seed));
        }
        p.set("time_stepping.scheme", std::string(scheme_rk2 ? "RK2" : "RK4"));
        p.set("time_stepping.fixed_dt", fixed_dt);
        p.set("time_stepping.t_end", -1.0);
        p.set("time_stepping.n_iters", static_cast<std::int64_t>(1));
        p.set("init_fields.type", std::string("constant"));
        p.set("init_fields.constant.value", 0.0);
        auto rs = std::make_unique<RefSim>();
        rs->sim = std::make_unique<Simulation>(p);
        rs->sim->set_quiet(true);
        *out = rs.release();
    });
}

void skref_destroy(RefSim* rs) { delete rs; }

long skref_spect_size(RefSim* rs) { return static_cast<long>(rs->sim->oper().spect_size); }
long skref_phys_size(RefSim* rs) { return static_cast<long>(rs->sim->oper().phys_size); }
int skref_nvars(RefSim* rs) { return static_cast<int>(rs->sim->state().spect().size()); }

int skref_set_state(RefSim* rs, const double* spect) {
    return guard([&] {
        StateVec& s = rs->sim->state().spect_mut();
        std::size_t S = rs->sim->oper().spect_size;
        for (std::size_t v = 0; v < s.size(); ++v)
            std::memcpy(s[v].data(), spect + 2 * S * v, S * sizeof(std::complex<double>));
    });
}

int skref_get_state(RefSim* rs, double* spect) {
    return guard([&] {
        const StateVec& s = rs->sim->state().spect();
        std::size_t S = rs->sim->oper().spect_size;
        for (std::size_t v = 0; v < s.size(); ++v)
            std::memcpy(spect + 2 * S * v, s[v].data(), S * sizeof(std::complex<double>));
    });
}

// Calls step_once nsteps times; *seconds = wall time of the loop.
int skref_step(RefSim* rs, long nsteps, double* seconds) {
    return guard(
        [&] {
            auto t0 = std::chrono::steady_clock::now();
            for (long i = 0; i < nsteps; ++i) rs->sim->step_once();
            std::chrono::duration<double> d = std::chrono::steady_clock::now() - t0;
            if (seconds) *seconds = d.count();
        },
        rs);
}

// Simulation::run() with n_iters = nsteps (adds per-step means + check_finite).
int skref_run(RefSim* rs, long nsteps, double* seconds) {
    return guard(
        [&] {
            rs->sim->set_n_iters(nsteps);
            RunSummary r = rs->sim->run();
            if (seconds) *seconds = r.walltime;
        },
        rs);
}

int skref_last_divergence(RefSim* rs, long* iteration, int* var) {
    *iteration = rs->div_iteration;
    *var = rs->div_var;
    return SKR_OK;
}

int skref_tendency(RefSim* rs, const double* in, double* out) {
    return guard([&] {
        std::size_t S = rs->sim->oper().spect_size;
        std::size_t nv = rs->sim->state().spect().size();
        StateVec s(nv, std::vector<std::complex<double>>(S));
        for (std::size_t v = 0; v < nv; ++v)
            std::memcpy(s[v].data(), in + 2 * S * v, S * sizeof(std::complex<double>));
        StateVec o;
        rs->sim->compute_tendency(s, o);
        for (std::size_t v = 0; v < nv; ++v)
            std::memcpy(out + 2 * S * v, o[v].data(), S * sizeof(std::complex<double>));
    });
}

double skref_energy(RefSim* rs) { return rs->sim->energy(); }
double skref_enstrophy(RefSim* rs) { return rs->sim->enstrophy(); }
double skref_time(RefSim* rs) { return rs->sim->t(); }
long skref_iteration(RefSim* rs) { return rs->sim->iteration(); }

// axis k values (length spect_shape[axis]) and, if mask != NULL, the full mask.
int skref_grid(RefSim* rs, int axis, double* k_axis, unsigned char* mask) {
    return guard([&] {
        const SpectralGrid& g = rs->sim->oper();
        if (axis < 0 || axis >= g.dims) throw ShapeError("axis out of range");
        std::memcpy(k_axis, g.k_axis[axis].data(), g.k_axis[axis].size() * sizeof(double));
        if (mask) std::memcpy(mask, g.dealias_mask.data(), g.dealias_mask.size());
    });
}

// Plain transform operators: FftPlan::forward / inverse for a shape.
int skref_fft_forward(int rank, const int* shape, const double* u, double* uhat) {
    return guard([&] {
        auto plan = plan_fft(std::vector<int>(shape, shape + rank));
        plan->forward(u, reinterpret_cast<std::complex<double>*>(uhat));
    });
}

int skref_fft_inverse(int rank, const int* shape, const double* uhat, double* u) {
    return guard([&] {
        auto plan = plan_fft(std::vector<int>(shape, shape + rank));
        plan->inverse(reinterpret_cast<const std::complex<double>*>(uhat), u);
    });
}

}  // extern "C"
