// integration/skgpu_solver.cpp -- reference-side plugin.
//
// What a spectralkit maintainer adds to run the reference's OWN Simulation /
// ExactLinStepper / OutputManager on the B200 tendency: a Solver subclass per
// equation whose tendency() calls skg_tendency() (include/skgpu.h), registered
// through the public registry exactly like the NanSolver precedent of
// proj/tests/unit/test_simulation.cpp:454-494.  Solver API:
// proj/include/spectralkit/simulation.hpp:23-68; registration:
// simulation.hpp:70-86, src/simulation.cpp:33-40.
//
// The extern "C" skgi_* functions let tests drive the reference Simulation
// with either the CPU solver ("ns2d") or this plugin ("ns2d_gpu").
#include <complex>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "skgpu.h"
#include "spectralkit/errors.hpp"
#include "spectralkit/simulation.hpp"

using namespace spectralkit;

namespace {

SolverInfo gpu_info(const std::string& name, int dims, std::vector<std::string> phys) {
    register_component_id("state." + name);
    SolverInfo i;
    i.short_name = name;
    i.dims = dims;
    static const char* oper[] = {"operators.spectral_1d", "operators.spectral_2d",
                                 "operators.spectral_3d"};
    i.classes = {{"Operators", oper[dims - 1]},     {"State", "state." + name},
                 {"TimeStepping", "time_stepping.exact_lin_rk"},
                 {"InitFields", "init_fields.full"}, {"Forcing", "forcing.random_band"},
                 {"Output", "output.standard"},      {"Preprocess", "preprocess.standard"}};
    for (auto& k : phys) i.keys_state_spect.push_back(k + "_fft");
    i.keys_state_phys = std::move(phys);
    return i;
}

// Maps skgpu status codes onto the reference's exception types (errors.hpp).
void check(int rc) {
    if (rc == SKG_OK) return;
    std::string msg = skg_last_error();
    if (rc == SKG_ECONFIG) throw ConfigError(msg);
    if (rc == SKG_ESHAPE) throw ShapeError(msg);
    throw Error("skgpu: " + msg);
}

class GpuSolver : public Solver {
public:
    GpuSolver(Simulation& sim, const char* base, int nvars) : Solver(sim), base_(base), nvars_(nvars) {}
    ~GpuSolver() override {
        if (ctx_) skg_destroy(ctx_);
    }

    // Solver::tendency (simulation.hpp:34): dealiased nonlinear term of an
    // arbitrary stage state, computed on the GPU.
    void tendency(const StateVec& state, StateVec& out) override {
        const std::size_t S = sim_.oper().spect_size;
        pack(state);
        res_.resize(nvars_ * S);
        check(skg_tendency(ctx_, reinterpret_cast<const double*>(in_.data()),
                           reinterpret_cast<double*>(res_.data())));
        out.resize(nvars_);
        for (int v = 0; v < nvars_; ++v) out[v].assign(res_.begin() + v * S, res_.begin() + (v + 1) * S);
    }

    // Solver::max_velocity_per_axis (solvers.cpp:176-194, 341-357) of the
    // current state, for compute_dt with time_stepping.fixed_dt = 0.
    std::vector<double> max_velocity_per_axis() override {
        pack(sim_.state().spect());
        std::vector<double> m(sim_.oper().dims, 0.0);
        check(skg_max_velocity(ctx_, reinterpret_cast<const double*>(in_.data()), m.data()));
        return m;
    }

protected:
    void pack(const StateVec& state) {
        const auto& g = sim_.oper();
        if (!ctx_) {
            std::vector<double> L(g.L.begin(), g.L.end());
            check(skg_create(&ctx_, base_, g.dims, g.n.data(), L.data(), g.dealias_coef,
                             nu(), SKG_RK4, 0));
        }
        const std::size_t S = g.spect_size;
        if (state.size() != static_cast<std::size_t>(nvars_))
            throw ShapeError("gpu tendency: wrong number of state variables");
        in_.resize(nvars_ * S);
        for (int v = 0; v < nvars_; ++v) {
            if (state[v].size() != S) throw ShapeError("gpu tendency: wrong state shape");
            std::memcpy(in_.data() + v * S, state[v].data(), S * sizeof(cplx));
        }
    }

    const char* base_;
    int nvars_;
    skg_ctx* ctx_ = nullptr;
    std::vector<cplx> in_, res_;
};

class GpuNs2d final : public GpuSolver {
public:
    explicit GpuNs2d(Simulation& sim) : GpuSolver(sim, "ns2d", 1) {}
    const SolverInfo& info() const override { return info_s(); }
    static const SolverInfo& info_s() {
        static const SolverInfo i = gpu_info("ns2d_gpu", 2, {"rot"});
        return i;
    }
    // ns2d energy metric (solvers.cpp:211-218): w |w_hat|^2 / (2 |k|^2)
    void mode_energy(std::vector<double>& e) const override {
        const auto& g = sim_.oper();
        const auto& w = sim_.state().spect()[0];
        e.assign(g.spect_size, 0.0);
        for (std::size_t i = 1; i < g.spect_size; ++i)
            if (g.k_sq[i] > 0.0) e[i] = 0.5 * g.parseval_w[i] * std::norm(w[i]) / g.k_sq[i];
    }
};

class GpuNs3d final : public GpuSolver {
public:
    explicit GpuNs3d(Simulation& sim) : GpuSolver(sim, "ns3d", 3) {}
    const SolverInfo& info() const override { return info_s(); }
    static const SolverInfo& info_s() {
        static const SolverInfo i = gpu_info("ns3d_gpu", 3, {"vx", "vy", "vz"});
        return i;
    }
};

void register_gpu_solvers() {
    ensure_builtin_solvers();
    if (!solver_registered("ns2d_gpu"))
        register_solver({GpuNs2d::info_s(),
                         [](Simulation& s) -> std::unique_ptr<Solver> { return std::make_unique<GpuNs2d>(s); },
                         nullptr});
    if (!solver_registered("ns3d_gpu"))
        register_solver({GpuNs3d::info_s(),
                         [](Simulation& s) -> std::unique_ptr<Solver> { return std::make_unique<GpuNs3d>(s); },
                         nullptr});
}

thread_local std::string g_err;

}  // namespace

extern "C" {

const char* skgi_last_error(void) { return g_err.c_str(); }

// Runs the REFERENCE Simulation (step_once x nsteps, fixed dt or, with
// dt = 0, the CFL dt of compute_dt; files and forcing off) with solver `name` ("ns2d", "ns2d_gpu", "ns3d", "ns3d_gpu")
// from the spectral state `in`; writes the final state to `out`.
int skgi_run(const char* name, int dims, const int* n, double nu, double dt, const double* in,
             long nsteps, double* out) {
    try {
        register_gpu_solvers();
        ParamTree p = create_default_params(name);
        static const char* ns[] = {"nx", "ny", "nz"};
        for (int d = 0; d < dims; ++d)
            p.set(std::string("oper.") + ns[d], static_cast<std::int64_t>(n[d]));
        p.set("nu_2", nu);
        p.set("output.enable_files", false);
        p.set("time_stepping.fixed_dt", dt);
        p.set("time_stepping.t_end", -1.0);
        p.set("time_stepping.n_iters", static_cast<std::int64_t>(nsteps));
        p.set("init_fields.type", std::string("constant"));
        p.set("init_fields.constant.value", 0.0);
        Simulation sim(p);
        sim.set_quiet(true);
        const std::size_t S = sim.oper().spect_size;
        auto& s = sim.state().spect_mut();
        for (std::size_t v = 0; v < s.size(); ++v)
            std::memcpy(s[v].data(), in + 2 * S * v, S * sizeof(cplx));
        for (long i = 0; i < nsteps; ++i) sim.step_once();
        const auto& r = sim.state().spect();
        for (std::size_t v = 0; v < r.size(); ++v)
            std::memcpy(out + 2 * S * v, r[v].data(), S * sizeof(cplx));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

}  // extern "C"
