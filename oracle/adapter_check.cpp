// adapter_check.cpp -- TEST INFRASTRUCTURE ONLY (built into oracle/_ref/ by
// oracle/Makefile where /root/reference is mounted; run by
// tests/test_cpp_adapter.py on the GPU box).
//
// Drives the reference's OWN C++ API twice on identical inputs: once through
// the unmodified reference engine (peridyn::compute_forces / simulate, from
// oracle/_ref/libperidyn_ref.so) and once through the drop-in adapter
// include/pd_b200_peridyn.hpp (peridyn::b200::*, libpd_b200.so on the GPU),
// and requires byte-identical results.  Prints one line per case and exits
// with the number of failures.
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "oracles.hpp" // /root/reference/proj/tests/oracles.hpp
#include "peridyn/engine.hpp"
#include "peridyn/geometry.hpp"

#include "../include/pd_b200_peridyn.hpp"

using namespace peridyn;
using oracles::RandomConfig;
using oracles::make_random_config;

namespace {

int failures = 0;

template <class T> bool same(const std::vector<T>& a, const std::vector<T>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), a.size() * sizeof(T)) == 0);
}

void report(const std::string& name, bool ok) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
    failures += ok ? 0 : 1;
}

bool same_state(const SimulationState& a, const SimulationState& b) {
    return same(a.u, b.u) && same(a.v, b.v) && same(a.a, b.a) && a.step == b.step &&
           same(a.connectivity.entries, b.connectivity.entries) &&
           same(a.connectivity.n_neigh, b.connectivity.n_neigh) &&
           same(a.bond_history, b.bond_history);
}

bool same_vec(const Vec3& a, const Vec3& b) {
    return std::memcmp(&a, &b, sizeof(Vec3)) == 0;
}

bool same_tips(const TipSeries& a, const TipSeries& b) {
    if (a.size() != b.size())
        return false;
    for (const auto& [name, ra] : a) {
        auto it = b.find(name);
        if (it == b.end() || it->second.size() != ra.size())
            return false;
        for (std::size_t k = 0; k < ra.size(); ++k) {
            const TipRecord &x = ra[k], &y = it->second[k];
            if (x.step != y.step || !same_vec(x.mean_u, y.mean_u) || !same_vec(x.mean_v, y.mean_v) ||
                !same_vec(x.mean_a, y.mean_a) || !same_vec(x.body_force_sum, y.body_force_sum) ||
                !same_vec(x.external_force_sum, y.external_force_sum))
                return false;
        }
    }
    return true;
}

void random_configs() {
    for (unsigned seed = 1000; seed < 1050; ++seed)
        for (KernelVariant kv : {KernelVariant::bond_parallel, KernelVariant::node_parallel}) {
            RandomConfig cfg = make_random_config(seed);
            SimulationState ref_state = cfg.state, gpu_state = cfg.state;
            ForceField ref_f, gpu_f;
            peridyn::compute_forces(kv, ref_state, cfg.particles, cfg.model, cfg.corrections, ref_f);
            peridyn::b200::compute_forces(kv, gpu_state, cfg.particles, cfg.model, cfg.corrections,
                                          gpu_f);
            report("compute_forces seed " + std::to_string(seed) +
                       (kv == KernelVariant::bond_parallel ? " bpr" : " node"),
                   same(ref_f.body_force, gpu_f.body_force) && same_state(ref_state, gpu_state));
        }
}

GridDesc bar_grid() {
    GridDesc g;
    g.spacing = 1.0;
    g.counts = {18, 8, 6};
    return g;
}

// A notched, ramp-loaded lattice bar exercising every integrator, BCs, tips,
// the write hook and fracture through simulate().
ModelBundle bar_bundle(const NeighborList& fam_in, NeighborList& fam, bool trilinear) {
    ModelBundle b;
    b.particles.coords = grid_coordinates(bar_grid());
    const Index n = Index(b.particles.coords.size() / 3);
    b.particles.volume.assign(std::size_t(n), 1.0);
    b.particles.density.assign(std::size_t(n), 1.0);
    b.particles.material_tag.assign(std::size_t(n), 0);
    fam = fam_in;
    b.model.laws.push_back(trilinear ? DamageLaw::trilinear(1.0, 2e-3, 4e-3, 8e-3)
                                     : DamageLaw::pmb(1.0, 6e-3));
    b.model.damping = trilinear ? 0.0 : 0.05;
    b.bc = BoundaryConditions::none(n);
    RampProfile quintic;
    quintic.kind = RampProfile::Kind::quintic_smooth;
    quintic.rise_steps = 40;
    quintic.target_scale = 1.0;
    b.bc.ramps.push_back(quintic);
    std::vector<Index> left, right;
    for (Index i = 0; i < n; ++i) {
        const double x = b.particles.coords[std::size_t(3 * i)];
        if (x < 1.5) {
            left.push_back(i);
            for (int ax = 0; ax < 3; ++ax)
                b.bc.kind[std::size_t(3 * i + ax)] = BCKind::displacement;
            b.bc.no_failure[std::size_t(i)] = 1;
        } else if (x > 15.5) {
            right.push_back(i);
            b.bc.kind[std::size_t(3 * i)] = BCKind::displacement;
            b.bc.magnitude[std::size_t(3 * i)] = 0.4;
            b.bc.ramp_id[std::size_t(3 * i)] = 1;
            b.bc.kind[std::size_t(3 * i + 2)] = BCKind::force;
            b.bc.magnitude[std::size_t(3 * i + 2)] = -1e-3;
            b.bc.ramp_id[std::size_t(3 * i + 2)] = 1;
        }
    }
    b.bc.tip_sets["left"] = left;
    b.bc.tip_sets["right"] = right;
    b.dt = 0.05;
    return b;
}

void simulate_runs() {
    const auto coords = grid_coordinates(bar_grid());
    NeighborList family = build_family(coords, 3.0);
    break_initial_bonds(family, coords, notch_predicate(0, 9.0, 1, 4.0));
    for (int trilinear = 0; trilinear < 2; ++trilinear)
        for (IntegratorKind ik :
             {IntegratorKind::velocity_verlet, IntegratorKind::euler, IntegratorKind::euler_cromer}) {
            NeighborList fam;
            const ModelBundle b = bar_bundle(family, fam, trilinear != 0);
            SimulateOptions o;
            o.steps = 120;
            o.write_every = 10;
            o.integrator = ik;
            SimulationState ref_state = make_state_for(b, fam), gpu_state = make_state_for(b, fam);
            int ref_calls = 0, gpu_calls = 0;
            std::vector<double> ref_hook_f, gpu_hook_f;
            const SimulateResult r = peridyn::simulate(
                b, ref_state, o, [&](const SimulationState&, const ForceField& f) {
                    ++ref_calls;
                    ref_hook_f.insert(ref_hook_f.end(), f.body_force.begin(), f.body_force.end());
                });
            const SimulateResult g = peridyn::b200::simulate(
                b, gpu_state, o, [&](const SimulationState&, const ForceField& f) {
                    ++gpu_calls;
                    gpu_hook_f.insert(gpu_hook_f.end(), f.body_force.begin(), f.body_force.end());
                });
            Index broken = 0;
            for (std::size_t i = 0; i < fam.n_neigh.size(); ++i)
                broken += fam.n_neigh[i] - ref_state.connectivity.n_neigh[i];
            report(std::string("simulate ") + (trilinear ? "trilinear " : "pmb ") +
                       (ik == IntegratorKind::velocity_verlet ? "verlet"
                        : ik == IntegratorKind::euler         ? "euler"
                                                              : "euler_cromer") +
                       " broken=" + std::to_string(broken),
                   same_state(ref_state, gpu_state) && same_tips(r.tips, g.tips) &&
                       ref_calls == gpu_calls && same(ref_hook_f, gpu_hook_f));
        }
}

void error_mapping() {
    RandomConfig cfg = make_random_config(1000);
    cfg.state.u[3] = std::numeric_limits<double>::quiet_NaN();
    cfg.state.step = 17;
    std::string ref_msg, gpu_msg;
    ForceField f;
    try {
        SimulationState s = cfg.state;
        peridyn::compute_forces(KernelVariant::bond_parallel, s, cfg.particles, cfg.model,
                                cfg.corrections, f);
    } catch (const std::runtime_error& e) {
        ref_msg = e.what();
    }
    try {
        SimulationState s = cfg.state;
        peridyn::b200::compute_forces(KernelVariant::bond_parallel, s, cfg.particles, cfg.model,
                                      cfg.corrections, f);
    } catch (const std::runtime_error& e) {
        gpu_msg = e.what();
    }
    report("non-finite u -> runtime_error '" + gpu_msg + "'", !ref_msg.empty() && ref_msg == gpu_msg);
    // a corrections array of the wrong size: same exception type and message
    ref_msg.clear();
    gpu_msg.clear();
    RandomConfig good = make_random_config(1001);
    good.corrections.lambda.assign(7, 1.0);
    try {
        SimulationState s = good.state;
        peridyn::compute_forces(KernelVariant::bond_parallel, s, good.particles, good.model,
                                good.corrections, f);
    } catch (const std::invalid_argument& e) {
        ref_msg = e.what();
    }
    try {
        SimulationState s = good.state;
        peridyn::b200::compute_forces(KernelVariant::bond_parallel, s, good.particles, good.model,
                                      good.corrections, f);
    } catch (const std::invalid_argument& e) {
        gpu_msg = e.what();
    }
    const bool ok = !ref_msg.empty() && ref_msg == gpu_msg;
    report("lambda size mismatch -> invalid_argument '" + gpu_msg + "'", ok);
}

// Hand-composed steps (test_engine.cpp:196-357): the reference's stand-alone
// integrators and boundary passes against peridyn::b200's, on random configs
// with a ForceEval that calls each side's compute_forces.
void hand_composed_steps() {
    for (unsigned seed : {1003u, 1011u, 1027u}) {
        RandomConfig cfg = make_random_config(seed);
        const Index n = cfg.state.size();
        SimulationState a = cfg.state, b = cfg.state;
        ForceField fa, fb;
        fa.resize(n);
        fb.resize(n);
        BoundaryConditions bc = BoundaryConditions::none(n);
        bc.ramps.push_back(RampProfile{RampProfile::Kind::quintic_smooth, 30, 1});
        for (Index i = 0; i < n; i += 7) {
            bc.kind[std::size_t(3 * i)] = BCKind::displacement;
            bc.magnitude[std::size_t(3 * i)] = Real(1e-3);
            bc.ramp_id[std::size_t(3 * i)] = 1;
            bc.kind[std::size_t(3 * i + 1)] = BCKind::force;
            bc.magnitude[std::size_t(3 * i + 1)] = Real(0.25);
        }
        const Real dt = Real(1e-3);
        const ForceEval ea = [&](SimulationState& s, ForceField& out) {
            peridyn::compute_forces(KernelVariant::bond_parallel, s, cfg.particles, cfg.model,
                                    cfg.corrections, out);
        };
        const ForceEval eb = [&](SimulationState& s, ForceField& out) {
            peridyn::b200::compute_forces(KernelVariant::bond_parallel, s, cfg.particles,
                                          cfg.model, cfg.corrections, out);
        };
        bool ok = true;
        for (Index k = 0; k < 12 && ok; ++k) {
            std::fill(fa.external_force.begin(), fa.external_force.end(), 0);
            std::fill(fb.external_force.begin(), fb.external_force.end(), 0);
            peridyn::apply_boundary(a, bc, k, dt, fa);
            peridyn::b200::apply_boundary(b, bc, k, dt, fb);
            if (k % 3 == 0) {
                peridyn::step_velocity_verlet(a, ea, fa, dt, Real(0.1), cfg.particles.density);
                peridyn::b200::step_velocity_verlet(b, eb, fb, dt, Real(0.1),
                                                    cfg.particles.density);
            } else {
                ea(a, fa);
                eb(b, fb);
                if (k % 3 == 1) {
                    peridyn::step_euler(a, fa, dt, cfg.particles.density);
                    peridyn::b200::step_euler(b, fb, dt, cfg.particles.density);
                } else {
                    peridyn::step_euler_cromer(a, fa, dt, cfg.particles.density);
                    peridyn::b200::step_euler_cromer(b, fb, dt, cfg.particles.density);
                }
            }
            ok = same_state(a, b) && same(fa.external_force, fb.external_force);
        }
        report("hand-composed steps (apply_boundary, step_velocity_verlet, step_euler, "
               "step_euler_cromer) seed " + std::to_string(seed), ok);
    }
    // errors: dt <= 0 and a density of the wrong size
    std::string ref_msg, gpu_msg;
    RandomConfig cfg = make_random_config(1001);
    try {
        peridyn::verlet_drift(cfg.state, 0);
    } catch (const std::domain_error& e) {
        ref_msg = e.what();
    }
    try {
        peridyn::b200::verlet_drift(cfg.state, 0);
    } catch (const std::domain_error& e) {
        gpu_msg = e.what();
    }
    report("verlet_drift dt <= 0 -> domain_error '" + gpu_msg + "'",
           !ref_msg.empty() && ref_msg == gpu_msg);
}

} // namespace

int main() {
    random_configs();
    simulate_runs();
    error_mapping();
    hand_composed_steps();
    std::printf("failures %d\n", failures);
    return failures;
}
