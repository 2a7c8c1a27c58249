// pd_b200_peridyn.hpp -- C++ host adapter: the reference's own engine API
// (peridyn::compute_forces / peridyn::simulate, /root/reference/proj/include/
// peridyn/engine.hpp) served by the B200 library through the C ABI in
// pd_b200.h.  Header-only; include it from the reference build (it needs the
// reference's peridyn/types.hpp + engine.hpp) and link libpd_b200.so.
//
//   peridyn::b200::compute_forces(KernelVariant, state, particles, model, corr, out)
//       == peridyn::compute_forces (engine.hpp:35-36): same arguments, same
//          in-place mutation of state.connectivity / bond_history, same
//          exception types and messages; bitwise-equal results.
//   peridyn::b200::step_euler / step_euler_cromer / verlet_drift / verlet_kick /
//   step_velocity_verlet / apply_displacement_positions / _kinematics /
//   accumulate_external_force / apply_boundary
//       == the reference's stand-alone integrators and boundary passes
//          (engine.hpp:38-78), same signatures, bitwise-equal results.
//   peridyn::b200::simulate(bundle, state, options, on_write[, fast])
//       == peridyn::simulate (engine.hpp:128-129), the whole loop device-resident;
//          the write hook sees the caller's SimulationState exactly as the
//          reference's hook does (engine.cpp:416-422).
//
// The reference dispatches on KernelVariant (engine.cpp:163-169); a maintainer
// adds a `cuda` value there and forwards to these functions.
#pragma once

#include <cstring>
#include <map>
#include <span>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "pd_b200.h"
#include "peridyn/engine.hpp"
#include "peridyn/types.hpp"

namespace peridyn::b200 {

static_assert(std::is_same_v<Real, double>,
              "the B200 backend consumes the reference's fp64 layout (PERIDYN_SINGLE_PRECISION off)");

namespace detail {

// pd status -> the reference's exception types (engine.cpp:23-49, types.cpp:8-48)
inline void raise(int rc) {
    if (rc == PD_OK)
        return;
    const std::string msg = pd_last_error();
    switch (rc) {
    case PD_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case PD_E_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
    }
}

template <class T> T* data_or_null(std::vector<T>& v) { return v.empty() ? nullptr : v.data(); }
template <class T> const T* data_or_null(const std::vector<T>& v) {
    return v.empty() ? nullptr : v.data();
}

inline pd_particles particles(const ParticleSet& p) {
    pd_particles o{};
    o.n = p.size();
    o.coords = data_or_null(p.coords);
    o.coords_size = Index(p.coords.size());
    o.volume = data_or_null(p.volume);
    o.density = data_or_null(p.density);
    o.density_size = Index(p.density.size());
    return o;
}

inline pd_neighbor_list family(NeighborList& f) {
    pd_neighbor_list o{};
    o.n = f.node_count();
    o.group_size = f.group_size;
    o.entries = data_or_null(f.entries);
    o.n_neigh = data_or_null(f.n_neigh);
    o.initial_n_neigh = data_or_null(f.initial_n_neigh);
    o.bond_type = data_or_null(f.bond_type);
    o.bond_type_size = Index(f.bond_type.size());
    o.horizon = f.horizon;
    return o;
}

struct Laws {
    std::vector<pd_law> laws;
    pd_damage_model model{};
    explicit Laws(const DamageModel& m) {
        for (const DamageLaw& l : m.laws) {
            if (l.breakpoints.size() > PD_MAX_BREAKPOINTS || l.forces.size() != l.breakpoints.size())
                l.validate();  // the reference's own message for malformed laws
            if (l.breakpoints.size() > PD_MAX_BREAKPOINTS)
                throw std::invalid_argument("DamageLaw: more than 8 breakpoints is not supported");
            pd_law d{};
            d.stiffness = l.stiffness;
            d.n_breakpoints = int32_t(l.breakpoints.size());
            for (std::size_t k = 0; k < l.breakpoints.size(); ++k) {
                d.breakpoints[k] = l.breakpoints[k];
                d.forces[k] = l.forces[k];
            }
            laws.push_back(d);
        }
        model.laws = laws.empty() ? nullptr : laws.data();
        model.n_laws = int32_t(laws.size());
        model.damping = m.damping;
    }
};

inline pd_corrections corrections(const Corrections& c) {
    pd_corrections o{};
    o.lambda = data_or_null(c.lambda);
    o.lambda_size = Index(c.lambda.size());
    o.beta = data_or_null(c.beta);
    o.beta_size = Index(c.beta.size());
    o.no_failure = data_or_null(c.no_failure);
    o.no_failure_size = Index(c.no_failure.size());
    return o;
}

inline pd_state state(SimulationState& s) {
    pd_state o{};
    o.u = data_or_null(s.u);
    o.v = data_or_null(s.v);
    o.a = data_or_null(s.a);
    o.step = s.step;
    o.connectivity = family(s.connectivity);
    o.bond_history = data_or_null(s.bond_history);
    o.bond_history_size = Index(s.bond_history.size());
    return o;
}

struct Boundary {
    std::vector<pd_ramp> ramps;
    std::vector<int64_t> offsets, nodes;
    std::vector<std::string> names;  // std::map order, as TipSeries
    pd_boundary bc{};
    explicit Boundary(const BoundaryConditions& b) {
        for (const RampProfile& r : b.ramps)
            ramps.push_back(pd_ramp{int32_t(r.kind), r.rise_steps, r.target_scale});
        offsets.push_back(0);
        for (const auto& [name, set] : b.tip_sets) {
            names.push_back(name);
            nodes.insert(nodes.end(), set.begin(), set.end());
            offsets.push_back(int64_t(nodes.size()));
        }
        static_assert(sizeof(BCKind) == 1);
        bc.kind = reinterpret_cast<const uint8_t*>(data_or_null(b.kind));
        bc.kind_size = Index(b.kind.size());
        bc.magnitude = data_or_null(b.magnitude);
        bc.magnitude_size = Index(b.magnitude.size());
        bc.ramp_id = data_or_null(b.ramp_id);
        bc.ramp_id_size = Index(b.ramp_id.size());
        bc.ramps = ramps.empty() ? nullptr : ramps.data();
        bc.n_ramps = int32_t(ramps.size());
        bc.no_failure = data_or_null(b.no_failure);
        bc.no_failure_size = Index(b.no_failure.size());
        bc.n_tip_sets = int32_t(names.size());
        bc.tip_offsets = offsets.data();
        bc.tip_nodes = nodes.empty() ? nullptr : nodes.data();
    }
};

struct HookCtx {
    const WriteHook* hook;
    SimulationState* state;
    std::exception_ptr error;
};

// pd_write_hook trampoline: the library has already written u, v, a,
// connectivity and history of the write step into the caller's arrays
// (pd_simulate's one-shot mode), so the reference hook sees `state` itself.
inline int hook_trampoline(void* user, const pd_state* view, const pd_force_field* ff) {
    auto* h = static_cast<HookCtx*>(user);
    try {
        h->state->step = view->step;
        ForceField forces;
        const std::size_t n3 = std::size_t(3 * h->state->size());
        forces.body_force.assign(ff->body_force, ff->body_force + n3);
        forces.external_force.assign(ff->external_force, ff->external_force + n3);
        (*h->hook)(*h->state, forces);
        return 0;
    } catch (...) {
        h->error = std::current_exception();
        return 1;
    }
}

} // namespace detail

/// compute_forces (engine.hpp:35-36) on the B200.  `fast` selects the
/// tolerance-bound fp32-bond-math path instead of the
/// bitwise variant named by `variant`.
inline void compute_forces(KernelVariant variant, SimulationState& state,
                           const ParticleSet& particles, const DamageModel& model,
                           const Corrections& corrections, ForceField& out, bool fast = false) {
    const Index n = state.size();
    // memory safety of the flat views handed to the C ABI (the reference
    // indexes these without a check)
    if (Index(state.u.size()) != 3 * n)
        throw std::invalid_argument("compute_forces: displacement array does not match node count");
    if (Index(out.body_force.size()) != 3 * n)
        out.body_force.assign(std::size_t(3 * n), 0);
    if (Index(out.external_force.size()) != 3 * n)
        out.external_force.assign(std::size_t(3 * n), 0);  // engine.cpp:116-118
    detail::Laws laws(model);
    pd_state st = detail::state(state);
    pd_particles p = detail::particles(particles);
    pd_corrections c = detail::corrections(corrections);
    pd_force_field ff{out.body_force.data(), out.external_force.data()};
    const int32_t v = fast ? PD_FAST
                           : (variant == KernelVariant::node_parallel ? PD_NODE_PARALLEL
                                                                      : PD_BOND_PARALLEL);
    detail::raise(pd_compute_forces(v, &st, &p, &laws.model, &c, &ff));
}

/// simulate (engine.hpp:128-129) with the whole loop on the B200.
inline SimulateResult simulate(const ModelBundle& bundle, SimulationState& state,
                               const SimulateOptions& options, const WriteHook& on_write = {},
                               bool fast = false) {
    if (options.steps < 1)
        throw std::invalid_argument("simulate: steps must be >= 1");
    if (bundle.model.needs_history() &&
        state.bond_history.size() != state.connectivity.entries.size())
        state.bond_history.assign(state.connectivity.entries.size(), 0);  // engine.cpp:382-384
    const Index n = state.size();
    if (Index(state.u.size()) != 3 * n || Index(state.v.size()) != 3 * n ||
        Index(state.a.size()) != 3 * n)
        throw std::invalid_argument("simulate: state fields do not match node count");
    detail::Laws laws(bundle.model);
    detail::Boundary bc(bundle.bc);
    pd_bundle b{};
    b.particles = detail::particles(bundle.particles);
    b.model = laws.model;
    b.corrections = detail::corrections(bundle.corrections);
    b.bc = bc.bc;
    b.dt = bundle.dt;
    pd_options o{};
    o.steps = options.steps;
    o.write_every = options.write_every;
    o.first_step = options.first_step;
    o.integrator = int32_t(options.integrator);
    o.variant = fast ? PD_FAST
                     : (options.variant == KernelVariant::node_parallel ? PD_NODE_PARALLEL
                                                                        : PD_BOND_PARALLEL);
    int64_t writes = 0;
    if (options.write_every > 0)
        for (Index s = options.first_step; s < options.first_step + options.steps; ++s)
            writes += (s + 1) % options.write_every == 0;
    std::vector<pd_tip_record> recs(std::size_t(std::max<int64_t>(1, writes * b.bc.n_tip_sets)));
    int64_t n_recs = 0;
    pd_state st = detail::state(state);
    detail::HookCtx hctx{&on_write, &state, nullptr};
    const int rc = pd_simulate(&b, &st, &o, on_write ? detail::hook_trampoline : nullptr, &hctx,
                               recs.data(), int64_t(recs.size()), &n_recs);
    state.step = st.step;
    if (hctx.error)
        std::rethrow_exception(hctx.error);
    detail::raise(rc);
    SimulateResult result;
    const std::size_t sets = bc.names.size();
    for (int64_t r = 0; r < n_recs; ++r) {
        const pd_tip_record& t = recs[std::size_t(r)];
        TipRecord rec;
        rec.step = t.step;
        rec.mean_u = {t.mean_u[0], t.mean_u[1], t.mean_u[2]};
        rec.mean_v = {t.mean_v[0], t.mean_v[1], t.mean_v[2]};
        rec.mean_a = {t.mean_a[0], t.mean_a[1], t.mean_a[2]};
        rec.body_force_sum = {t.body_force_sum[0], t.body_force_sum[1], t.body_force_sum[2]};
        rec.external_force_sum = {t.external_force_sum[0], t.external_force_sum[1],
                                  t.external_force_sum[2]};
        result.tips[bc.names[std::size_t(r) % sets]].push_back(rec);
    }
    return result;
}

// ---- stand-alone integrators and boundary passes (engine.hpp:38-78) -------

namespace detail {
inline void check_sizes(const SimulationState& s, const char* who) {
    const Index n = s.size();
    if (Index(s.u.size()) != 3 * n || Index(s.v.size()) != 3 * n || Index(s.a.size()) != 3 * n)
        throw std::invalid_argument(std::string(who) + ": state fields do not match node count");
}
inline pd_force_field forces(const ForceField& f) {
    return pd_force_field{const_cast<double*>(f.body_force.data()),
                          const_cast<double*>(f.external_force.data())};
}
} // namespace detail

inline void step_euler(SimulationState& state, const ForceField& forces, Real dt,
                       std::span<const Real> density) {
    detail::check_sizes(state, "step_euler");
    pd_state st = detail::state(state);
    pd_force_field ff = detail::forces(forces);
    detail::raise(pd_step_euler(&st, &ff, dt, density.data(), Index(density.size())));
}

inline void step_euler_cromer(SimulationState& state, const ForceField& forces, Real dt,
                              std::span<const Real> density) {
    detail::check_sizes(state, "step_euler_cromer");
    pd_state st = detail::state(state);
    pd_force_field ff = detail::forces(forces);
    detail::raise(pd_step_euler_cromer(&st, &ff, dt, density.data(), Index(density.size())));
}

inline void verlet_drift(SimulationState& state, Real dt) {
    detail::check_sizes(state, "verlet_drift");
    pd_state st = detail::state(state);
    detail::raise(pd_verlet_drift(&st, dt));
}

inline void verlet_kick(SimulationState& state, const ForceField& forces, Real dt, Real damping,
                        std::span<const Real> density) {
    detail::check_sizes(state, "verlet_kick");
    pd_state st = detail::state(state);
    pd_force_field ff = detail::forces(forces);
    detail::raise(pd_verlet_kick(&st, &ff, dt, damping, density.data(), Index(density.size())));
}

inline void step_velocity_verlet(SimulationState& state, const ForceEval& forces,
                                 ForceField& scratch, Real dt, Real damping,
                                 std::span<const Real> density) {
    b200::verlet_drift(state, dt);  // qualified: ADL also finds peridyn::verlet_drift
    forces(state, scratch);
    b200::verlet_kick(state, scratch, dt, damping, density);
    state.step += 1;
}

inline void apply_displacement_positions(SimulationState& state, const BoundaryConditions& bc,
                                         Index step) {
    detail::Boundary b(bc);
    pd_state st = detail::state(state);
    detail::raise(pd_apply_displacement_positions(&st, &b.bc, step));
}

inline void apply_displacement_kinematics(SimulationState& state, const BoundaryConditions& bc,
                                          Index step, Real dt) {
    detail::Boundary b(bc);
    pd_state st = detail::state(state);
    detail::raise(pd_apply_displacement_kinematics(&st, &b.bc, step, dt));
}

inline void accumulate_external_force(const BoundaryConditions& bc, Index step, ForceField& out) {
    detail::Boundary b(bc);
    pd_force_field ff{out.body_force.data(), out.external_force.data()};
    detail::raise(pd_accumulate_external_force(&b.bc, step, &ff,
                                               Index(out.external_force.size()) / 3));
}

inline void apply_boundary(SimulationState& state, const BoundaryConditions& bc, Index step,
                           Real dt, ForceField& out) {
    detail::Boundary b(bc);
    pd_state st = detail::state(state);
    pd_force_field ff{out.body_force.data(), out.external_force.data()};
    detail::raise(pd_apply_boundary(&st, &b.bc, step, dt, &ff));
}

} // namespace peridyn::b200
