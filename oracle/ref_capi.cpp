// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI over the *unmodified* reference library, compiled from the sources
// under /root/reference/proj/src by oracle/Makefile into oracle/_ref/.  It is
// the reference-side binding a maintainer would add: it takes
// the same pd_* descriptors as include/pd_b200.h, copies them into the
// reference's value types, calls the reference entry point and copies the
// results back.  Used to generate tests/golden/ and as bench.py's
// `--impl reference` arm.  Never linked into the product.
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "oracles.hpp" // /root/reference/proj/tests/oracles.hpp (make_random_config)
#include "peridyn/engine.hpp"
#include "peridyn/formulas.hpp"
#include "peridyn/geometry.hpp"
#include "peridyn/io.hpp"
#include "peridyn/parallel.hpp"

#include "../include/pd_b200.h"

using namespace peridyn;

namespace {

thread_local std::string g_err;

int map_exceptions(const std::function<void()>& fn) {
    try {
        fn();
        g_err.clear();
        return PD_OK;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return PD_E_INVALID_ARGUMENT;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return PD_E_DOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return PD_E_RUNTIME;
    }
}

template <class T> std::vector<T> vec(const T* p, int64_t n) {
    return p && n > 0 ? std::vector<T>(p, p + n) : std::vector<T>{};
}

ParticleSet to_particles(const pd_particles& p) {
    ParticleSet out;
    out.coords = vec(p.coords, p.coords_size);
    out.volume = vec(p.volume, p.n);
    out.density = vec(p.density, p.density_size);
    out.material_tag.assign(std::size_t(p.n), 0);
    return out;
}

NeighborList to_family(const pd_neighbor_list& f) {
    NeighborList out;
    out.group_size = f.group_size;
    out.horizon = f.horizon;
    out.entries = vec(f.entries, f.n * f.group_size);
    out.n_neigh = vec(f.n_neigh, f.n);
    out.initial_n_neigh = vec(f.initial_n_neigh, f.n);
    out.bond_type = vec(f.bond_type, f.bond_type_size);
    return out;
}

DamageModel to_model(const pd_damage_model& m) {
    DamageModel out;
    for (int k = 0; k < m.n_laws; ++k) {
        const pd_law& l = m.laws[k];
        DamageLaw law;
        law.stiffness = l.stiffness;
        law.breakpoints.assign(l.breakpoints, l.breakpoints + l.n_breakpoints);
        law.forces.assign(l.forces, l.forces + l.n_breakpoints);
        out.laws.push_back(law);
    }
    out.damping = m.damping;
    return out;
}

Corrections to_corr(const pd_corrections& c) {
    Corrections out;
    out.lambda = vec(c.lambda, c.lambda_size);
    out.beta = vec(c.beta, c.beta_size);
    out.no_failure = vec(c.no_failure, c.no_failure_size);
    return out;
}

SimulationState to_state(const pd_state& s) {
    SimulationState out;
    out.connectivity = to_family(s.connectivity);
    const int64_t n = s.connectivity.n;
    out.u = vec(s.u, 3 * n);
    out.v = vec(s.v, 3 * n);
    out.a = vec(s.a, 3 * n);
    out.step = s.step;
    out.bond_history = vec(s.bond_history, s.bond_history_size);
    return out;
}

void from_state(const SimulationState& st, pd_state& s) {
    const int64_t n = s.connectivity.n;
    std::memcpy(s.u, st.u.data(), sizeof(double) * 3 * n);
    std::memcpy(s.v, st.v.data(), sizeof(double) * 3 * n);
    std::memcpy(s.a, st.a.data(), sizeof(double) * 3 * n);
    s.step = st.step;
    std::memcpy(s.connectivity.entries, st.connectivity.entries.data(),
                sizeof(int32_t) * st.connectivity.entries.size());
    std::memcpy(s.connectivity.n_neigh, st.connectivity.n_neigh.data(),
                sizeof(int32_t) * st.connectivity.n_neigh.size());
    if (s.bond_history && !st.bond_history.empty())
        std::memcpy(s.bond_history, st.bond_history.data(),
                    sizeof(double) * std::min<std::size_t>(st.bond_history.size(),
                                                           std::size_t(s.bond_history_size)));
}

BoundaryConditions to_bc(const pd_boundary& b) {
    BoundaryConditions out;
    out.kind.resize(std::size_t(b.kind_size));
    for (int64_t k = 0; k < b.kind_size; ++k)
        out.kind[std::size_t(k)] = BCKind(b.kind[k]);
    out.magnitude = vec(b.magnitude, b.magnitude_size);
    out.ramp_id = vec(b.ramp_id, b.ramp_id_size);
    for (int k = 0; k < b.n_ramps; ++k) {
        RampProfile r;
        r.kind = RampProfile::Kind(b.ramps[k].kind);
        r.rise_steps = b.ramps[k].rise_steps;
        r.target_scale = b.ramps[k].target_scale;
        out.ramps.push_back(r);
    }
    out.no_failure = vec(b.no_failure, b.no_failure_size);
    // std::map orders by name; zero-padded names keep the caller's set order
    for (int s = 0; s < b.n_tip_sets; ++s) {
        char name[32];
        std::snprintf(name, sizeof name, "set%06d", s);
        out.tip_sets[name] = vec(b.tip_nodes + b.tip_offsets[s], b.tip_offsets[s + 1] - b.tip_offsets[s]);
    }
    return out;
}

struct RandomHandle {
    oracles::RandomConfig cfg;
};

} // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// io::save_state / io::save_cache / load_state of the reference (golden files)
int ref_save_state(const pd_state* st, const char* path) {
    return map_exceptions([&] { io::save_state(to_state(*st), path); });
}

int ref_save_cache(const pd_neighbor_list* fam, const pd_corrections* corr, const char* path) {
    return map_exceptions([&] { io::save_cache(to_family(*fam), to_corr(*corr), path); });
}

int ref_write_snapshot(const pd_state* st, const pd_particles* p, const char* path) {
    return map_exceptions(
        [&] { io::write_snapshot(path, io::make_snapshot(to_state(*st), to_particles(*p))); });
}

int ref_load_state_step(const char* path, int64_t* step) {
    return map_exceptions([&] { *step = io::load_state(path).step; });
}
void ref_set_threads(int threads) { set_worker_cap(unsigned(threads < 0 ? 0 : threads)); }
unsigned ref_worker_count(void) { return worker_count(); }

int ref_reduce_group(double* c, int64_t n, double out[3]) {
    return map_exceptions([&] {
        std::vector<Vec3> v(static_cast<std::size_t>(n));
        for (int64_t k = 0; k < n; ++k)
            v[std::size_t(k)] = {c[3 * k], c[3 * k + 1], c[3 * k + 2]};
        const Vec3 r = reduce_group(v);
        out[0] = r.x;
        out[1] = r.y;
        out[2] = r.z;
    });
}

int ref_compute_forces(int32_t variant, pd_state* state, const pd_particles* particles,
                       const pd_damage_model* model, const pd_corrections* corr,
                       pd_force_field* out) {
    return map_exceptions([&] {
        SimulationState st = to_state(*state);
        ForceField f;
        const int64_t n = state->connectivity.n;
        f.body_force.assign(std::size_t(3 * n), 0);
        f.external_force = vec(out->external_force, 3 * n);
        compute_forces(variant == PD_NODE_PARALLEL ? KernelVariant::node_parallel
                                                   : KernelVariant::bond_parallel,
                       st, to_particles(*particles), to_model(*model), to_corr(*corr), f);
        from_state(st, *state);
        std::memcpy(out->body_force, f.body_force.data(), sizeof(double) * 3 * n);
    });
}

int ref_step(int32_t which, pd_state* state, const pd_force_field* f, double dt, double damping,
             const double* density, int64_t density_size) {
    return map_exceptions([&] {
        SimulationState st = to_state(*state);
        const int64_t n = state->connectivity.n;
        ForceField ff;
        ff.body_force = vec(f->body_force, 3 * n);
        ff.external_force = vec(f->external_force, 3 * n);
        const std::vector<Real> rho = vec(density, density_size);
        if (which == 0)
            verlet_drift(st, dt);
        else if (which == 1)
            verlet_kick(st, ff, dt, damping, rho);
        else if (which == 2)
            step_euler(st, ff, dt, rho);
        else
            step_euler_cromer(st, ff, dt, rho);
        from_state(st, *state);
    });
}

double ref_ramp(int32_t which, const pd_ramp* r, int64_t step) {
    RampProfile p;
    p.kind = RampProfile::Kind(r->kind);
    p.rise_steps = r->rise_steps;
    p.target_scale = r->target_scale;
    return which == 0 ? p.scale(step) : which == 1 ? p.rate(step) : p.accel(step);
}

struct HookBridge {
    pd_write_hook hook;
    void* user;
    int64_t n;
};

int ref_simulate(const pd_bundle* b, pd_state* state, const pd_options* opt, pd_write_hook on_write,
                 void* user, pd_tip_record* tips_out, int64_t tips_capacity, int64_t* n_tips_out) {
    if (n_tips_out)
        *n_tips_out = 0;
    return map_exceptions([&] {
        ModelBundle bundle;
        bundle.particles = to_particles(b->particles);
        bundle.model = to_model(b->model);
        bundle.corrections = to_corr(b->corrections);
        bundle.bc = to_bc(b->bc);
        bundle.dt = b->dt;
        SimulationState st = to_state(*state);
        SimulateOptions o;
        o.steps = opt->steps;
        o.write_every = opt->write_every;
        o.first_step = opt->first_step;
        o.integrator = IntegratorKind(opt->integrator);
        o.variant = opt->variant == PD_NODE_PARALLEL ? KernelVariant::node_parallel
                                                      : KernelVariant::bond_parallel;
        WriteHook hook;
        if (on_write)
            hook = [&](const SimulationState& s, const ForceField& f) {
                // host views of the reference's own vectors
                pd_state view = *state;
                view.u = const_cast<double*>(s.u.data());
                view.v = const_cast<double*>(s.v.data());
                view.a = const_cast<double*>(s.a.data());
                view.step = s.step;
                view.connectivity.entries = const_cast<int32_t*>(s.connectivity.entries.data());
                view.connectivity.n_neigh = const_cast<int32_t*>(s.connectivity.n_neigh.data());
                view.bond_history = const_cast<double*>(s.bond_history.data());
                view.bond_history_size = int64_t(s.bond_history.size());
                pd_force_field ff{const_cast<double*>(f.body_force.data()),
                                  const_cast<double*>(f.external_force.data())};
                if (on_write(user, &view, &ff) != 0)
                    throw std::runtime_error("simulate: write hook failed");
            };
        SimulateResult res;
        try {
            res = simulate(bundle, st, o, hook);
        } catch (...) {
            from_state(st, *state);
            throw;
        }
        from_state(st, *state);
        int64_t k = 0;
        const auto& tips = res.tips;
        if (!tips.empty()) {
            const std::size_t writes = tips.begin()->second.size();
            if (int64_t(writes * tips.size()) > tips_capacity)
                throw std::invalid_argument("simulate: tips_out capacity too small");
            for (std::size_t w = 0; w < writes; ++w)
                for (const auto& [name, series] : tips) {
                    const TipRecord& r = series[w];
                    pd_tip_record& o2 = tips_out[k++];
                    o2.step = r.step;
                    for (int ax = 0; ax < 3; ++ax) {
                        o2.mean_u[ax] = r.mean_u[ax];
                        o2.mean_v[ax] = r.mean_v[ax];
                        o2.mean_a[ax] = r.mean_a[ax];
                        o2.body_force_sum[ax] = r.body_force_sum[ax];
                        o2.external_force_sum[ax] = r.external_force_sum[ax];
                    }
                }
        }
        if (n_tips_out)
            *n_tips_out = k;
    });
}

int ref_grid_coordinates(const double origin[3], double spacing, const int64_t counts[3],
                         double* out) {
    return map_exceptions([&] {
        GridDesc g;
        g.origin = {origin[0], origin[1], origin[2]};
        g.spacing = spacing;
        g.counts = {counts[0], counts[1], counts[2]};
        const auto c = grid_coordinates(g);
        std::memcpy(out, c.data(), c.size() * sizeof(double));
    });
}

// build_family; grid_hint = {ox, oy, oz, spacing, nx, ny, nz} or NULL.
int ref_build_family(const double* coords, int64_t n, double horizon, const double* grid_hint,
                     int32_t** entries_out, int32_t** n_neigh_out, int32_t** initial_out,
                     int64_t* group_size_out) {
    return map_exceptions([&] {
        GridDesc g;
        const GridDesc* hint = nullptr;
        if (grid_hint) {
            g.origin = {grid_hint[0], grid_hint[1], grid_hint[2]};
            g.spacing = grid_hint[3];
            g.counts = {Index(grid_hint[4]), Index(grid_hint[5]), Index(grid_hint[6])};
            hint = &g;
        }
        const NeighborList f =
            build_family(std::span<const Real>(coords, std::size_t(3 * n)), horizon, hint);
        *group_size_out = f.group_size;
        *entries_out = static_cast<int32_t*>(std::malloc(f.entries.size() * sizeof(int32_t)));
        *n_neigh_out = static_cast<int32_t*>(std::malloc(f.n_neigh.size() * sizeof(int32_t)));
        *initial_out = static_cast<int32_t*>(std::malloc(f.n_neigh.size() * sizeof(int32_t)));
        std::memcpy(*entries_out, f.entries.data(), f.entries.size() * sizeof(int32_t));
        std::memcpy(*n_neigh_out, f.n_neigh.data(), f.n_neigh.size() * sizeof(int32_t));
        std::memcpy(*initial_out, f.initial_n_neigh.data(), f.n_neigh.size() * sizeof(int32_t));
    });
}

void ref_free(void* p) { std::free(p); }

// build_family with a BondClassifier (geometry.hpp:45-54) that applies the
// same region rules as pd_classifier: class = last matching region (else the
// default), type = table[class_a][class_b].  The reference calls it per slot
// from pack_rows; the bond types come back n x N.
int ref_build_family_classified(const double* coords, int64_t n, double horizon,
                                const double* grid_hint, const pd_classifier* cls,
                                int32_t** entries_out, uint8_t** types_out,
                                int64_t* group_size_out) {
    return map_exceptions([&] {
        GridDesc g;
        const GridDesc* hint = nullptr;
        if (grid_hint) {
            g.origin = {grid_hint[0], grid_hint[1], grid_hint[2]};
            g.spacing = grid_hint[3];
            g.counts = {Index(grid_hint[4]), Index(grid_hint[5]), Index(grid_hint[6])};
            hint = &g;
        }
        auto in_region = [](const pd_region& r, const Vec3& x) {
            const Real p[3] = {x.x, x.y, x.z};
            if (r.kind == PD_REGION_BOX) {
                for (int d = 0; d < 3; ++d)
                    if (!(p[d] >= r.lo[d] && p[d] <= r.hi[d]))
                        return false;
                return true;
            }
            const int a = r.axis, b0 = a == 0 ? 1 : 0, b1 = a == 2 ? 1 : 2;
            if (!(p[a] >= r.lo[a] && p[a] <= r.hi[a]))
                return false;
            const Real d0 = p[b0] - r.c[0], d1 = p[b1] - r.c[1];
            return d0 * d0 + d1 * d1 <= r.radius * r.radius;
        };
        auto class_of = [&](const Vec3& x) {
            int c = cls->default_class;
            for (int k = 0; k < cls->n_regions; ++k)
                if (in_region(cls->regions[k], x))
                    c = cls->regions[k].cls;
            return c;
        };
        const BondClassifier classify = [&](const Vec3& a, const Vec3& b) {
            return std::uint8_t(cls->type_table[class_of(a) * cls->n_classes + class_of(b)]);
        };
        const NeighborList f = build_family(std::span<const Real>(coords, std::size_t(3 * n)),
                                            horizon, hint, classify);
        *group_size_out = f.group_size;
        *entries_out = static_cast<int32_t*>(std::malloc(f.entries.size() * sizeof(int32_t)));
        *types_out = static_cast<uint8_t*>(std::malloc(f.bond_type.size()));
        std::memcpy(*entries_out, f.entries.data(), f.entries.size() * sizeof(int32_t));
        std::memcpy(*types_out, f.bond_type.data(), f.bond_type.size());
    });
}

int ref_neighborhood_volumes(const double* volumes, const pd_neighbor_list* family, double* out) {
    return map_exceptions([&] {
        const auto v = neighborhood_volumes(std::span<const Real>(volumes, std::size_t(family->n)),
                                            to_family(*family));
        std::memcpy(out, v.data(), v.size() * sizeof(double));
    });
}

void ref_break_bonds(pd_neighbor_list* family, const double* coords, int kind, int axis,
                     double position, int sweep_axis, double depth) {
    NeighborList f = to_family(*family);
    const std::span<const Real> c(coords, std::size_t(3 * family->n));
    break_initial_bonds(f, c,
                        kind == 0 ? plane_crossing_predicate(axis, position)
                                  : notch_predicate(axis, position, sweep_axis, depth));
    std::memcpy(family->entries, f.entries.data(), f.entries.size() * sizeof(int32_t));
    std::memcpy(family->n_neigh, f.n_neigh.data(), f.n_neigh.size() * sizeof(int32_t));
}

int ref_damage(const pd_neighbor_list* family, const double* coords, double* phi) {
    return map_exceptions([&] {
        SimulationState st;
        st.connectivity = to_family(*family);
        ParticleSet p;
        p.coords = vec(coords, 3 * family->n);
        const io::Snapshot snap = io::make_snapshot(st, p);
        std::memcpy(phi, snap.damage.data(), snap.damage.size() * sizeof(double));
    });
}

int ref_surface_correction_factors(const double* volumes, const pd_neighbor_list* family,
                                   double v0, double* lambda) {
    return map_exceptions([&] {
        const auto l = surface_correction_factors(
            std::span<const Real>(volumes, std::size_t(family->n)), to_family(*family), v0);
        std::memcpy(lambda, l.data(), l.size() * sizeof(double));
    });
}

int ref_stable_timestep_hint(const pd_particles* p, const pd_damage_model* model,
                             const pd_neighbor_list* family, double safety, const double* beta,
                             double* dt_out) {
    return map_exceptions([&] {
        const int64_t slots = family->n * family->group_size;
        *dt_out = stable_timestep_hint(to_particles(*p), to_model(*model), to_family(*family),
                                       safety,
                                       beta ? std::span<const Real>(beta, std::size_t(slots))
                                            : std::span<const Real>{});
    });
}

// ---- oracles::make_random_config (tests/oracles.hpp:140-210) -------------

void* ref_random_config(unsigned seed) {
    auto* h = new RandomHandle{oracles::make_random_config(seed)};
    return h;
}

void ref_random_free(void* h) { delete static_cast<RandomHandle*>(h); }

// field names: coords volume density entries n_neigh initial_n_neigh lambda beta u bond_history
int ref_random_field(void* h, const char* field, void** ptr, int64_t* count) {
    auto& c = static_cast<RandomHandle*>(h)->cfg;
    const std::string f(field);
    auto put = [&](auto& v) {
        *ptr = v.data();
        *count = int64_t(v.size());
    };
    if (f == "coords")
        put(c.particles.coords);
    else if (f == "volume")
        put(c.particles.volume);
    else if (f == "density")
        put(c.particles.density);
    else if (f == "entries")
        put(c.state.connectivity.entries);
    else if (f == "n_neigh")
        put(c.state.connectivity.n_neigh);
    else if (f == "initial_n_neigh")
        put(c.state.connectivity.initial_n_neigh);
    else if (f == "lambda")
        put(c.corrections.lambda);
    else if (f == "beta")
        put(c.corrections.beta);
    else if (f == "u")
        put(c.state.u);
    else if (f == "bond_history")
        put(c.state.bond_history);
    else
        return 1;
    return 0;
}

int64_t ref_random_group_size(void* h) {
    return static_cast<RandomHandle*>(h)->cfg.state.connectivity.group_size;
}

double ref_random_horizon(void* h) { return static_cast<RandomHandle*>(h)->cfg.family.horizon; }

void ref_random_law(void* h, pd_law* out) {
    const DamageLaw& l = static_cast<RandomHandle*>(h)->cfg.model.laws[0];
    std::memset(out, 0, sizeof *out);
    out->stiffness = l.stiffness;
    out->n_breakpoints = int32_t(l.breakpoints.size());
    for (std::size_t k = 0; k < l.breakpoints.size(); ++k) {
        out->breakpoints[k] = l.breakpoints[k];
        out->forces[k] = l.forces[k];
    }
}

// ---- CPU baseline: bench::benchmark_bundle (bench.cpp:76-104) + simulate ---

// Builds the reference bench lattice (spacing 1, V = rho = 1, PMB c = 1,
// s_c, dt = 1e-3, seeded u) with the reference's own build_family, then times
// `steps` velocity-Verlet steps of simulate() (bond_parallel) with
// std::chrono, exactly like bench::time_run (bench.cpp:106-117).
int ref_bench_lattice(const int64_t dims[3], double horizon, double s_c, int64_t steps,
                      int threads, double* seconds_out, int64_t* live_bonds_out,
                      double* build_seconds_out) {
    return map_exceptions([&] {
        set_worker_cap(unsigned(threads));
        GridDesc grid;
        grid.spacing = 1;
        grid.counts = {dims[0], dims[1], dims[2]};
        ModelBundle bundle;
        bundle.particles.coords = grid_coordinates(grid);
        const Index n = grid.node_count();
        bundle.particles.volume.assign(std::size_t(n), 1);
        bundle.particles.density.assign(std::size_t(n), 1);
        bundle.particles.material_tag.assign(std::size_t(n), 0);
        bundle.model.laws.push_back(DamageLaw::pmb(1, s_c));
        bundle.bc = BoundaryConditions::none(n);
        bundle.dt = Real(1e-3);
        const auto b0 = std::chrono::steady_clock::now();
        NeighborList family = build_family(bundle.particles.coords, horizon, &grid);
        const auto b1 = std::chrono::steady_clock::now();
        *build_seconds_out = std::chrono::duration<double>(b1 - b0).count();
        SimulationState state = make_state_for(bundle, family);
        for (Index i = 0; i < n; ++i) {
            const Vec3 x = load_vec3(bundle.particles.coords, i);
            store_vec3(state.u, i,
                       {Real(1e-4) * std::sin(Real(0.1) * x.x + Real(0.2) * x.y),
                        Real(1e-4) * std::cos(Real(0.15) * x.y + Real(0.1) * x.z),
                        Real(1e-4) * std::sin(Real(0.12) * x.z + Real(0.17) * x.x)});
        }
        int64_t live = 0;
        for (auto c : state.connectivity.n_neigh)
            live += c;
        *live_bonds_out = live;
        SimulateOptions opts;
        opts.steps = steps;
        opts.variant = KernelVariant::bond_parallel;
        const auto t0 = std::chrono::steady_clock::now();
        simulate(bundle, state, opts);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds_out = std::chrono::duration<double>(t1 - t0).count();
        set_worker_cap(0);
    });
}

// The bench fixture (bench.cpp:76-104) built once, then `n_runs` consecutive
// simulate(bond_parallel, velocity-Verlet) calls continuing the same state:
// run r takes run_steps[r] steps on threads[r] workers (set_worker_cap; 0 =
// all) and its wall time goes to seconds_out[r] (bench.cpp:106-117 time_run,
// family build excluded).
int ref_bench_lattice_runs(const int64_t dims[3], double horizon, double s_c, int law,
                           const int64_t* run_steps, const int* threads, int n_runs,
                           double* seconds_out, int64_t* live_bonds_out,
                           double* build_seconds_out) {
    return map_exceptions([&] {
        set_worker_cap(0);
        GridDesc grid;
        grid.spacing = 1;
        grid.counts = {dims[0], dims[1], dims[2]};
        ModelBundle bundle;
        bundle.particles.coords = grid_coordinates(grid);
        const Index n = grid.node_count();
        bundle.particles.volume.assign(std::size_t(n), 1);
        bundle.particles.density.assign(std::size_t(n), 1);
        bundle.particles.material_tag.assign(std::size_t(n), 0);
        bundle.model.laws.push_back(law == 1 ? DamageLaw::trilinear(1, Real(1e-3), Real(2e-3), s_c)
                                             : DamageLaw::pmb(1, s_c));
        bundle.bc = BoundaryConditions::none(n);
        bundle.dt = Real(1e-3);
        const auto b0 = std::chrono::steady_clock::now();
        NeighborList family = build_family(bundle.particles.coords, horizon, &grid);
        const auto b1 = std::chrono::steady_clock::now();
        *build_seconds_out = std::chrono::duration<double>(b1 - b0).count();
        SimulationState state = make_state_for(bundle, family);
        family = NeighborList{};  // the state holds its own copy
        for (Index i = 0; i < n; ++i) {
            const Vec3 x = load_vec3(bundle.particles.coords, i);
            store_vec3(state.u, i,
                       {Real(1e-4) * std::sin(Real(0.1) * x.x + Real(0.2) * x.y),
                        Real(1e-4) * std::cos(Real(0.15) * x.y + Real(0.1) * x.z),
                        Real(1e-4) * std::sin(Real(0.12) * x.z + Real(0.17) * x.x)});
        }
        int64_t live = 0;
        for (auto c : state.connectivity.n_neigh)
            live += c;
        *live_bonds_out = live;
        int64_t step = 0;
        for (int r = 0; r < n_runs; ++r) {
            set_worker_cap(unsigned(threads[r]));
            SimulateOptions opts;
            opts.steps = run_steps[r];
            opts.first_step = step;
            opts.variant = KernelVariant::bond_parallel;
            const auto t0 = std::chrono::steady_clock::now();
            simulate(bundle, state, opts);
            const auto t1 = std::chrono::steady_clock::now();
            seconds_out[r] = std::chrono::duration<double>(t1 - t0).count();
            step += run_steps[r];
        }
        set_worker_cap(0);
    });
}

} // extern "C"
