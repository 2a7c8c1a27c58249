/*
 * pd_oracle.c -- TEST INFRASTRUCTURE ONLY (see pd_oracle.h).
 *
 * Plain-C restatement of the reference CPU path.  Each function cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 * Expression order is kept operation for operation so that, compiled without
 * FMA contraction, results are bitwise equal to the reference build; the
 * golden fixtures in tests/golden/ pin that claim.
 */
#define _GNU_SOURCE
#include "pd_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];
static int g_threads = 1;

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }
void orc_set_threads(int threads) { g_threads = threads < 1 ? 1 : threads; }
void orc_free(void* p) { free(p); }

/* ---- parallel_chunks (parallel.cpp:42-75): contiguous node chunks ------- */

typedef void (*chunk_fn)(void* ctx, int64_t begin, int64_t end);
typedef struct {
    chunk_fn fn;
    void* ctx;
    int64_t begin, end;
} chunk_job;

static void* chunk_main(void* p) {
    chunk_job* j = (chunk_job*)p;
    j->fn(j->ctx, j->begin, j->end);
    return NULL;
}

static void parallel_chunks(int64_t n, chunk_fn fn, void* ctx) {
    if (n <= 0)
        return;
    int64_t k = g_threads < n ? g_threads : n;
    if (k <= 1) {
        fn(ctx, 0, n);
        return;
    }
    const int64_t chunk = (n + k - 1) / k;
    pthread_t* th = (pthread_t*)calloc((size_t)k, sizeof(pthread_t));
    chunk_job* jobs = (chunk_job*)calloc((size_t)k, sizeof(chunk_job));
    int* started = (int*)calloc((size_t)k, sizeof(int));
    for (int64_t w = 1; w < k; ++w) {
        const int64_t b = w * chunk, e = (b + chunk < n) ? b + chunk : n;
        if (b < e) {
            jobs[w] = (chunk_job){fn, ctx, b, e};
            started[w] = pthread_create(&th[w], NULL, chunk_main, &jobs[w]) == 0;
            if (!started[w])
                fn(ctx, b, e);
        }
    }
    fn(ctx, 0, chunk < n ? chunk : n);
    for (int64_t w = 1; w < k; ++w)
        if (started[w])
            pthread_join(th[w], NULL);
    free(th);
    free(jobs);
    free(started);
}

/* ---- reduce_group (engine.cpp:11-19) ------------------------------------ */

static int is_pow2(int64_t n) { return n > 0 && (n & (n - 1)) == 0; }

static void tree_reduce(double* c, int64_t n) {
    for (int64_t stride = n / 2; stride > 0; stride /= 2)
        for (int64_t k = 0; k < stride; ++k) {
            c[3 * k] += c[3 * (k + stride)];
            c[3 * k + 1] += c[3 * (k + stride) + 1];
            c[3 * k + 2] += c[3 * (k + stride) + 2];
        }
}

int orc_reduce_group(double* c, int64_t n, double out[3]) {
    if (n == 0 || !is_pow2(n))
        return fail(PD_E_INVALID_ARGUMENT, "reduce_group: size must be a power of two");
    tree_reduce(c, n);
    out[0] = c[0];
    out[1] = c[1];
    out[2] = c[2];
    return PD_OK;
}

/* ---- DamageLaw / DamageModel validation (types.cpp:50-105) -------------- */

static int law_validate(const pd_law* l) {
    if (!(l->stiffness > 0))
        return fail(PD_E_INVALID_ARGUMENT, "DamageLaw: stiffness must be positive");
    if (l->n_breakpoints < 1)
        return fail(PD_E_INVALID_ARGUMENT,
                    "DamageLaw: breakpoints and forces must match and be non-empty");
    if (l->n_breakpoints > PD_MAX_BREAKPOINTS)
        return fail(PD_E_INVALID_ARGUMENT, "DamageLaw: more than %d breakpoints",
                    PD_MAX_BREAKPOINTS);
    double prev = 0;
    for (int k = 0; k < l->n_breakpoints; ++k) {
        if (!(l->breakpoints[k] > prev))
            return fail(PD_E_INVALID_ARGUMENT,
                        "DamageLaw: breakpoints must be strictly increasing and positive");
        prev = l->breakpoints[k];
    }
    const double f0 = l->stiffness * l->breakpoints[0];
    const double af0 = fabs(f0);
    if (fabs(l->forces[0] - f0) > 1e-9 * (af0 > 1.0 ? af0 : 1.0))
        return fail(PD_E_INVALID_ARGUMENT, "DamageLaw: envelope must leave the origin with slope c");
    return PD_OK;
}

static int model_validate(const pd_damage_model* m) {
    if (m->n_laws < 1)
        return fail(PD_E_INVALID_ARGUMENT, "DamageModel: no laws defined");
    for (int k = 0; k < m->n_laws; ++k) {
        int rc = law_validate(&m->laws[k]);
        if (rc)
            return rc;
    }
    if (m->damping < 0)
        return fail(PD_E_INVALID_ARGUMENT, "DamageModel: negative damping");
    return PD_OK;
}

static int model_needs_history(const pd_damage_model* m) {
    for (int k = 0; k < m->n_laws; ++k)
        if (m->laws[k].n_breakpoints > 1)
            return 1;
    return 0;
}

/* ---- formulas (formulas.hpp:77-96) -------------------------------------- */

static double envelope_force(const pd_law* law, double s) {
    double s_prev = 0, f_prev = 0;
    for (int k = 0; k < law->n_breakpoints; ++k) {
        const double s_k = law->breakpoints[k];
        if (s < s_k || k + 1 == law->n_breakpoints) {
            const double t = (s - s_prev) / (s_k - s_prev);
            return f_prev + t * (law->forces[k] - f_prev);
        }
        s_prev = s_k;
        f_prev = law->forces[k];
    }
    return law->stiffness * s;
}

static double secant_stiffness(const pd_law* law, double h) {
    if (h <= 0)
        return law->stiffness;
    return envelope_force(law, h) / h;
}

/* ---- compute_forces (engine.cpp:23-169) --------------------------------- */

typedef struct {
    pd_state* state;
    const pd_particles* p;
    const pd_damage_model* model;
    const pd_corrections* corr;
    pd_force_field* out;
    int64_t group;
} force_ctx;

/* bond_contribution (engine.cpp:53-109); writes the slot's Vec3 into c. */
static void bond_contribution(force_ctx* fc, int64_t i, const double xi[3], const double ui[3],
                              int i_no_fail, int64_t idx, double c[3]) {
    pd_state* st = fc->state;
    int32_t* slot = &st->connectivity.entries[idx];
    const int32_t j = *slot;
    c[0] = c[1] = c[2] = 0;
    if (j < 0)
        return;
    const double* xj = fc->p->coords + 3 * (int64_t)j;
    const double* uj = st->u + 3 * (int64_t)j;
    const double ref[3] = {xj[0] - xi[0], xj[1] - xi[1], xj[2] - xi[2]};
    const double du[3] = {uj[0] - ui[0], uj[1] - ui[1], uj[2] - ui[2]};
    const double cur[3] = {ref[0] + du[0], ref[1] + du[1], ref[2] + du[2]};
    const double ref_len = sqrt(ref[0] * ref[0] + ref[1] * ref[1] + ref[2] * ref[2]);
    const double cur_len = sqrt(cur[0] * cur[0] + cur[1] * cur[1] + cur[2] * cur[2]);
    const double s = (cur_len - ref_len) / ref_len;

    const pd_law* law = st->connectivity.bond_type_size == 0
                            ? &fc->model->laws[0]
                            : &fc->model->laws[st->connectivity.bond_type[idx]];
    double f_scalar;
    const int no_fail =
        i_no_fail || (fc->corr->no_failure_size != 0 && fc->corr->no_failure[j] != 0);
    if (no_fail) {
        f_scalar = law->stiffness * s;
    } else if (law->n_breakpoints == 1) {
        if (s >= law->breakpoints[0]) {
            *slot = -1;
            --st->connectivity.n_neigh[i];
            return;
        }
        f_scalar = law->stiffness * s;
    } else {
        const double s_c = law->breakpoints[law->n_breakpoints - 1];
        double* hist = &st->bond_history[idx];
        const double h = *hist;
        if (s > h)
            *hist = s;
        if (h >= s_c || s >= s_c) {
            *slot = -1;
            --st->connectivity.n_neigh[i];
            return;
        }
        f_scalar = (s >= h) ? envelope_force(law, s) : secant_stiffness(law, h) * s;
    }
    if (cur_len < 1e-30)
        return;
    double scale = f_scalar * fc->p->volume[j];
    if (fc->corr->lambda_size != 0)
        scale *= fc->corr->lambda[idx];
    if (fc->corr->beta_size != 0)
        scale *= fc->corr->beta[idx];
    const double q = scale / cur_len;
    c[0] = cur[0] * q;
    c[1] = cur[1] * q;
    c[2] = cur[2] * q;
}

static void bpr_chunk(void* vctx, int64_t begin, int64_t end) {
    force_ctx* fc = (force_ctx*)vctx;
    const int64_t group = fc->group;
    double* cache = (double*)malloc((size_t)(3 * group) * sizeof(double));
    for (int64_t i = begin; i < end; ++i) {
        const double* xi = fc->p->coords + 3 * i;
        const double* ui = fc->state->u + 3 * i;
        const int i_no_fail = fc->corr->no_failure_size != 0 && fc->corr->no_failure[i] != 0;
        for (int64_t k = 0; k < group; ++k)
            bond_contribution(fc, i, xi, ui, i_no_fail, i * group + k, cache + 3 * k);
        tree_reduce(cache, group);
        fc->out->body_force[3 * i] = cache[0];
        fc->out->body_force[3 * i + 1] = cache[1];
        fc->out->body_force[3 * i + 2] = cache[2];
    }
    free(cache);
}

static void node_chunk(void* vctx, int64_t begin, int64_t end) {
    force_ctx* fc = (force_ctx*)vctx;
    const int64_t group = fc->group;
    for (int64_t i = begin; i < end; ++i) {
        const double* xi = fc->p->coords + 3 * i;
        const double* ui = fc->state->u + 3 * i;
        const int i_no_fail = fc->corr->no_failure_size != 0 && fc->corr->no_failure[i] != 0;
        double sum[3] = {0, 0, 0}, c[3];
        for (int64_t k = 0; k < group; ++k) {
            bond_contribution(fc, i, xi, ui, i_no_fail, i * group + k, c);
            sum[0] += c[0];
            sum[1] += c[1];
            sum[2] += c[2];
        }
        fc->out->body_force[3 * i] = sum[0];
        fc->out->body_force[3 * i + 1] = sum[1];
        fc->out->body_force[3 * i + 2] = sum[2];
    }
}

/* check_force_inputs (engine.cpp:30-49) + check_state_finite (engine.cpp:23-28) */
static int check_force_inputs(const pd_state* st, const pd_particles* p,
                              const pd_damage_model* m, const pd_corrections* corr) {
    const int64_t n = st->connectivity.n;
    if (p->n != n)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: particle set does not match state");
    const int64_t slots = n * st->connectivity.group_size;
    if (corr->lambda_size != 0 && corr->lambda_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: lambda size mismatch");
    if (corr->beta_size != 0 && corr->beta_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: beta size mismatch");
    if (corr->no_failure_size != 0 && corr->no_failure_size != n)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: no_failure size mismatch");
    if (model_needs_history(m) && st->bond_history_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: model needs per-bond history");
    if (st->connectivity.bond_type_size != 0 && m->n_laws < 2 &&
        st->connectivity.bond_type_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "compute_forces: bond_type size mismatch");
    int rc = model_validate(m);
    if (rc)
        return rc;
    /* out-of-range bond types are UB in the reference; reject them */
    if (st->connectivity.bond_type_size != 0)
        for (int64_t k = 0; k < slots; ++k)
            if (st->connectivity.entries[k] >= 0 && st->connectivity.bond_type[k] >= m->n_laws)
                return fail(PD_E_INVALID_ARGUMENT, "compute_forces: bond_type out of range");
    for (int64_t k = 0; k < 3 * n; ++k)
        if (!isfinite(st->u[k]))
            return fail(PD_E_RUNTIME, "compute_forces: non-finite displacement at step %lld",
                        (long long)st->step);
    return PD_OK;
}

int orc_compute_forces(int32_t variant, pd_state* state, const pd_particles* particles,
                       const pd_damage_model* model, const pd_corrections* corr,
                       pd_force_field* out) {
    int rc = check_force_inputs(state, particles, model, corr);
    if (rc)
        return rc;
    force_ctx fc = {state, particles, model, corr, out, state->connectivity.group_size};
    parallel_chunks(state->connectivity.n, variant == PD_NODE_PARALLEL ? node_chunk : bpr_chunk,
                    &fc);
    return PD_OK;
}

/* ---- integrators (engine.cpp:171-252) ----------------------------------- */

static int check_density(const double* density, int64_t density_size, int64_t n) {
    if (density_size != n)
        return fail(PD_E_INVALID_ARGUMENT, "integrator: density array does not match node count");
    for (int64_t i = 0; i < n; ++i)
        if (!(density[i] > 0))
            return fail(PD_E_DOMAIN, "integrator: density must be positive");
    return PD_OK;
}

int orc_step_euler(pd_state* st, const pd_force_field* f, double dt, const double* density,
                   int64_t density_size) {
    if (!(dt > 0))
        return fail(PD_E_DOMAIN, "step_euler: dt must be positive");
    const int64_t n = st->connectivity.n;
    int rc = check_density(density, density_size, n);
    if (rc)
        return rc;
    for (int64_t i = 0; i < n; ++i) {
        const double inv = 1.0 / density[i];
        for (int ax = 0; ax < 3; ++ax) {
            const int64_t k = 3 * i + ax;
            const double acc = (f->body_force[k] + f->external_force[k]) * inv;
            const double v_old = st->v[k];
            st->a[k] = acc;
            st->v[k] = v_old + acc * dt;
            st->u[k] = st->u[k] + v_old * dt;
        }
    }
    return PD_OK;
}

int orc_step_euler_cromer(pd_state* st, const pd_force_field* f, double dt,
                          const double* density, int64_t density_size) {
    if (!(dt > 0))
        return fail(PD_E_DOMAIN, "step_euler_cromer: dt must be positive");
    const int64_t n = st->connectivity.n;
    int rc = check_density(density, density_size, n);
    if (rc)
        return rc;
    for (int64_t i = 0; i < n; ++i) {
        const double inv = 1.0 / density[i];
        for (int ax = 0; ax < 3; ++ax) {
            const int64_t k = 3 * i + ax;
            const double acc = (f->body_force[k] + f->external_force[k]) * inv;
            const double v_new = st->v[k] + acc * dt;
            st->a[k] = acc;
            st->v[k] = v_new;
            st->u[k] = st->u[k] + v_new * dt;
        }
    }
    return PD_OK;
}

int orc_verlet_drift(pd_state* st, double dt) {
    if (!(dt > 0))
        return fail(PD_E_DOMAIN, "verlet_drift: dt must be positive");
    const int64_t n3 = 3 * st->connectivity.n;
    const double half_dt2 = dt * dt / 2;
    for (int64_t k = 0; k < n3; ++k)
        st->u[k] = st->u[k] + st->v[k] * dt + st->a[k] * half_dt2;
    return PD_OK;
}

int orc_verlet_kick(pd_state* st, const pd_force_field* f, double dt, double damping,
                    const double* density, int64_t density_size) {
    if (!(dt > 0))
        return fail(PD_E_DOMAIN, "verlet_kick: dt must be positive");
    const int64_t n = st->connectivity.n;
    int rc = check_density(density, density_size, n);
    if (rc)
        return rc;
    const double half_dt = dt / 2;
    for (int64_t i = 0; i < n; ++i) {
        const double inv = 1.0 / density[i];
        for (int ax = 0; ax < 3; ++ax) {
            const int64_t k = 3 * i + ax;
            const double v_half = st->v[k] + st->a[k] * half_dt;
            const double a_new =
                ((f->body_force[k] + f->external_force[k]) - v_half * damping) * inv;
            st->a[k] = a_new;
            st->v[k] = v_half + a_new * half_dt;
        }
    }
    return PD_OK;
}

/* ---- RampProfile (types.cpp:119-169) ------------------------------------ */

double orc_ramp_scale(const pd_ramp* r, int64_t step) {
    switch (r->kind) {
    case PD_RAMP_CONSTANT:
        return r->target_scale;
    case PD_RAMP_LINEAR:
        if (r->rise_steps <= 0 || step >= r->rise_steps)
            return r->target_scale;
        return r->target_scale * (double)step / (double)r->rise_steps;
    case PD_RAMP_QUINTIC: {
        if (r->rise_steps <= 0 || step >= r->rise_steps)
            return r->target_scale;
        const double t = (double)step / (double)r->rise_steps;
        return r->target_scale * t * t * t * (10 + t * (-15 + 6 * t));
    }
    }
    return r->target_scale;
}

double orc_ramp_rate(const pd_ramp* r, int64_t step) {
    switch (r->kind) {
    case PD_RAMP_CONSTANT:
        return 0;
    case PD_RAMP_LINEAR:
        if (r->rise_steps <= 0 || step >= r->rise_steps)
            return 0;
        return r->target_scale / (double)r->rise_steps;
    case PD_RAMP_QUINTIC: {
        if (r->rise_steps <= 0 || step >= r->rise_steps)
            return 0;
        const double t = (double)step / (double)r->rise_steps;
        return r->target_scale * 30 * t * t * (t - 1) * (t - 1) / (double)r->rise_steps;
    }
    }
    return 0;
}

double orc_ramp_accel(const pd_ramp* r, int64_t step) {
    switch (r->kind) {
    case PD_RAMP_CONSTANT:
    case PD_RAMP_LINEAR:
        return 0;
    case PD_RAMP_QUINTIC: {
        if (r->rise_steps <= 0 || step >= r->rise_steps)
            return 0;
        const double t = (double)step / (double)r->rise_steps;
        return r->target_scale * 60 * t * (2 * t - 1) * (t - 1) /
               ((double)r->rise_steps * (double)r->rise_steps);
    }
    }
    return 0;
}

/* ---- boundary conditions (types.cpp:181-196, engine.cpp:262-297) -------- */

int orc_bc_validate(const pd_boundary* bc, int64_t n) {
    if (bc->kind_size != 3 * n || bc->magnitude_size != 3 * n || bc->ramp_id_size != 3 * n ||
        bc->no_failure_size != n)
        return fail(PD_E_INVALID_ARGUMENT,
                    "BoundaryConditions: field lengths do not match node count");
    if (bc->n_ramps < 1)
        return fail(PD_E_INVALID_ARGUMENT, "BoundaryConditions: no ramp profiles");
    for (int64_t k = 0; k < 3 * n; ++k)
        if (bc->ramp_id[k] >= bc->n_ramps)
            return fail(PD_E_INVALID_ARGUMENT, "BoundaryConditions: ramp id out of range");
    for (int32_t s = 0; s < bc->n_tip_sets; ++s)
        for (int64_t t = bc->tip_offsets[s]; t < bc->tip_offsets[s + 1]; ++t)
            if (bc->tip_nodes[t] < 0 || bc->tip_nodes[t] >= n)
                return fail(PD_E_INVALID_ARGUMENT,
                            "BoundaryConditions: tip set #%d has an invalid node index", s);
    return PD_OK;
}

void orc_apply_displacement_positions(pd_state* st, const pd_boundary* bc, int64_t step) {
    const int64_t n3 = 3 * st->connectivity.n;
    for (int64_t k = 0; k < n3; ++k) {
        if (bc->kind[k] != PD_BC_DISPLACEMENT)
            continue;
        st->u[k] = bc->magnitude[k] * orc_ramp_scale(&bc->ramps[bc->ramp_id[k]], step);
    }
}

void orc_apply_displacement_kinematics(pd_state* st, const pd_boundary* bc, int64_t step,
                                       double dt) {
    const int64_t n3 = 3 * st->connectivity.n;
    for (int64_t k = 0; k < n3; ++k) {
        if (bc->kind[k] != PD_BC_DISPLACEMENT)
            continue;
        const pd_ramp* r = &bc->ramps[bc->ramp_id[k]];
        st->v[k] = bc->magnitude[k] * orc_ramp_rate(r, step) / dt;
        st->a[k] = bc->magnitude[k] * orc_ramp_accel(r, step) / (dt * dt);
    }
}

void orc_accumulate_external_force(const pd_boundary* bc, int64_t step, double* ext, int64_t n) {
    for (int64_t k = 0; k < 3 * n; ++k) {
        if (bc->kind[k] != PD_BC_FORCE)
            continue;
        ext[k] += bc->magnitude[k] * orc_ramp_scale(&bc->ramps[bc->ramp_id[k]], step);
    }
}

/* ---- simulate (engine.cpp:335-425) -------------------------------------- */

static int particles_validate(const pd_particles* p) {
    const int64_t n = p->n;
    if (n < 1)
        return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: empty");
    if (p->coords_size != 3 * n || p->density_size != n)
        return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: field lengths differ");
    for (int64_t i = 0; i < n; ++i) {
        if (!(p->volume[i] > 0))
            return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: non-positive volume at node %lld",
                        (long long)i);
        if (!(p->density[i] > 0))
            return fail(PD_E_INVALID_ARGUMENT, "ParticleSet: non-positive density at node %lld",
                        (long long)i);
    }
    return PD_OK;
}

static void record_tips(const pd_boundary* bc, const pd_particles* p, const pd_state* st,
                        const pd_force_field* f, pd_tip_record* out) {
    for (int32_t s = 0; s < bc->n_tip_sets; ++s) {
        pd_tip_record rec;
        memset(&rec, 0, sizeof rec);
        rec.step = st->step;
        const int64_t b = bc->tip_offsets[s], e = bc->tip_offsets[s + 1];
        for (int64_t t = b; t < e; ++t) {
            const int64_t i = bc->tip_nodes[t];
            const double vol = p->volume[i];
            for (int ax = 0; ax < 3; ++ax) {
                rec.mean_u[ax] += st->u[3 * i + ax];
                rec.mean_v[ax] += st->v[3 * i + ax];
                rec.mean_a[ax] += st->a[3 * i + ax];
                rec.body_force_sum[ax] += f->body_force[3 * i + ax] * vol;
                rec.external_force_sum[ax] += f->external_force[3 * i + ax] * vol;
            }
        }
        if (e > b) {
            const double inv = 1.0 / (double)(e - b);
            for (int ax = 0; ax < 3; ++ax) {
                rec.mean_u[ax] = rec.mean_u[ax] * inv;
                rec.mean_v[ax] = rec.mean_v[ax] * inv;
                rec.mean_a[ax] = rec.mean_a[ax] * inv;
            }
        }
        out[s] = rec;
    }
}

int orc_simulate(const pd_bundle* bundle, pd_state* state, const pd_options* opt,
                 pd_write_hook on_write, void* user, pd_tip_record* tips_out,
                 int64_t tips_capacity, int64_t* n_tips_out) {
    if (n_tips_out)
        *n_tips_out = 0;
    if (opt->steps < 1)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: steps must be >= 1");
    int rc = particles_validate(&bundle->particles);
    if (!rc)
        rc = model_validate(&bundle->model);
    if (!rc)
        rc = orc_bc_validate(&bundle->bc, bundle->particles.n);
    if (rc)
        return rc;
    if (!(bundle->dt > 0))
        return fail(PD_E_INVALID_ARGUMENT, "ModelBundle: dt must be positive");
    const int64_t n = bundle->particles.n;
    if (state->connectivity.n != n)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: state does not match the bundle");
    const int64_t slots = n * state->connectivity.group_size;
    if (model_needs_history(&bundle->model) && state->bond_history_size != slots)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: bond_history must be sized n x N");
    int64_t writes = 0;
    if (opt->write_every > 0)
        for (int64_t s = opt->first_step; s < opt->first_step + opt->steps; ++s)
            if ((s + 1) % opt->write_every == 0)
                ++writes;
    if (writes * bundle->bc.n_tip_sets > tips_capacity)
        return fail(PD_E_INVALID_ARGUMENT, "simulate: tips_out capacity too small");

    pd_corrections corr = bundle->corrections;
    corr.no_failure = bundle->bc.no_failure;
    corr.no_failure_size = bundle->bc.no_failure_size;

    const double dt = bundle->dt;
    double* body = (double*)calloc((size_t)(3 * n), sizeof(double));
    double* ext = (double*)calloc((size_t)(3 * n), sizeof(double));
    pd_force_field forces = {body, ext};
    state->step = opt->first_step;
    int64_t n_tips = 0;

    const int64_t last = opt->first_step + opt->steps;
    for (int64_t s = opt->first_step; s < last && rc == PD_OK; ++s) {
        if (opt->integrator == PD_VELOCITY_VERLET) {
            rc = orc_verlet_drift(state, dt);
            if (rc)
                break;
            orc_apply_displacement_positions(state, &bundle->bc, s + 1);
            memset(ext, 0, (size_t)(3 * n) * sizeof(double));
            orc_accumulate_external_force(&bundle->bc, s + 1, ext, n);
            rc = orc_compute_forces(opt->variant, state, &bundle->particles, &bundle->model, &corr,
                                    &forces);
            if (rc)
                break;
            rc = orc_verlet_kick(state, &forces, dt, bundle->model.damping,
                                 bundle->particles.density, bundle->particles.density_size);
            if (rc)
                break;
            orc_apply_displacement_kinematics(state, &bundle->bc, s + 1, dt);
        } else {
            memset(ext, 0, (size_t)(3 * n) * sizeof(double));
            orc_accumulate_external_force(&bundle->bc, s, ext, n);
            rc = orc_compute_forces(opt->variant, state, &bundle->particles, &bundle->model, &corr,
                                    &forces);
            if (rc)
                break;
            if (opt->integrator == PD_EULER)
                rc = orc_step_euler(state, &forces, dt, bundle->particles.density,
                                    bundle->particles.density_size);
            else
                rc = orc_step_euler_cromer(state, &forces, dt, bundle->particles.density,
                                           bundle->particles.density_size);
            if (rc)
                break;
            orc_apply_displacement_positions(state, &bundle->bc, s + 1);
            orc_apply_displacement_kinematics(state, &bundle->bc, s + 1, dt);
        }
        state->step = s + 1;
        if (opt->write_every > 0 && (s + 1) % opt->write_every == 0) {
            if (bundle->bc.n_tip_sets > 0) {
                record_tips(&bundle->bc, &bundle->particles, state, &forces, tips_out + n_tips);
                n_tips += bundle->bc.n_tip_sets;
            }
            if (on_write && on_write(user, state, &forces) != 0)
                rc = fail(PD_E_RUNTIME, "simulate: write hook failed at step %lld",
                          (long long)(s + 1));
        }
    }
    if (n_tips_out)
        *n_tips_out = n_tips;
    free(body);
    free(ext);
    return rc;
}

/* ---- geometry (geometry.cpp:25-38, 86-211, 285-319) --------------------- */

int orc_grid_coordinates(const double origin[3], double spacing, const int64_t counts[3],
                         double* out) {
    if (!(spacing > 0) || counts[0] < 1 || counts[1] < 1 || counts[2] < 1)
        return fail(PD_E_INVALID_ARGUMENT, "grid: spacing and counts must be positive");
    int64_t k = 0;
    for (int64_t kz = 0; kz < counts[2]; ++kz)
        for (int64_t ky = 0; ky < counts[1]; ++ky)
            for (int64_t kx = 0; kx < counts[0]; ++kx) {
                out[k++] = origin[0] + (double)kx * spacing;
                out[k++] = origin[1] + (double)ky * spacing;
                out[k++] = origin[2] + (double)kz * spacing;
            }
    return PD_OK;
}

typedef struct {
    double origin[3];
    double cell;
    int64_t nx, ny, nz;
    /* dense cell table: nodes of cell c are order[start[c] .. start[c+1]) */
    int64_t ncells;
    int64_t* start;
    int32_t* order;
    /* sparse fallback: sorted (cell, node) pairs */
    int64_t* sorted_cell;
} cell_index;

static int64_t clamp_coord(double x, double o, double cell, int64_t count) {
    int64_t c = (int64_t)floor((x - o) / cell);
    if (c < 0)
        c = 0;
    if (c > count - 1)
        c = count - 1;
    return c;
}

typedef struct {
    int64_t cell;
    int32_t node;
} cell_pair;

static int cmp_pair(const void* a, const void* b) {
    const cell_pair* x = (const cell_pair*)a;
    const cell_pair* y = (const cell_pair*)b;
    if (x->cell != y->cell)
        return x->cell < y->cell ? -1 : 1;
    return x->node < y->node ? -1 : (x->node > y->node);
}

/* make_cell_index (geometry.cpp:97-129) */
static void make_cell_index(const double* coords, int64_t n, double horizon,
                            const double* hint, cell_index* ix) {
    double lo[3], hi[3];
    if (hint && hint[3] > 0) {
        for (int d = 0; d < 3; ++d) {
            lo[d] = hint[d];
            hi[d] = hint[d] + (double)((int64_t)hint[4 + d] - 1) * hint[3];
        }
    } else {
        for (int d = 0; d < 3; ++d)
            lo[d] = hi[d] = coords[d];
        for (int64_t i = 1; i < n; ++i)
            for (int d = 0; d < 3; ++d) {
                const double x = coords[3 * i + d];
                lo[d] = x < lo[d] ? x : lo[d];
                hi[d] = x > hi[d] ? x : hi[d];
            }
    }
    ix->cell = horizon;
    for (int d = 0; d < 3; ++d)
        ix->origin[d] = lo[d];
    int64_t c[3];
    for (int d = 0; d < 3; ++d) {
        c[d] = (int64_t)floor((hi[d] - lo[d]) / ix->cell) + 1;
        if (c[d] < 1)
            c[d] = 1;
    }
    ix->nx = c[0];
    ix->ny = c[1];
    ix->nz = c[2];
    ix->ncells = c[0] * c[1] * c[2];
    cell_pair* pairs = (cell_pair*)malloc((size_t)n * sizeof(cell_pair));
    for (int64_t i = 0; i < n; ++i) {
        const int64_t cx = clamp_coord(coords[3 * i], lo[0], ix->cell, ix->nx);
        const int64_t cy = clamp_coord(coords[3 * i + 1], lo[1], ix->cell, ix->ny);
        const int64_t cz = clamp_coord(coords[3 * i + 2], lo[2], ix->cell, ix->nz);
        pairs[i].cell = (cz * ix->ny + cy) * ix->nx + cx;
        pairs[i].node = (int32_t)i;
    }
    ix->order = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    ix->start = NULL;
    ix->sorted_cell = NULL;
    if (ix->ncells <= 8 * n + 4096) {
        ix->start = (int64_t*)calloc((size_t)(ix->ncells + 1), sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i)
            ix->start[pairs[i].cell + 1]++;
        for (int64_t k = 0; k < ix->ncells; ++k)
            ix->start[k + 1] += ix->start[k];
        int64_t* fill = (int64_t*)malloc((size_t)ix->ncells * sizeof(int64_t));
        memcpy(fill, ix->start, (size_t)ix->ncells * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i)
            ix->order[fill[pairs[i].cell]++] = (int32_t)i;
        free(fill);
    } else {
        qsort(pairs, (size_t)n, sizeof(cell_pair), cmp_pair);
        ix->sorted_cell = (int64_t*)malloc((size_t)n * sizeof(int64_t));
        for (int64_t i = 0; i < n; ++i) {
            ix->sorted_cell[i] = pairs[i].cell;
            ix->order[i] = pairs[i].node;
        }
    }
    free(pairs);
}

static void cell_range(const cell_index* ix, int64_t n, int64_t id, int64_t* b, int64_t* e) {
    if (ix->start) {
        *b = ix->start[id];
        *e = ix->start[id + 1];
        return;
    }
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (ix->sorted_cell[mid] < id)
            lo = mid + 1;
        else
            hi = mid;
    }
    *b = lo;
    hi = n;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (ix->sorted_cell[mid] <= id)
            lo = mid + 1;
        else
            hi = mid;
    }
    *e = lo;
}

static int cmp_i32(const void* a, const void* b) {
    const int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return x < y ? -1 : (x > y);
}

typedef struct {
    const double* coords;
    int64_t n;
    double h2;
    const cell_index* ix;
    int32_t** rows;
    int32_t* counts;
    volatile int error;
    int64_t err_i, err_j;
} family_ctx;

static void family_chunk(void* vctx, int64_t begin, int64_t end) {
    family_ctx* fc = (family_ctx*)vctx;
    const cell_index* ix = fc->ix;
    int32_t cap = 64;
    int32_t* buf = (int32_t*)malloc((size_t)cap * sizeof(int32_t));
    for (int64_t i = begin; i < end && !fc->error; ++i) {
        const double* xi = fc->coords + 3 * i;
        const int64_t cx = clamp_coord(xi[0], ix->origin[0], ix->cell, ix->nx);
        const int64_t cy = clamp_coord(xi[1], ix->origin[1], ix->cell, ix->ny);
        const int64_t cz = clamp_coord(xi[2], ix->origin[2], ix->cell, ix->nz);
        int32_t cnt = 0;
        for (int64_t dz = -1; dz <= 1; ++dz)
            for (int64_t dy = -1; dy <= 1; ++dy)
                for (int64_t dx = -1; dx <= 1; ++dx) {
                    const int64_t ccx = cx + dx, ccy = cy + dy, ccz = cz + dz;
                    if (ccx < 0 || ccy < 0 || ccz < 0 || ccx >= ix->nx || ccy >= ix->ny ||
                        ccz >= ix->nz)
                        continue;
                    int64_t b, e;
                    cell_range(ix, fc->n, (ccz * ix->ny + ccy) * ix->nx + ccx, &b, &e);
                    for (int64_t t = b; t < e; ++t) {
                        const int32_t j = ix->order[t];
                        if ((int64_t)j == i)
                            continue;
                        const double* xj = fc->coords + 3 * (int64_t)j;
                        const double d0 = xj[0] - xi[0], d1 = xj[1] - xi[1], d2 = xj[2] - xi[2];
                        const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
                        if (r2 <= fc->h2) {
                            if (r2 < 1e-24) {
                                fc->err_i = i;
                                fc->err_j = j;
                                fc->error = 1;
                            }
                            if (cnt == cap) {
                                cap *= 2;
                                buf = (int32_t*)realloc(buf, (size_t)cap * sizeof(int32_t));
                            }
                            buf[cnt++] = j;
                        }
                    }
                }
        qsort(buf, (size_t)cnt, sizeof(int32_t), cmp_i32);
        fc->rows[i] = (int32_t*)malloc((size_t)(cnt > 0 ? cnt : 1) * sizeof(int32_t));
        memcpy(fc->rows[i], buf, (size_t)cnt * sizeof(int32_t));
        fc->counts[i] = cnt;
    }
    free(buf);
}

int orc_build_family(const double* coords, int64_t n, double horizon, const double* grid_hint,
                     int32_t** entries_out, int32_t** n_neigh_out, int32_t** initial_out,
                     int64_t* group_size_out) {
    if (!(horizon > 0))
        return fail(PD_E_DOMAIN, "build_family: horizon must be positive");
    if (n < 1)
        return fail(PD_E_INVALID_ARGUMENT, "build_family: bad coordinate array");
    cell_index ix;
    make_cell_index(coords, n, horizon, grid_hint, &ix);
    family_ctx fc;
    memset(&fc, 0, sizeof fc);
    fc.coords = coords;
    fc.n = n;
    fc.h2 = horizon * horizon;
    fc.ix = &ix;
    fc.rows = (int32_t**)calloc((size_t)n, sizeof(int32_t*));
    fc.counts = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    parallel_chunks(n, family_chunk, &fc);
    int rc = PD_OK;
    if (fc.error) {
        rc = fail(PD_E_INVALID_ARGUMENT, "build_family: coincident nodes %lld and %lld",
                  (long long)fc.err_i, (long long)fc.err_j);
    } else {
        /* pack_rows (geometry.cpp:131-161) */
        int64_t max_count = 1;
        for (int64_t i = 0; i < n; ++i)
            if (fc.counts[i] > max_count)
                max_count = fc.counts[i];
        int64_t group = 1;
        while (group < max_count)
            group *= 2;
        int32_t* entries = (int32_t*)malloc((size_t)(n * group) * sizeof(int32_t));
        int32_t* nn = (int32_t*)malloc((size_t)n * sizeof(int32_t));
        int32_t* init = (int32_t*)malloc((size_t)n * sizeof(int32_t));
        for (int64_t i = 0; i < n; ++i) {
            int32_t* row = entries + i * group;
            for (int64_t k = 0; k < group; ++k)
                row[k] = k < fc.counts[i] ? fc.rows[i][k] : -1;
            nn[i] = init[i] = fc.counts[i];
        }
        *entries_out = entries;
        *n_neigh_out = nn;
        *initial_out = init;
        *group_size_out = group;
    }
    for (int64_t i = 0; i < n; ++i)
        free(fc.rows[i]);
    free(fc.rows);
    free(fc.counts);
    free(ix.start);
    free(ix.order);
    free(ix.sorted_cell);
    return rc;
}

/* break_initial_bonds + predicates (geometry.cpp:285-319) */
static void break_with(pd_neighbor_list* family, const double* coords, int kind, int axis,
                       double position, int sweep_axis, double depth) {
    const int64_t n = family->n, N = family->group_size;
    for (int64_t i = 0; i < n; ++i) {
        const double* a = coords + 3 * i;
        for (int64_t k = 0; k < N; ++k) {
            int32_t* slot = &family->entries[i * N + k];
            if (*slot == -1)
                continue;
            const double* b = coords + 3 * (int64_t)*slot;
            int hit;
            const double da = a[axis] - position, db = b[axis] - position;
            if (kind == 0) {
                hit = da * db < 0;
            } else if (da * db >= 0) {
                hit = 0;
            } else {
                const double t = da / (da - db);
                const double cross = a[sweep_axis] + t * (b[sweep_axis] - a[sweep_axis]);
                hit = cross <= depth;
            }
            if (hit) {
                *slot = -1;
                --family->n_neigh[i];
            }
        }
    }
}

void orc_break_plane(pd_neighbor_list* family, const double* coords, int axis, double position) {
    break_with(family, coords, 0, axis, position, 0, 0);
}

void orc_break_notch(pd_neighbor_list* family, const double* coords, int axis, double position,
                     int sweep_axis, double depth) {
    break_with(family, coords, 1, axis, position, sweep_axis, depth);
}

/* local_damage (formulas.hpp:49-55) via make_snapshot (io.cpp:243-247) */
int orc_damage(const pd_neighbor_list* family, double* phi) {
    for (int64_t i = 0; i < family->n; ++i) {
        const int32_t init = family->initial_n_neigh[i];
        const int32_t cur = family->n_neigh[i];
        if (init > 0) {
            if (cur < 0 || cur > init)
                return fail(PD_E_DOMAIN, "local_damage: current count out of range");
            phi[i] = 1.0 - (double)cur / (double)init;
        } else {
            phi[i] = 0;
        }
    }
    return PD_OK;
}

/* neighborhood_volumes + surface_correction_factors (geometry.cpp:238-283) */
int orc_surface_correction_factors(const double* volumes, const pd_neighbor_list* family,
                                   double v0, double* lambda) {
    if (!(v0 > 0))
        return fail(PD_E_DOMAIN, "surface_correction_factors: V0 must be positive");
    const int64_t n = family->n, N = family->group_size;
    double* nbhd = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        double sum = 0;
        for (int64_t k = 0; k < N; ++k) {
            const int32_t j = family->entries[i * N + k];
            if (j != -1)
                sum += volumes[j];
        }
        nbhd[i] = sum;
    }
    int rc = PD_OK;
    for (int64_t i = 0; i < n && !rc; ++i)
        for (int64_t k = 0; k < N; ++k) {
            const int32_t j = family->entries[i * N + k];
            lambda[i * N + k] = 1;
            if (j == -1)
                continue;
            const double denom = nbhd[i] + nbhd[j];
            if (!(denom > 0)) {
                rc = fail(PD_E_DOMAIN,
                          "surface_correction_factors: zero neighborhood volume for bond %lld-%d",
                          (long long)i, j);
                break;
            }
            lambda[i * N + k] = 2 * v0 / denom;
        }
    free(nbhd);
    return rc;
}

/* stable_timestep_hint (engine.cpp:307-333) */
int orc_stable_timestep_hint(const pd_particles* p, const pd_damage_model* model,
                             const pd_neighbor_list* family, double safety, const double* beta,
                             double* dt_out) {
    const int64_t n = family->n, N = family->group_size;
    double best = INFINITY;
    for (int64_t i = 0; i < n; ++i) {
        double stiffness_sum = 0;
        for (int64_t k = 0; k < N; ++k) {
            const int64_t idx = i * N + k;
            const int32_t j = family->entries[idx];
            if (j == -1)
                continue;
            const double r0 = p->coords[3 * (int64_t)j] - p->coords[3 * i];
            const double r1 = p->coords[3 * (int64_t)j + 1] - p->coords[3 * i + 1];
            const double r2 = p->coords[3 * (int64_t)j + 2] - p->coords[3 * i + 2];
            const pd_law* law =
                family->bond_type_size == 0 ? &model->laws[0] : &model->laws[family->bond_type[idx]];
            double term = law->stiffness * p->volume[j] / sqrt(r0 * r0 + r1 * r1 + r2 * r2);
            if (beta)
                term *= beta[idx];
            stiffness_sum += term;
        }
        if (stiffness_sum > 0) {
            const double cand = sqrt(2 * p->density[i] / stiffness_sum);
            best = cand < best ? cand : best;
        }
    }
    if (!isfinite(best))
        return fail(PD_E_DOMAIN, "stable_timestep_hint: family has no bonds");
    *dt_out = safety * best;
    return PD_OK;
}
