/*
 * pd_b200.h -- C ABI of the B200-native bond-based peridynamics time step.
 *
 * This is the drop-in boundary for the reference engine
 * (/root/reference/proj/include/peridyn/engine.hpp).  Every entry point takes
 * plain pointers and sizes; there are no C++ or torch types in the
 * signatures, no exceptions cross the ABI, and every function returns a
 * status code whose value names the exception type the reference would have
 * thrown (pd_last_error() holds the reference's message text).
 *
 * Descriptor structs mirror the reference's value types field for field:
 *   pd_particles      <- ParticleSet          (types.hpp:52-60)
 *   pd_neighbor_list  <- NeighborList         (types.hpp:66-76)
 *   pd_law            <- DamageLaw            (types.hpp:83-96)
 *   pd_damage_model   <- DamageModel          (types.hpp:99-110)
 *   pd_state          <- SimulationState      (types.hpp:115-122)
 *   pd_ramp           <- RampProfile          (types.hpp:131-142)
 *   pd_boundary       <- BoundaryConditions   (types.hpp:145-155)
 *   pd_corrections    <- Corrections          (types.hpp:161-165)
 *   pd_force_field    <- ForceField           (types.hpp:170-178)
 *   pd_bundle         <- ModelBundle          (engine.hpp:90-98)
 *   pd_options        <- SimulateOptions      (engine.hpp:100-106)
 *   pd_tip_record     <- TipRecord            (engine.hpp:110-114)
 * Arrays are the reference's flat row-major layouts (n x 3 for vectors,
 * n x N for per-slot arrays), so a std::vector's data()/size() pass through
 * unchanged.  A NULL pointer with size 0 means "empty vector".
 */
#ifndef PD_B200_H
#define PD_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PD_ABI_VERSION 1
#define PD_MAX_BREAKPOINTS 32 /* per law (the reference allows any count, types.hpp:86); the fast variant takes <= 8 */
#define PD_MAX_LAWS 256      /* bond_type is uint8 (types.hpp:71) */

/* Status codes.  Each maps to the exception type the reference throws. */
enum {
    PD_OK = 0,
    PD_E_INVALID_ARGUMENT = 1, /* std::invalid_argument (size mismatches, engine.cpp:34-46) */
    PD_E_DOMAIN = 2,           /* std::domain_error (dt <= 0, rho <= 0, engine.cpp:177-190) */
    PD_E_RUNTIME = 3,          /* std::runtime_error (non-finite u at step K, engine.cpp:23-28) */
    PD_E_CUDA = 4,             /* CUDA failure (no reference counterpart) */
    PD_E_NO_DEVICE = 5         /* no sm_100 device visible */
};

/* KernelVariant (engine.hpp:15) plus the B200 fast path.
 * PD_BOND_PARALLEL: fp64, bitwise equal to compute_forces_bond_parallel.
 * PD_NODE_PARALLEL: fp64, bitwise equal to compute_forces_node_parallel.
 * PD_FAST:          fp64 state/integration, fp32 bond arithmetic; tolerance
 *                   documented in DESIGN.md (not bitwise). */
enum { PD_BOND_PARALLEL = 0, PD_NODE_PARALLEL = 1, PD_FAST = 2 };

/* IntegratorKind (engine.hpp:87) */
enum { PD_VELOCITY_VERLET = 0, PD_EULER = 1, PD_EULER_CROMER = 2 };

/* BCKind (types.hpp:127) */
enum { PD_BC_FREE = 0, PD_BC_DISPLACEMENT = 1, PD_BC_FORCE = 2 };

/* RampProfile::Kind (types.hpp:132) */
enum { PD_RAMP_CONSTANT = 0, PD_RAMP_LINEAR = 1, PD_RAMP_QUINTIC = 2 };

typedef struct pd_particles {
    int64_t n;             /* volume.size() */
    const double* coords;  /* n x 3 */
    int64_t coords_size;   /* coords.size() */
    const double* volume;  /* n */
    const double* density; /* n */
    int64_t density_size;  /* density.size() */
} pd_particles;

typedef struct pd_neighbor_list {
    int64_t n;                      /* n_neigh.size() */
    int64_t group_size;             /* N, a power of two */
    int32_t* entries;               /* n x N, -1 = broken or padding (mutated by the force pass) */
    int32_t* n_neigh;               /* n (mutated by the force pass) */
    const int32_t* initial_n_neigh; /* n */
    const uint8_t* bond_type;       /* n x N or NULL */
    int64_t bond_type_size;         /* bond_type.size() */
    double horizon;
} pd_neighbor_list;

typedef struct pd_law {
    double stiffness;     /* micromodulus c */
    int32_t n_breakpoints; /* >= 1; 1 = PMB */
    double breakpoints[PD_MAX_BREAKPOINTS];
    double forces[PD_MAX_BREAKPOINTS];
} pd_law;

typedef struct pd_damage_model {
    const pd_law* laws;
    int32_t n_laws;
    double damping; /* eta */
} pd_damage_model;

typedef struct pd_corrections {
    const double* lambda; /* n x N or NULL */
    int64_t lambda_size;
    const double* beta; /* n x N or NULL */
    int64_t beta_size;
    const uint8_t* no_failure; /* n or NULL */
    int64_t no_failure_size;
} pd_corrections;

typedef struct pd_state {
    double* u; /* n x 3 */
    double* v; /* n x 3 */
    double* a; /* n x 3 */
    int64_t step;
    pd_neighbor_list connectivity;
    double* bond_history; /* n x N or NULL */
    int64_t bond_history_size;
} pd_state;

typedef struct pd_force_field {
    double* body_force;     /* n x 3 (written) */
    double* external_force; /* n x 3 (read by integrators; preserved by the force pass) */
} pd_force_field;

typedef struct pd_ramp {
    int32_t kind;
    int64_t rise_steps;
    double target_scale;
} pd_ramp;

typedef struct pd_boundary {
    const uint8_t* kind; /* n x 3, PD_BC_* */
    int64_t kind_size;
    const double* magnitude; /* n x 3 */
    int64_t magnitude_size;
    const uint8_t* ramp_id; /* n x 3 */
    int64_t ramp_id_size;
    const pd_ramp* ramps;
    int32_t n_ramps;
    const uint8_t* no_failure; /* n */
    int64_t no_failure_size;
    /* tip_sets (std::map order): set k holds tip_nodes[tip_offsets[k] .. tip_offsets[k+1]) */
    int32_t n_tip_sets;
    const int64_t* tip_offsets;
    const int64_t* tip_nodes;
} pd_boundary;

typedef struct pd_bundle {
    pd_particles particles;
    pd_damage_model model;
    pd_corrections corrections;
    pd_boundary bc;
    double dt;
} pd_bundle;

typedef struct pd_options {
    int64_t steps;
    int64_t write_every; /* 0 = no periodic writes */
    int64_t first_step;
    int32_t integrator; /* PD_VELOCITY_VERLET | PD_EULER | PD_EULER_CROMER */
    int32_t variant;    /* PD_BOND_PARALLEL | PD_NODE_PARALLEL | PD_FAST */
} pd_options;

typedef struct pd_tip_record {
    int64_t step;
    double mean_u[3], mean_v[3], mean_a[3];
    double body_force_sum[3], external_force_sum[3];
} pd_tip_record;

/* WriteHook (engine.hpp:118).  Called at every write step with host views of
 * the state and forces; a nonzero return aborts the run with PD_E_RUNTIME. */
typedef int (*pd_write_hook)(void* user, const pd_state* state, const pd_force_field* forces);

/* ---- library ---------------------------------------------------------- */

int pd_abi_version(void);
/* Message of the last failing call on this thread ("" after success). */
const char* pd_last_error(void);
/* Number of usable sm_100 devices (0 on a machine without a B200). */
int pd_device_count(void);
/* Device blocks of destroyed contexts are kept mapped for reuse by the next
 * context of the same size (repeated simulate() calls, calibration loops);
 * this returns them to the driver.  PD_NO_BLOCK_CACHE=1 disables the cache. */
void pd_release_cached_memory(void);

/* ---- one-shot drop-ins (host buffers in, host buffers out) ------------ */

/* compute_forces(variant, state, particles, model, corrections, out)
 * (engine.hpp:35-36, engine.cpp:163-169).  Mutates state->connectivity.entries,
 * n_neigh and bond_history exactly as the reference; writes out->body_force;
 * out->external_force is not touched. */
int pd_compute_forces(int32_t variant, pd_state* state, const pd_particles* particles,
                      const pd_damage_model* model, const pd_corrections* corrections,
                      pd_force_field* out);

/* simulate(bundle, state, options, on_write) (engine.hpp:128-129,
 * engine.cpp:374-425).  The caller sizes state->bond_history to n x N when the
 * model needs history (the reference resizes it itself, engine.cpp:382-384).
 * Tip records of every write step are appended to tips_out in
 * (write step, tip set) order; n_tips_out receives the count.  When
 * tips_capacity is too small the run fails with PD_E_INVALID_ARGUMENT before
 * any work. */
int pd_simulate(const pd_bundle* bundle, pd_state* state, const pd_options* options,
                pd_write_hook on_write, void* user, pd_tip_record* tips_out,
                int64_t tips_capacity, int64_t* n_tips_out);

/* K independent simulate() calls run concurrently on one GPU: the
 * calibration / UQ outer loop (calibrate.cpp:116-218 runs hundreds of short
 * simulations of small models).  Each model gets its own context and stream
 * and a pool of `threads` host threads (0 = up to 8) drives them, so kernels
 * of different models share the SMs.  Tip records of model m go to
 * tips_out[tips_offset[m] .. tips_offset[m+1]) (both may be NULL when no
 * model records tips); status[m] is model m's code; the return value is the
 * first failing code (its message names the model). */
int pd_simulate_batch(int32_t k, const pd_bundle* bundles, pd_state* states,
                      const pd_options* options, pd_tip_record* tips_out,
                      const int64_t* tips_offset, int64_t* n_tips_out, int32_t* status,
                      int32_t threads);

/* local_damage over all nodes from a host connectivity (formulas.hpp:49-55,
 * io.cpp:243-247): phi_i = 1 - n_neigh_i / initial_i, 0 when initial_i == 0. */
int pd_damage(const pd_neighbor_list* family, double* phi_out);

/* ---- family construction on the device (geometry.cpp:97-211) ---------- */

typedef struct pd_family pd_family;

/* build_family(coords, horizon, grid_hint) (geometry.hpp:60-62): rows sorted
 * ascending, padded with -1 to N = bit_ceil(max family size); identical to the
 * reference's cell-list result.  grid_hint = {ox, oy, oz, spacing, nx, ny, nz}
 * or NULL.  The rows stay on the device until pd_family_download. */
int pd_build_family(const double* coords, int64_t n, double horizon, const double* grid_hint,
                    pd_family** out, int64_t* group_size_out);
/* entries: n x N; n_neigh and initial_n_neigh: n (both = family sizes). */
int pd_family_download(pd_family* family, int32_t* entries, int32_t* n_neigh,
                       int32_t* initial_n_neigh);
void pd_family_free(pd_family* family);

/* ---- the reference's stand-alone integrators and boundary passes -------
 * (engine.hpp:38-78, engine.cpp:187-305) on the device, over host buffers:
 * each call reads and writes the same arrays as the reference function, in
 * its expression order, so hand-composed steps (test_engine.cpp:196-357)
 * give the reference's bits.  Errors: dt <= 0 -> PD_E_DOMAIN "<fn>: dt must
 * be positive"; density size -> PD_E_INVALID_ARGUMENT, density <= 0 ->
 * PD_E_DOMAIN (check_density, engine.cpp:177-183). */
int pd_verlet_drift(pd_state* state, double dt);
int pd_verlet_kick(pd_state* state, const pd_force_field* forces, double dt, double damping,
                   const double* density, int64_t density_size);
int pd_step_euler(pd_state* state, const pd_force_field* forces, double dt,
                  const double* density, int64_t density_size);
int pd_step_euler_cromer(pd_state* state, const pd_force_field* forces, double dt,
                         const double* density, int64_t density_size);
/* ForceEval (engine.hpp:56): fill forces->body_force for the state's u;
 * nonzero = failure (the step fails with PD_E_RUNTIME). */
typedef int (*pd_force_eval)(void* user, pd_state* state, pd_force_field* forces);
/* step_velocity_verlet (engine.cpp:254-260): drift, forces(state, scratch),
 * kick, ++step. */
int pd_step_velocity_verlet(pd_state* state, pd_force_eval forces, void* user,
                            pd_force_field* scratch, double dt, double damping,
                            const double* density, int64_t density_size);
int pd_apply_displacement_positions(pd_state* state, const pd_boundary* bc, int64_t step);
int pd_apply_displacement_kinematics(pd_state* state, const pd_boundary* bc, int64_t step,
                                     double dt);
/* adds force-BC densities into out->external_force (n nodes); no clearing */
int pd_accumulate_external_force(const pd_boundary* bc, int64_t step, pd_force_field* out,
                                 int64_t n);
/* apply_boundary: bc.validate, positions, kinematics, external force */
int pd_apply_boundary(pd_state* state, const pd_boundary* bc, int64_t step, double dt,
                      pd_force_field* out);

/* ---- setup-time family operations on the device (geometry.cpp) -------- */

/* A rule-table BondClassifier (geometry.hpp:45-54, applied in pack_rows,
 * geometry.cpp:131-161): each node's class is the class of the LAST region
 * rule containing it (default_class when none does); the bond type of slot
 * (i, j) is type_table[class_i * n_classes + class_j] (symmetric, as the
 * reference requires of a classifier).  Padding slots keep type 0. */
enum { PD_REGION_BOX = 0, PD_REGION_CYLINDER = 1 };
typedef struct pd_region {
    int32_t kind;   /* PD_REGION_BOX: lo <= x <= hi on every axis (inclusive) */
    int32_t axis;   /* PD_REGION_CYLINDER: axis 0/1/2, lo[axis] <= x[axis] <= hi[axis] and */
    int32_t cls;    /* (x[b0] - c[0])^2 + (x[b1] - c[1])^2 <= radius^2, b0 < b1 the other axes */
    int32_t pad;
    double lo[3];
    double hi[3];
    double c[2];
    double radius;
} pd_region;
typedef struct pd_classifier {
    int32_t n_classes;           /* 1..256 */
    int32_t default_class;
    int32_t n_regions;
    int32_t pad;
    const pd_region* regions;
    const uint8_t* type_table;   /* n_classes x n_classes */
} pd_classifier;

/* bond_type (n x N) of a family under a rule-table classifier. */
int pd_classify_bonds(const double* coords, const pd_neighbor_list* family,
                      const pd_classifier* classifier, uint8_t* bond_type_out);
/* neighborhood_volumes (geometry.cpp:238-252): per node the in-order sum of
 * its live members' volumes. */
int pd_neighborhood_volumes(const double* volumes, const pd_neighbor_list* family, double* out);
/* surface_correction_factors (geometry.cpp:263-283): lambda_ij = 2 V0 /
 * (V_i + V_j) per live slot, 1 on padding; domain errors as the reference. */
int pd_surface_correction_factors(const double* volumes, const pd_neighbor_list* family,
                                  double v0, double* lambda_out);

/* break_initial_bonds (geometry.cpp:285-306) with plane_crossing_predicate
 * (:300-305) or notch_predicate (:308-319): matching slots become -1 and
 * n_neigh drops; initial_n_neigh is untouched. */
enum { PD_PREDICATE_PLANE = 0, PD_PREDICATE_NOTCH = 1 };
typedef struct pd_bond_predicate {
    int32_t kind;
    int32_t axis;
    int32_t sweep_axis;  /* notch only */
    int32_t pad;
    double position;
    double depth;        /* notch only: crossing point along sweep_axis <= depth */
} pd_bond_predicate;
int pd_break_initial_bonds(pd_neighbor_list* family, const double* coords,
                           const pd_bond_predicate* predicate);

/* ---- device-resident context ------------------------------------------ */

typedef struct pd_ctx pd_ctx;

/* Field selectors for pd_ctx_download / write hooks (bitmask). */
enum {
    PD_FIELD_U = 1,
    PD_FIELD_V = 2,
    PD_FIELD_A = 4,
    PD_FIELD_CONNECTIVITY = 8, /* entries + n_neigh */
    PD_FIELD_HISTORY = 16,
    PD_FIELD_FORCES = 32, /* body_force + external_force of the last step */
    PD_FIELD_ALL = 63
};

int pd_ctx_create(int device, pd_ctx** out);
void pd_ctx_destroy(pd_ctx* ctx);

/* Upload the fixed model and an initial state; validates like
 * ModelBundle::validate (engine.cpp:335-341) and NeighborList::validate. */
int pd_ctx_upload(pd_ctx* ctx, const pd_bundle* bundle, const pd_state* state, int32_t variant);

/* Advance the resident state (simulate() semantics, without host copies
 * except at write steps when a hook is given; fields = PD_FIELD_* the hook
 * needs). */
int pd_ctx_run(pd_ctx* ctx, const pd_options* options, pd_write_hook on_write, void* user,
               int32_t hook_fields, pd_tip_record* tips_out, int64_t tips_capacity,
               int64_t* n_tips_out);

/* One force pass on the resident state (compute_forces semantics). */
int pd_ctx_compute_forces(pd_ctx* ctx);

/* Copy the resident state back into host arrays (only the selected fields;
 * pointers of unselected fields may be NULL). */
int pd_ctx_download(pd_ctx* ctx, pd_state* state, pd_force_field* forces, int32_t fields);

/* Damage phi of every node from the resident alive mask (K3). */
int pd_ctx_damage(pd_ctx* ctx, double* phi_out);

/* The cudaStream_t every kernel of this context is launched on, so callers
 * can bracket a run with events on the right stream. */
void* pd_ctx_stream(pd_ctx* ctx);

/* Kernel launches issued by this context since creation. */
int64_t pd_ctx_launch_count(pd_ctx* ctx);

/* Live directed bonds in the resident alive mask (sum of n_neigh). */
int64_t pd_ctx_live_bonds(pd_ctx* ctx);

/* Which step kernel the uploaded model runs on. */
enum {
    PD_LAYOUT_EXACT = 0,   /* PD_BOND_PARALLEL / PD_NODE_PARALLEL: padded rows + alive bits */
    PD_LAYOUT_TILES = 1,   /* PD_FAST, any mesh: brick tiles, compact 16-bit slot offsets */
    PD_LAYOUT_LATTICE = 2  /* PD_FAST on a lattice: implicit 122-offset pattern + live mask */
};
int pd_ctx_layout(pd_ctx* ctx);
/* The step kernel instantiation the last step launched, e.g.
 * "lattice_step_kernel<1,8,3,0,0>" (MODE, brick depth, CTAs/SM, BC, NF);
 * "" before the first step.  The string is static. */
const char* pd_ctx_kernel(pd_ctx* ctx);

/* ---- binary containers (io.cpp:297-564), byte-compatible with the reference
 * PDST = restart state (save_state/load_state), PDNL = family cache
 * (save_cache/load_cache).  Readers validate like the reference and report
 * its IoError text ("<path>: <what>") with PD_E_RUNTIME. ---------------- */
typedef struct pd_file_header {
    int64_t n;
    int64_t group_size;
    int64_t step; /* PDST only */
    double horizon;
    int32_t has_bond_type, has_history, has_lambda, has_beta;
} pd_file_header;

int pd_save_state(const pd_state* state, const char* path);
int pd_state_file_header(const char* path, pd_file_header* out);
/* Fills caller arrays sized from the header (bond_type / history may be NULL
 * to skip those sections). */
int pd_load_state(const char* path, pd_state* state);
int pd_save_cache(const pd_neighbor_list* family, const pd_corrections* corrections,
                  const char* path);
int pd_cache_file_header(const char* path, pd_file_header* out);
int pd_load_cache(const char* path, pd_neighbor_list* family, pd_corrections* corrections);
/* save_state of the resident state, streamed from device memory (no host
 * copy of the state); one-GPU contexts only. */
int pd_ctx_save_state(pd_ctx* ctx, const char* path);

/* write_snapshot(make_snapshot(state, particles)) (io.cpp:235-269): the ASCII
 * pdsnap file, byte for byte.  Lines are formatted by several host threads. */
int pd_write_snapshot(const pd_state* state, const pd_particles* particles, const char* path);
/* The same file from the resident state (one-GPU contexts). */
int pd_ctx_write_snapshot(pd_ctx* ctx, const char* path);
/* Snapshots during pd_ctx_run: every `every` steps (absolute step count, like
 * write_every) the resident fields are copied on the device and a host thread
 * downloads, formats and writes `pattern` (printf with the step as %lld)
 * while the GPU keeps stepping.  every = 0 turns it off. */
int pd_ctx_snapshot_every(pd_ctx* ctx, int64_t every, const char* pattern);

/* ---- multi-GPU z-slabs (no reference counterpart: the reference is one
 * process) ------------------------------------------------
 *
 * One pd_ctx per GPU (per rank) holds that rank's LOCAL model: its owned nodes
 * plus a ghost layer one horizon deep, in a numbering where the owned nodes
 * are the contiguous range [own_begin, own_end).  Rows of owned nodes are the
 * global rows with their slot order kept (so parity mode stays bitwise equal
 * to one GPU); ghost rows are ignored.  Each time step the fused step kernel
 * stores the new displacement of every owned node that is a ghost on a
 * neighbouring rank straight into that rank's u buffer over NVLink (peer
 * stores), then a one-thread sync kernel publishes the step (and the rank's
 * non-finite flag) to every rank and waits until all ranks have published it.
 * Host code only exchanges the pd_peer_handle records once (any transport,
 * e.g. torch.distributed). */
#define PD_MAX_RANKS 16

typedef struct pd_peer_handle {
    int32_t device; /* CUDA device ordinal in the owning process */
    int32_t pid;    /* owning process id (same pid: raw pointers, else CUDA IPC) */
    uint8_t ipc_u0[64], ipc_u1[64], ipc_sync[64]; /* cudaIpcMemHandle_t */
    uint64_t u0, u1, sync; /* raw device pointers in the owning process */
} pd_peer_handle;

/* pd_ctx_upload for a rank's local model; only [own_begin, own_end) is
 * integrated.  Requires variant PD_BOND_PARALLEL, PD_NODE_PARALLEL or PD_FAST. */
int pd_ctx_upload_part(pd_ctx* ctx, const pd_bundle* bundle, const pd_state* state,
                       int32_t variant, int64_t own_begin, int64_t own_end);
/* Device row index of local nodes (PD_FAST renumbers nodes into bricks). */
int pd_ctx_internal_index(pd_ctx* ctx, const int64_t* local, int64_t count, int64_t* out);
int pd_ctx_export(pd_ctx* ctx, pd_peer_handle* out);
/* Join a world of `world` ranks (peers[world], this rank's entry ignored).
 * send_lo / send_hi (length n_local, indexed by LOCAL node id): the device row
 * index on rank lo / hi of each owned node that is a ghost there, else -1
 * (lo or hi = -1 when there is no such neighbour). */
int pd_ctx_connect(pd_ctx* ctx, int32_t rank, int32_t world, const pd_peer_handle* peers,
                   int32_t lo, int32_t hi, const int64_t* send_lo, const int64_t* send_hi);
/* u, v, a of the listed local nodes, plus body/external force x V of the
 * last write step, 15 doubles per node (multi-rank tip records). */
int pd_ctx_node_values(pd_ctx* ctx, const int64_t* local, int64_t count, double* out);

#ifdef __cplusplus
}
#endif

#endif /* PD_B200_H */
