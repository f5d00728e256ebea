/*
 * ignis_b200.h — C ABI of the B200-native RHS + SSP-RK3 path.
 *
 * Drop-in boundary for the reference's C++ `ignis::Simulation`
 * (/root/reference/proj/include/ignis/solver.hpp:53-853).  Every entry point
 * below replaces one public member of that class (cited per function); the
 * configuration structs are POD restatements of the reference's config types.
 * No torch or CUDA types appear in any signature: plain pointers, sizes and
 * status codes.  One context per GPU (or per ensemble member).
 *
 * Array convention (host side, identical to ignis::Field::raw(),
 * field.hpp:45-47): each field is one contiguous padded buffer of
 * (nx+2g)*(ny+2g) doubles, row-major, i fastest, element (i,j) at
 * (j+g)*(nx+2g)+(i+g).  Multi-component arguments are the component buffers
 * concatenated in component order [rhoY_0..rhoY_{ns-1}, rho u, rho v, E]
 * (flux.hpp:13), i.e. component c starts at c*(nx+2g)*(ny+2g).
 *
 * Errors: every call returns an ign_status.  The reference's exception
 * types (errors.hpp:10-47) map 1:1 onto IGN_CONFIG_ERROR ... IGN_USAGE_ERROR;
 * ign_last_error() returns the message and, for IGN_STEP_FAILURE, the
 * (stage, i, j) the reference's StepFailure carries.
 */
#ifndef IGNIS_B200_H
#define IGNIS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGN_ABI_VERSION 3
#define IGN_MAX_SPECIES 8   /* thermo.hpp:16 kMaxSpecies */
#define IGN_MAX_COMP 11     /* flux.hpp:14 kMaxComp */
#define IGN_MAX_PIECES 4    /* polynomial ranges per species */
#define IGN_MAX_SEGMENTS 4  /* inflow segments per edge */
#define IGN_NAME_LEN 16

typedef enum {
    IGN_OK = 0,
    IGN_CONFIG_ERROR = 1,   /* ignis::ConfigError   errors.hpp:11 */
    IGN_STATE_ERROR = 2,    /* ignis::StateError    errors.hpp:17 */
    IGN_NUMERICS_ERROR = 3, /* ignis::NumericsError errors.hpp:23 */
    IGN_STEP_FAILURE = 4,   /* ignis::StepFailure   errors.hpp:29 */
    IGN_FORMAT_ERROR = 5,   /* ignis::FormatError   errors.hpp:39 */
    IGN_USAGE_ERROR = 6,    /* ignis::UsageError    errors.hpp:45 */
    IGN_CUDA_ERROR = 7,     /* device/runtime failure (no reference analogue) */
    IGN_INTERNAL_ERROR = 8
} ign_status;

/* thermo.hpp:23-39 ThermoPiece */
typedef struct {
    double t_lo, t_hi;
    double cm2, cm1, c0, c1, c2, c3, c4, b;
} ign_thermo_piece;

/* thermo.hpp:41-58 SpeciesData */
typedef struct {
    char name[IGN_NAME_LEN];
    double W, mu_ref, t_ref, n_exp;
    int32_t npieces;
    int32_t _pad;
    ign_thermo_piece pieces[IGN_MAX_PIECES];
} ign_species;

/* thermo.hpp:66-104 MixtureModel; mode 0 = CaloricallyPerfect, 1 = MultiSpecies */
typedef struct {
    int32_t mode;
    int32_t ns;
    double R, Le, Pr;
    ign_species species[IGN_MAX_SPECIES];
} ign_mixture;

/* reconstruction.hpp:12-40 SchemeConfig.
 * scheme: 0 = WENO3Z, 1 = TENO6; split: 0 = Componentwise, 1 = Characteristic;
 * metrics: 0 = Scheme, 1 = AnalyticSkew, 2 = Central2 */
typedef struct {
    int32_t scheme;
    int32_t split;
    double teno_ct, eps, cfl;
    int32_t metrics;
    int32_t _pad;
} ign_scheme;

/* boundary.hpp:25-32 InflowSegment */
typedef struct {
    double lo, hi, u, v, T;
    double Y[IGN_MAX_SPECIES];
} ign_inflow_segment;

/* boundary.hpp:16-41 BCType/EdgeSpec.
 * type: 0 Periodic, 1 NoslipIsothermal, 2 NoslipAdiabatic, 3 Inflow, 4 Outflow */
typedef struct {
    int32_t type;
    int32_t nseg;
    double T_wall;
    ign_inflow_segment seg[IGN_MAX_SEGMENTS];
    double smooth_width, p_target, sigma_out;
} ign_edge;

/* boundary.hpp:45-89 BoundarySpec */
typedef struct {
    ign_edge left, right, bottom, top;
} ign_bc;

/* chemistry.hpp:16-24 ReactionMechanism (present = 0 means std::nullopt) */
typedef struct {
    int32_t present;
    int32_t i_fuel, i_ox, i_co2, i_h2o;
    int32_t _pad;
    double A, Ta, a, b, T_cutoff;
    double nu[IGN_MAX_SPECIES];
} ign_mechanism;

/* laser.hpp:18-46 LaserParams + ShapedProfile (present = 0 means nullopt).
 * kernel: 0 = Gaussian, 1 = Shaped */
typedef struct {
    int32_t present;
    int32_t kernel;
    double energy, sigma_r, sigma_t, x0, y0, t0, edot_rate;
    double lobe_sep, width_up, width_down, amp_down, width_radial;
    /* 3D extension (no reference path): zmode 0 = the reference's 2D kernel
     * on every z plane (a line source along z; the z-extrusion check),
     * 1 = a point kernel at (x0, y0, z0): Gaussian with r^2 over (x, y, z) and
     * the 3D normalisation E / ((2 pi)^2 sigma_r^3 sigma_t), so E is the
     * deposited energy; shaped with the radial factor over (y, z). */
    double z0;
    int32_t zmode;
    int32_t _pad;
} ign_laser;

/* solver.hpp:29-35 IntegratorConfig */
typedef struct {
    double fixed_dt, t_end;
    int64_t max_iter;
    int32_t chem_dt_limit;
    int32_t _pad;
    double chem_dt_factor;
} ign_integrator;

/* Everything Simulation::init (solver.hpp:82-101) and its public knobs
 * (solver.hpp:55-76) receive.  The mesh is build_uniform (mesh.hpp:48-77),
 * optionally followed by apply_skew(skew_beta) (mesh.hpp:92-117). */
typedef struct {
    int32_t abi_version;         /* must be IGN_ABI_VERSION */
    int32_t nx, ny, g;           /* g = 3 (mesh.hpp:14) */
    double lx, ly, center_x, center_y;
    int32_t periodic_x, periodic_y;
    int32_t apply_skew;          /* 1: apply_skew(mesh, skew_beta) */
    int32_t metric_mode;         /* -1: Simulation::metric_mode_for(scheme);
                                    0 Central2, 1 Order4, 2 Order6, 3 AnalyticSkew */
    double skew_beta;
    ign_mixture mix;
    ign_scheme scheme;
    ign_bc bc;
    ign_mechanism mech;
    ign_laser laser;
    int32_t viscous;
    int32_t partitions;          /* ThreadTeam workers (CPU oracle only) */
    ign_integrator integ;
    int32_t device;              /* CUDA device ordinal */
    /* Slab decomposition along y (rows) across GPUs: ny is the
     * GLOBAL row count; this context owns slab slab_rank of slab_count
     * (ThreadTeam's block split, thread_team.hpp:63-69).  0 or 1 = whole mesh. */
    int32_t slab_count;
    int32_t slab_rank;
    /* 3D extension (BASELINE configs[1]; no reference path — SURVEY §0):
     * nz > 0 extrudes the (x, y) mesh uniformly over lz in z.  Component order
     * then [rhoY_s, rho u, rho v, rho w, E]; primitive cache rho,u,v,w,p,T,c,Y;
     * the x / y edges take the reference's rules on every z plane, z is
     * periodic (periodic_z = 1) or bounded by zlo / zhi below.  With
     * slab_count > 1, 3D contexts split z. */
    int32_t nz;
    int32_t periodic_z;
    int32_t _pad;
    double lz, center_z;
    /* A hand-built ignis::Mesh (mesh.hpp:23-42): its padded node coordinates
     * mesh.x, mesh.y ((nx+2g)(ny+2g) doubles each, field.hpp layout, GLOBAL
     * rows for slabs), read during ign_create only.  NULL = build_uniform
     * (mesh.hpp:48-77) [+ apply_skew].  lx, ly, center_* and the periodic
     * flags stay the Mesh's own fields (inflow profiles and the laser use the
     * computational coordinates xi, eta, as the reference does); the metrics are
     * compute_metrics of these coordinates (metrics.hpp:73-118). */
    const double* mesh_x;
    const double* mesh_y;
    /* 3D extension: the z edges (back = k < 0, front = k >= nz) when
     * periodic_z = 0 — no-slip walls (isothermal / adiabatic) or outflow, the
     * reference's y-edge rules with w the wall-normal velocity; filled after
     * the x and y edges, over the full padded (x, y) plane.  Ignored (must be
     * periodic) when periodic_z = 1; inflow is not supported on z edges. */
    ign_edge zlo, zhi;
} ign_config;

/* errors.hpp:29-35 StepFailure payload + message; k is the z plane of a 3D
 * failure (0 in 2D — the reference's payload is (stage, i, j)) */
typedef struct {
    int32_t status;
    int32_t stage, i, j, k;
    char msg[256];
} ign_error;

/* solver.hpp:114-128: primitive point of set_initial_condition's callback */
typedef struct {
    double rho, u, v, p, T;
    double Y[IGN_MAX_SPECIES];
} ign_prim_point;

typedef void (*ign_ic_fn)(double x, double y, void* user, ign_prim_point* out);
/* advance's step_hook (solver.hpp:336,347); return nonzero to stop. */
typedef int (*ign_step_hook)(void* ctx, void* user);

typedef struct ign_context ign_context;

/* ---- lifecycle -------------------------------------------------------- */
uint64_t ign_config_size(void); /* sizeof(ign_config), ABI self-check */
/* Simulation::init (solver.hpp:82-101) incl. scheme/bc validation */
int ign_create(const ign_config* cfg, ign_context** out);
void ign_destroy(ign_context* ctx);
int ign_last_error(const ign_context* ctx, ign_error* err);
int ign_dims(const ign_context* ctx, int32_t* nx, int32_t* ny, int32_t* g,
             int32_t* ns);
/* 3D extension: this context's cells in z (0 for the reference's 2D path),
 * its first global z cell k0 and the global count (z-slabs: nz < nz_glob).
 * In 3D the padded planes are (nx+2g)(ny+2g)(nz+2g), k slowest;
 * set_initial_primitives takes rho,u,v,w,T,Y_s and get_cache returns
 * rho,u,v,w,p,T,c,Y_s.  Any pointer may be NULL. */
int ign_dims3(const ign_context* ctx, int32_t* nz, int32_t* k0, int32_t* nz_glob);

/* ---- setup / host mirrors --------------------------------------------- */
/* mesh.x/mesh.y padded arrays (mesh.hpp:33-34) */
int ign_get_mesh(const ign_context* ctx, double* x, double* y);
/* which 0: met (solver.hpp:56), 1: met_v (solver.hpp:57); out = 5 padded
 * fields [jac, m_xi_x, m_xi_y, m_eta_x, m_eta_y] (metrics.hpp:28-35) */
int ign_get_metrics(const ign_context* ctx, int which, double* out);
/* Simulation::set_initial_condition (solver.hpp:115-128), callback form */
int ign_set_initial_condition(ign_context* ctx, ign_ic_fn fn, void* user);
/* Same, from padded primitive arrays rho,u,v,T then Y_0..Y_{ns-1}
 * ((4+ns) fields); p is not used by conservative_from_primitives. */
int ign_set_initial_primitives(ign_context* ctx, const double* prim);
/* Direct Ut write (nc fields) plus optional primitive T cache (1 field,
 * NULL keeps the current cache). Mirrors mutating sim.Ut / sim.T. */
int ign_set_state(ign_context* ctx, const double* Ut, const double* Tcache);
int ign_get_state(ign_context* ctx, double* Ut);
/* Primitive cache (solver.hpp:79-80): rho,u,v,p,T,c then Y_s ((6+ns) fields) */
int ign_get_cache(ign_context* ctx, double* prim);
int ign_get_time(const ign_context* ctx, double* time, int64_t* iter);
int ign_set_time(ign_context* ctx, double time, int64_t iter);
int ign_set_integrator(ign_context* ctx, const ign_integrator* integ);

/* ---- the hot path ----------------------------------------------------- */
int ign_refill_ghosts(ign_context* ctx);                 /* solver.hpp:144 */
int ign_refresh_primitives(ign_context* ctx, int stage); /* solver.hpp:148-177 */
int ign_prepare_stage(ign_context* ctx, int stage);      /* solver.hpp:422-425 */
/* solver.hpp:185-232; rhs = nc padded fields (interior written, ghosts 0);
 * rhs may be NULL (result stays on the device). */
int ign_compute_rhs(ign_context* ctx, double t_stage, int stage, double* rhs);
int ign_stable_dt(ign_context* ctx, double* dt);          /* solver.hpp:240-299 */
int ign_rk3_step(ign_context* ctx, double dt);            /* solver.hpp:304-332 */
int ign_advance(ign_context* ctx, ign_step_hook hook, void* user); /* :336-349 */
/* n steps of rk3_step(dt) with no host round trip in between (fixed dt). */
int ign_rk3_steps(ign_context* ctx, double dt, int64_t nsteps);

/* ---- diagnostics ------------------------------------------------------ */
int ign_conserved_totals(ign_context* ctx, double* tot);  /* solver.hpp:411-418 */
int ign_product_mole_fraction(ign_context* ctx, double* out); /* :387-407 */
int ign_last_clip(const ign_context* ctx, double* clip);  /* solver.hpp:75 */
/* How conserved_totals / product_mole_fraction (and the trace advance()
 * samples) reduce: IGN_DIAG_DEVICE (default) = deterministic fixed-shape tree
 * on the device, no field download, within ~1e-15 sum|x| of the reference's
 * serial sum; IGN_DIAG_REFERENCE = the reference's serial left fold
 * (solver.hpp:387-418) on the host, bitwise.  Slab groups read the lead's. */
#define IGN_DIAG_DEVICE 0
#define IGN_DIAG_REFERENCE 1
int ign_set_diagnostics(ign_context* ctx, int mode);

/* ---- host-only helpers (no device needed; used by the CPU tests) ------- */
/* compute_metrics over the configured mesh: which 0 = inviscid set, 1 = Central2 */
int ign_host_metrics(const ign_config* cfg, int which, double* out,
                     ign_error* err);
int ign_host_mesh(const ign_config* cfg, double* x, double* y, ign_error* err);

/* ---- device statistics (bench evidence) -------------------------------- */
/* Number of kernels this context has launched since creation. */
int64_t ign_kernel_launches(const ign_context* ctx);

/* Live per-kernel-class device time: CUDA events recorded on the context's
 * stream around every launch of a class while enabled (enable resets). */
#define IGN_PROF_CLASSES 8
#define IGN_PROF_BC 0       /* ghost fill (x+y passes)           */
#define IGN_PROF_PRIM 1     /* primitive cache / Newton T solve  */
#define IGN_PROF_FACES 2    /* inviscid faces, every direction   */
#define IGN_PROF_VISC 3     /* viscous node fluxes               */
#define IGN_PROF_ASSEMBLE 4 /* RHS assembly + RK update + clip   */
#define IGN_PROF_DT 5       /* stable_dt reduction               */
int ign_profile_enable(ign_context* ctx, int on);
int ign_profile_read(ign_context* ctx, double* ms, int64_t* counts);
/* The cudaStream_t every kernel of this context runs on (for external events). */
void* ign_stream_handle(const ign_context* ctx);

/* Measured FP64 FMA peak of a device: a DFMA-chain kernel over every SM
 * (2 flops per FMA); the roofline denominator of the FP64-bound path. */
int ign_probe_fp64_peak(int device, double* tflops);

/* Red-zone guard (memory-safety check in place of compute-sanitizer, which
 * the GPU pool does not run).  With IGN_GUARD=1 in the environment every
 * device buffer a context allocates gets 32 KB of signalling-NaN canary on
 * each side; frees and this call scan them.  *enabled = guard mode on,
 * *checked = guarded buffers scanned so far (freed + live on the current
 * device), *corrupted = canary words found overwritten (0 = no out-of-bounds
 * write seen).  No reference counterpart. */
int ign_guard_status(int* enabled, unsigned long long* checked, unsigned long long* corrupted);
/* Detector self-test: writes one word past the end and one before the start
 * of a guarded scratch buffer; *detected = canary words the scan saw changed (2). */
int ign_guard_selftest(int device, unsigned long long* detected);

/* ---- multi-GPU slabs --------------------------------------- */
/* One process per GPU: rank 0 creates an NCCL unique id, every rank passes it
 * to ign_attach_nccl with its slab config (slab_count/slab_rank).  Halo rows
 * (g rows of every component) then travel by ncclSend/ncclRecv between the
 * x- and y-edge ghost passes of every prepare_stage; stable_dt, the error word
 * and the clip diagnostics are all-reduced (MIN/MAX, exact); conserved_totals
 * and product_mole_fraction fold rank by rank in the reference's serial order. */
#define IGN_NCCL_ID_BYTES 128
int ign_nccl_unique_id(uint8_t* id);
int ign_attach_nccl(ign_context* ctx, const uint8_t* id, int nranks, int rank);

/* Single-process slab group (validation on one GPU): the members (slab
 * contexts of one config, ranks 0..n-1, same device) run in lockstep on one
 * stream; halo rows move by device-to-device copies. */
typedef struct ign_group ign_group;
int ign_group_create(ign_context** members, int n, ign_group** out);
void ign_group_destroy(ign_group* grp);
int ign_group_last_error(const ign_group* grp, ign_error* err);
int ign_group_prepare_stage(ign_group* grp, int stage);
int ign_group_rk3_steps(ign_group* grp, double dt, int64_t nsteps);
int ign_group_stable_dt(ign_group* grp, double* dt);
int ign_group_conserved_totals(ign_group* grp, double* tot);
int ign_group_advance(ign_group* grp);
int ign_group_write_snapshot(ign_group* grp, const char* path, int version, int with_t);
int ign_group_read_snapshot(ign_group* grp, const char* path);

/* ---- ensemble (BASELINE configs[4]) ---------------------------------- */
/* n independent single-GPU contexts on ONE device advanced nsteps each with
 * their own pinned dt (rk3_steps semantics per member), launched
 * step-interleaved on the members' streams so small members share the SMs.
 * status[q] = member q's outcome (its message via ign_last_error); a failed
 * member stops, the others continue.  Returns IGN_OK or a failing status. */
int ign_ensemble_rk3_steps(ign_context** members, int n, const double* dt, int64_t nsteps,
                           int* status);

/* ---- outputs (the reference's field output and diagnostics) ------------ */
/* Simulation::add_probe (solver.hpp:130-135): inclusive interior box in
 * global cell indices; ConfigError when out of range (2D only). */
int ign_add_probe(ign_context* ctx, int32_t i0, int32_t j0, int32_t i1, int32_t j1);
/* 3D extension: box [i0,i1] x [j0,j1] x [k0,k1] (global k), sampled k-outermost;
 * rows are rho, u, v, w, p, T, Y_s (6 + ns values). */
int ign_add_probe3(ign_context* ctx, int32_t i0, int32_t j0, int32_t k0, int32_t i1, int32_t j1,
                   int32_t k1);
/* probe_interval / trace_interval (solver.hpp:71-73): advance() samples the
 * probes and the product-fraction trace every k-th iteration (0 = off). */
int ign_set_sampling(ign_context* ctx, int32_t probe_interval, int32_t trace_interval);
/* ProbeSeries (solver.hpp:42-46): n samples; times[n], rows[n][5+ns] =
 * box means of rho, u, v, p, T, Y_s (3D: rows[n][6+ns] with w after v).
 * NULL arrays: query n only. */
int ign_probe_samples(const ign_context* ctx, int32_t probe, int64_t* n, double* times,
                      double* rows);
/* TraceSeries product_fraction (solver.hpp:48-51, 379-384) */
int ign_trace_samples(const ign_context* ctx, int64_t* n, double* times, double* values);
/* Simulation::config_hash (solver.hpp:68), carried by snapshots */
int ign_set_config_hash(ign_context* ctx, uint64_t hash);
int ign_get_config_hash(const ign_context* ctx, uint64_t* hash);
/* write_snapshot (snapshot.hpp:52-76): IGNS v1, byte-identical to the
 * reference's file for the same state (3D contexts write v2). */
int ign_write_snapshot(ign_context* ctx, const char* path);
/* IGNS v2 (this library): v1 + nz after ns + u32 flags after the hash; flags
 * bit 0 appends the T cache (the Newton guess) for a bit-exact restart. */
int ign_write_snapshot_v2(ign_context* ctx, const char* path, int with_t);
/* read_snapshot + apply_snapshot (snapshot.hpp:78-145): v1 or v2; FormatError
 * on bad magic / version / truncation / shape or species mismatch. */
int ign_read_snapshot(ign_context* ctx, const char* path);

#ifdef __cplusplus
}
#endif

#endif /* IGNIS_B200_H */
