/* etd_b200.h — C-ABI drop-in boundary for the B200-native ETD2RK-DS spectral
 * time step (arXiv 2601.06849).  Plain pointers and sizes only; no torch or
 * C++ types cross this boundary.
 *
 * The reference (`etdrd`, /root/reference/proj/core) exposes this path as a
 * C++ value-semantics API (include/etdrd/stepper.hpp).  Each entry point below
 * names the reference interface it replaces.  A C++ mirror of that interface
 * built on these calls lives in include/etdrd_b200/stepper.hpp, and
 * INTEGRATION.md shows the reference-side binding (a BackendKind::CudaSpectral
 * dispatch in stepper.cpp:318-331).
 *
 * Layout conventions follow the reference Field (field.hpp:13-54): host arrays
 * are dense FP64, x-fastest, index i + nx*(j + ny*k), interior points only.
 * Error codes map 1:1 onto the reference exception types (errors.hpp:8-30).
 */
#ifndef ETD_B200_H
#define ETD_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ETD_B200_ABI_VERSION 4

/* Status codes (0 = OK).  errors.hpp:8-30; CLI mapping cli.cpp:204-217. */
enum etd_status {
    ETD_OK = 0,
    ETD_ERR_CONFIG = 1,      /* etdrd::ConfigError      */
    ETD_ERR_NUMERICS = 2,    /* etdrd::NumericsError    */
    ETD_ERR_ABORT = 3,       /* etdrd::StepperAbort{t,step} */
    ETD_ERR_MEMORY = 4,      /* etdrd::MemoryGuardError */
    ETD_ERR_CUDA = 5,        /* device/driver failure (no reference equivalent) */
    ETD_ERR_NODEVICE = 6     /* no CUDA device: there is no CPU fallback */
};

/* Pade family: rational.hpp:31 PadeFamily {P02, P04}.  ETD_EXACT selects the
 * reference's BackendKind::ExactExpReference step (stepper.cpp:259-295: exact
 * e^{-tau A}, phi_1, phi_2 multipliers on the same transforms), without its
 * 64-points-per-axis cap. */
enum etd_family { ETD_P02 = 0, ETD_P04 = 1, ETD_EXACT = 2 };

/* Directional rational applies: tensor_ops.hpp:31 BackendKind.  ETD_SPECTRAL is
 * the eigenbasis-transform step (BackendKind::Spectral, DMMA tensor cores);
 * ETD_THOMAS the per-pole complex tridiagonal solves (BackendKind::Thomas,
 * thomas.cpp:14-160) with the same step structure (stepper.cpp:231-240,
 * 243-266, system_stepper.cpp:74-114).  Thomas plans run on one GPU. */
enum etd_backend { ETD_SPECTRAL = 0, ETD_THOMAS = 1 };

/* Device source descriptors.  The reference takes a std::function
 * (SourceFunction / SystemSource, stepper.hpp:18-29) which cannot run on the
 * device; the GPU backend takes a pointwise kind + parameters instead and
 * rejects anything else with ETD_ERR_CONFIG. */
enum etd_source_kind {
    ETD_SRC_ZERO = 0,        /* f = 0                                             */
    ETD_SRC_AC_CUBIC = 1,    /* f = u - u^3 (config 0-2; test_stepper.cpp:459-465) */
    ETD_SRC_POLY3 = 2,       /* f = ((p3 u + p2) u + p1) u + p0                    */
    ETD_SRC_NAN = 3,         /* f = NaN at grid point 0, else 0 (abort probe,
                                test_stepper.cpp:304-321)                          */
    ETD_SRC_AC_MANUFACTURED = 4, /* u(1-u^2) + p1 u* - u*(1-u*^2), u* = e^{-p0 t} prod sin(pi x_a):
                                the catalogue Allen-Cahn source (problems.cpp:93-104);
                                p0 = lambda, p1 = -lambda + kappa dim pi^2, p2 = kappa */
    ETD_SRC_SINGULAR = 5,    /* p0 u/(1-u), abort (step -1) if any u >= 1 (problems.cpp:122-133) */
    ETD_SRC_FHN_CUBIC = 10,  /* fu = u(1-u)(u-p0) - v, fv = p1 (p2 u - v) (config 3-4) */
    ETD_SRC_FHN_CLASSIC = 11,/* fu = u - u^3/3 - v, fv = p0 (u - p1 v) (problems.cpp:170-171) */
    ETD_SRC_MIRROR_AC = 12,  /* fu = u - u^3, fv = v - v^3 (test_stepper.cpp:432-438) */
    ETD_SRC_DECOUPLED = 13   /* fu = u - u^3, fv = p0 v + p1                     */
};

typedef struct etd_desc {
    int dim;                 /* 2 or 3 (grid.hpp:17)                               */
    int n[3];                /* interior points per axis = reference Grid::m[a]-1 */
    double low[3], high[3];  /* box bounds (build_grid, grid.hpp:43-45)            */
    double tau;              /* step size, > 0                                      */
    int family;              /* etd_family                                          */
    int nspecies;            /* 1: make_plan (stepper.hpp:59-61); 2: make_system_plan
                                (stepper.hpp:107-108), 2D and 3D                     */
    double kappa[2];         /* kappa (scalar) or kappa_u, kappa_v                  */
    double q;                /* linear reaction, >= 0, split q/dim per axis         */
    int src_kind;            /* etd_source_kind                                     */
    double src_params[8];
    int device;              /* CUDA device ordinal                                  */
    /* z-slab sharding (3D): rank `rank` of `world_size` owns planes
     * [etd_slab_range) ; world_size==1 -> whole grid on one GPU. */
    int world_size, rank;
    const void* nccl_unique_id; /* 128-byte ncclUniqueId (world_size > 1)          */
    int backend;             /* etd_backend (0 = spectral transforms)               */
    /* make_plan's memory_cap_bytes (stepper.hpp:58-61; the reference guards its
     * banded factorisation with it): here the cap on the plan's DEVICE memory
     * on this rank.  0 = the device's free memory.  etd_create fails with
     * ETD_ERR_MEMORY (MemoryGuardError) before allocating when the plan needs more. */
    unsigned long long memory_cap_bytes;
} etd_desc;

typedef struct etd_handle etd_handle;

/* make_plan (stepper.cpp:118-177) / make_system_plan (system_stepper.cpp:31-70):
 * host setup (closed-form eigensystems, Pade d-vectors) + one upload.  */
int etd_create(const etd_desc* desc, etd_handle** out);
/* Device bytes etd_create would allocate for this desc on this rank (state ping-pong,
 * step scratch, sharded exchange blocks, transform matrices).  Host only: the
 * per-rank budget check behind ETD_ERR_MEMORY, callable without a GPU. */
int etd_plan_device_bytes(const etd_desc* desc, unsigned long long* bytes);
/* Plan destruction (plans are immutable values in the reference). */
int etd_destroy(etd_handle* h);

/* This rank's z-slab [z0, z1) (3D) or [0,1) (2D). */
int etd_slab_range(const etd_handle* h, int* z0, int* z1);
/* The balanced partition every sharded plan uses for z planes (x/y stages) and
 * y rows (z stage): rank r gets [lo, hi), sizes differ by at most one.  Host only. */
int etd_zslab_partition(int n, int world_size, int rank, int* lo, int* hi);
/* The data movement of one sharded step for rank `rank` (host only), with the
 * z stage split into `chunks` chunks of each rank's y rows (plans use 4): records
 * of 13 int64 {kind(0 copy2d,1 send,2 recv), phase(0 pack,1 fwd,2 back,3 unpack),
 * peer, dst_buf, dst_off, dst_pitch, src_buf, src_off, src_pitch, width, height,
 * count, chunk}, element units; buffers 0 state,1 send,2 zin,3 wz,4 recv,5 w
 * (zin / wz: the chunk blocks [2 nspecies][nz][chunk rows][pitch] back to back).
 * out may be NULL to query *count. */
int etd_sharded_schedule(int nx, int ny, int nz, int nspecies, int world_size, int rank, long long pitch,
                         int chunks, long long* out, int capacity, int* count);
/* Where the sharded level-2 step's y stack pass reads each y row of this rank's slab
 * from the backward exchange's receive blocks (buffer 4 above; the unpack copies are
 * fused into that pass): out[3 j .. 3 j + 2] = {element offset, field stride, z stride}
 * for global y row j < ny.  Host only. */
int etd_sharded_recv_rows(int ny, int nz, int nspecies, int world_size, int rank, long long pitch, int chunks,
                          long long* out);
/* 128-byte ncclUniqueId for etd_desc.nccl_unique_id (rank 0 creates, all ranks
 * receive it out of band, e.g. over torch.distributed). */
int etd_nccl_unique_id(void* out128);
/* Virtual ranks: plans created with world_size = G and nccl_unique_id = NULL on
 * one device form a group stepped here in lock-step (exchanges become device
 * copies).  Same schedule and abort semantics as the NCCL path. */
int etd_group_step(etd_handle** handles, int count, int nsteps);

/* StepperState/SystemState upload (stepper.hpp:63-67,110-114): species 0=U,
 * 1=V; count = nx*ny*(z1-z0) values (this rank's slab), n,t = state.n,state.t. */
int etd_set_state(etd_handle* h, int species, const double* host, size_t count, long n, double t);
/* State download (materialises the reference Field). */
int etd_get_state(etd_handle* h, int species, double* host, size_t count, long* n, double* t);

/* advance (stepper.cpp:318-331) / etd2rkds_step_system (system_stepper.cpp:74-114)
 * applied nsteps times on the device-resident state.  On a non-finite value the
 * call returns ETD_ERR_ABORT, the state is left at the INPUT of the failing
 * step and etd_last_error reports that step's t and n (stepper.cpp:18-23). */
int etd_step(etd_handle* h, int nsteps);

/* Value-semantics one-shot, the reference's advance(plan, state, f) shape:
 * upload u (and v), step nsteps times, download into u_out (v_out).  Any of
 * v/v_out may be NULL for scalar plans. */
int etd_advance(etd_handle* h, const double* u, const double* v, long n, double t, int nsteps,
                double* u_out, double* v_out, long* n_out, double* t_out);

/* ETRD field snapshot of the device state (reference save_field / load_field,
 * field.cpp:46-81: "ETRD", u32 1, u32 dim, u32 shape[3], f64 t, f64 data), streamed
 * through pinned staging.  Non-finite data is refused (ETD_ERR_NUMERICS).  load
 * restores state t and n (n < 0: n = round(t / tau)).  Sharded plans use their slab. */
int etd_save_snapshot(etd_handle* h, int species, const char* path);
int etd_load_snapshot(etd_handle* h, int species, const char* path, long n);

/* Replace the device source descriptor (the reference passes the source per
 * advance() call, stepper.hpp:85-86; plans do not own it). */
int etd_set_source(etd_handle* h, int src_kind, const double* src_params /* 8 values or NULL */);

/* Last error of this handle: message, abort time and step (errors.hpp:22-28). */
int etd_last_error(const etd_handle* h, char* msg, size_t len, double* t, long* step);

/* ---- introspection / measurement (no reference equivalent) ---------------- */
/* cudaStream_t the handle launches on (as an integer). */
unsigned long long etd_stream(const etd_handle* h);
/* Ranks of the plan's exchange group: ncclCommCount of its NCCL communicator
 * (NCCL-sharded plans), else world_size (1 unsharded, G for virtual ranks). */
int etd_comm_ranks(const etd_handle* h, int* out);
/* Number of kernel launches one step issues (this rank). */
int etd_launches_per_step(const etd_handle* h);
/* Per-stage profiling: when enabled, etd_step records CUDA events around every
 * launch (no CUDA graph) and accumulates device milliseconds per stage. */
int etd_set_profiling(etd_handle* h, int on);
/* stage names/times (ms summed since enable) and FLOPs per launch of stage i. */
int etd_stage_count(const etd_handle* h);
int etd_stage_info(const etd_handle* h, int i, char* name, size_t len, double* ms_total,
                   long* launches, double* flops_per_launch, double* bytes_per_launch);
/* FLOPs per launch of stage i as executed (the parity-split transform does
 * 2 (2h) h / n per point, h = (n+1)/2) and as the dense n x n contraction would
 * (2 n per point, SURVEY §8(d)'s algorithmic count). */
int etd_stage_flops(const etd_handle* h, int i, double* executed, double* dense);
/* Which axes run parity-split transforms (P(n-1-i,k) = (-1)^k P(i,k) of the DST-I
 * eigenbasis, operators.cpp:43-53): out[a] = 1 for a folded axis a < dim. */
int etd_parity_split(const etd_handle* h, int* out);
/* The host-built parity-split half matrices of one axis (etd_plan.cu
 * fold_matrices): forward and backward, 2h interleaved rows x h columns; mode 0
 * stores rows contiguous with leading dimension round_up(h, 16), mode 1 the
 * transpose [h][2h].  Returns ETD_ERR_CONFIG unless h % 8 == 0.  Host only. */
int etd_setup_fold_matrices(int n, int mode, double* ff, double* fb);
/* The second-level split matrices of one axis with n = 4H - 1, H % 8 == 0
 * (etd_plan.cu fold2_matrices): forward ga (FOLD 5, even modes)
 * and gb (FOLD 4, odd modes), backward go (FOLD 4 over sigma/delta) and ge
 * (FOLD 2, odd modes), each 2H interleaved rows x H columns; fb = the
 * first-level backward matrix reading the level-2 mode positions (2h rows x h).
 * Layouts as etd_setup_fold_matrices; go/ge may be NULL.  Returns
 * ETD_ERR_CONFIG otherwise.  Host only. */
int etd_setup_fold2_matrices(int n, int mode, double* ga, double* gb, double* fb, double* go, double* ge);
/* The fused level-2 backward matrix G6 of one axis with n = 32m - 1 (etd_plan.cu
 * back6_matrix): 4H rows x H columns, H = (n+1)/4, rows in blocks of
 * 32 (parity b & 1, orbit base b >> 1) of four 8-row fragments (o_k, o_{2H-2-k},
 * eo_k, ee_k); mode 0 rows contiguous with leading dimension round_up(H, 16), mode
 * 1 the transpose [H][4H].  Host only. */
int etd_setup_back6_matrix(int n, int mode, double* g6);
/* Parity-split level the step runs per axis: 0 dense, 1 first level (§4a),
 * 2 second level (§4b); out[a] for a < 3. */
int etd_fold_level(const etd_handle* h, int* out);

/* Single eigenbasis transform on host data, for kernel-level parity tests:
 * out = op(P_axis) contracted along `axis` (tensor_ops.cpp:107-119 contract_axis
 * with M = P, transpose = !back), optionally followed by scaling with the
 * d-vector d_ell (ell 1..3, 0 = none).  ell>0 && apply_q!=0 runs the full
 * apply_Q_spectral (tensor_ops.cpp:164-172): 2 P (d_ell ⊙ P^T in). */
int etd_debug_transform(etd_handle* h, int species, int axis, int back, int ell, int apply_q,
                        const double* in, double* out);

/* Determinism check: re-run the step's stage kernel `name` (e.g. "x_fwd_corr")
 * `reps` times on its current inputs; *mismatches = max number of output
 * elements (operand `out`) that differ bitwise from the first re-run, pos[0..cap)
 * their element offsets.  A correct (race-free) kernel reports 0. */
int etd_debug_repeat_op(etd_handle* h, const char* name, int out, int reps, long long* mismatches,
                        long long* pos, int cap);

/* Seeded initial conditions for BASELINE configs 0-4;
 * counter-based RNG, identical on every host, multithreaded.  Host only.
 * Writes this rank's slab [z0,z1) of species `species` (x-fastest). */
int etd_fill_config_ic(int config, unsigned long long seed, int species, int n, int z0, int z1,
                       double* out);

/* Host setup exported for parity tests of the one-time plan construction:
 * operators.cpp:11-56 (P column-major n*n, ascending lambda) and
 * rational.cpp:187-198 (d-vector for ell 1..3). */
int etd_setup_axis(int n, double low, double high, int dim, double kappa, double q, double* P,
                   double* lambda);
int etd_setup_dvector(int n, const double* lambda, double tau, int family, int ell, double* d);
/* rational.cpp:133-177: out[(ell-1)*nterms + t] = {pole.re, pole.im, res.re, res.im} */
int etd_setup_scheme(int family, double* out, int* nterms);

/* stepper.cpp:38-46: phi_1(x) = (1 - e^{-x})/x, phi_2(x) = (x - 1 + e^{-x})/x^2 with
 * the reference's series branch below x = 1e-4 (which = 1 or 2; NaN otherwise). */
double etd_setup_phi(int which, double x);

/* ABI version. */
int etd_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ETD_B200_H */
