/*
 * tslb_cuda.h -- C-ABI of the B200-native thread-safe lattice-Boltzmann
 * hot path (libtslb_cuda.so, built from paper_2304_06437_b200/csrc/).
 *
 * The reference (tslb, /root/reference/proj) is a header-only C++20 library
 * with no FFI; its hot path sits behind these C++ entry points, which this
 * ABI replaces one for one (all paths relative to proj/include/tslb/):
 *
 *   tslb_cuda_create            SingleFluidSim ctor   solver.hpp:76-85
 *                               TwoFluidSim ctor      solver.hpp:141-151
 *                               (+ classify_nodes     boundary.hpp:61-111,
 *                                  allocate_fields    fields.hpp:82-125)
 *   tslb_cuda_step              Sim::step / run       solver.hpp:87-94, 153-159
 *                               fused_step            kernels.hpp:209-215
 *                               two_fluid_step        multicomponent.hpp:405-414
 *   tslb_cuda_compute_moments   compute_moments       kernels.hpp:74-107
 *   tslb_cuda_stream_collide    stream_collide_fused  kernels.hpp:154-204
 *   tslb_cuda_reference_step    reference_step        kernels.hpp:262-291
 *   tslb_cuda_stream_only       stream_only           kernels.hpp:219-256
 *   tslb_cuda_color_moments     color_moments         multicomponent.hpp:55-119
 *   tslb_cuda_gradient_and_nci  gradient_and_nci      multicomponent.hpp:154-242
 *   tslb_cuda_prepare_stress    prepare_stress        multicomponent.hpp:271-309
 *   tslb_cuda_stream_collide_recolor  stream_collide_recolor  multicomponent.hpp:315-401
 *   tslb_cuda_refresh_moments   Sim::refresh_moments  solver.hpp:96, 163-166
 *   tslb_cuda_totals            SingleFluidSim::totals solver.hpp:104-113
 *   tslb_cuda_stability         scan_stability        solver.hpp:39-65
 *   tslb_cuda_color_masses      TwoFluidSim::color_masses solver.hpp:172-181
 *   tslb_cuda_upload_f / download_f / upload_field / download_field
 *                               Sim::fields() host access solver.hpp:115-122
 *   tslb_cuda_download_geometry Sim::geometry()       solver.hpp:118 (NodeGeometry)
 *   tslb_cuda_plane_digests     state_digest          bench.hpp:93-109
 *                               (chunked, decomposition-independent form)
 *
 * Conventions
 *   - Host buffers are SoA, x fastest (fields.hpp:26-29): one array of
 *     nx*ny*nz_local scalars per direction / moment component, arrays packed
 *     back to back. Scalars are double (TSLB_F64) or float (TSLB_F32).
 *   - Moment block order: rho, mom[D], pineq[D(D+1)/2] with pineq
 *     xx yy [zz] xy [xz yz] (fields.hpp:50-53).
 *   - Every call returns 0 on success, nonzero on failure, with the message
 *     in tslb_cuda_last_error() (thread-local). Error classes mirror the
 *     reference exceptions: TSLB_EINVAL ~ std::invalid_argument (bad dims,
 *     mask size, half-periodic axis), TSLB_ECUDA ~ std::runtime_error.
 *   - step/run and every phase call block until the device work is done
 *     (the reference's WorkerPool::run is synchronous, parallel.hpp:60-67);
 *     tslb_cuda_step_async only enqueues.
 *   - One host thread per handle; handles are not re-entrant.
 */
#ifndef TSLB_CUDA_H
#define TSLB_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSLB_CUDA_ABI_VERSION 3

typedef struct tslb_cuda_sim* tslb_cuda_handle;

enum tslb_lattice { TSLB_D2Q9 = 0, TSLB_D3Q19 = 1, TSLB_D3Q27 = 2 };
enum tslb_scalar { TSLB_F64 = 0, TSLB_F32 = 1 };
/* boundary.hpp:18 FaceKind */
enum tslb_face { TSLB_FACE_PERIODIC = 0, TSLB_FACE_WALL = 1, TSLB_FACE_MOVING = 2 };
/* node-local arithmetic: F64 is the reference's (bit-exact); F32 opt-in */
enum tslb_math { TSLB_MATH_F64 = 0, TSLB_MATH_F32 = 1 };
/* step schedule of single-fluid box geometries: F1 = moments pass + fused
 * stream-collide (populations in HBM); M = moment-resident single pass
 * (populations rebuilt in shared memory, f materialised on demand). Both are
 * bit-identical to fused_step (kernels.hpp:209-215). */
enum tslb_schedule { TSLB_SCHED_F1 = 0, TSLB_SCHED_M = 1 };
enum tslb_status { TSLB_OK = 0, TSLB_EINVAL = 1, TSLB_ECUDA = 2, TSLB_ENOMEM = 3, TSLB_ESTATE = 4 };

/* field ids for upload_field / download_field */
enum tslb_field {
  TSLB_FIELD_RHO = 0,      /* n scalars */
  TSLB_FIELD_MOM = 1,      /* D arrays */
  TSLB_FIELD_PINEQ = 2,    /* D(D+1)/2 arrays */
  TSLB_FIELD_RHO_R = 3,    /* two-fluid */
  TSLB_FIELD_RHO_B = 4,
  TSLB_FIELD_PHI = 5,
  TSLB_FIELD_GRADPHI = 6,  /* D arrays */
  TSLB_FIELD_NCI_FLAG = 7, /* n bytes */
  TSLB_FIELD_SOLID = 8,    /* n bytes (download only) */
  TSLB_FIELD_SLOW_MASK = 9 /* n uint32 (download only; classify_nodes bits) */
};

/* device analytic initialisers (throughput runs; parity runs upload f) */
enum tslb_init { TSLB_INIT_REST = 0, TSLB_INIT_SHEAR = 1, TSLB_INIT_TAYLOR_GREEN = 2, TSLB_INIT_DROPLET = 3 };

/* profiled kernel classes for tslb_cuda_profile_read */
enum tslb_kclass {
  TSLB_K_MOMENTS = 0, TSLB_K_STREAMCOLL = 1, TSLB_K_CG_MOMENTS = 2,
  TSLB_K_CG_GRADIENT = 3, TSLB_K_CG_STREAMCOLL = 4, TSLB_K_EXCHANGE = 5,
  TSLB_K_MSTEP = 6, TSLB_K_COUNT = 7
};

int tslb_cuda_abi_version(void);
const char* tslb_cuda_last_error(void);
int tslb_cuda_device_count(int* count);

/* Construct a solver on `device`. components = 1 (SingleFluidSim) or 2
 * (TwoFluidSim). face_kind[6] in XMin XMax YMin YMax ZMin ZMax order,
 * face_uwall[18] the three wall-velocity components per face.
 * solid: NULL or nx*ny*nz bytes (1 = solid). color: NULL or
 * {sigma, beta, nci_strength, eps_bulk, grad_threshold}; color_i: NULL or
 * {nci_reach, form (0 squared, 1 linear)} (multicomponent.hpp:24-33). */
int tslb_cuda_create(int lattice, int scalar, int components, int nx, int ny,
                     int nz, double omega, const int* face_kind,
                     const double* face_uwall, const uint8_t* solid,
                     const double* color, const int* color_i, int device,
                     tslb_cuda_handle* out);

/* Same, for one z slab [z0, z0 + nz_local) of an nx*ny*nz global box
 * (multi-GPU decomposition). solid is the GLOBAL mask or NULL. Faces between
 * slabs are exchanged with tslb_cuda_attach_nccl or tslb_cuda_link_local. */
int tslb_cuda_create_slab(int lattice, int scalar, int components, int nx,
                          int ny, int nz, int z0, int nz_local, double omega,
                          const int* face_kind, const double* face_uwall,
                          const uint8_t* solid, const double* color,
                          const int* color_i, int device,
                          tslb_cuda_handle* out);

int tslb_cuda_destroy(tslb_cuda_handle h);
int tslb_cuda_set_math(tslb_cuda_handle h, int math);
/* Select the single-fluid step schedule (default: M where supported -- 3-D:
 * D3Q19/D3Q27 with nx * sizeof(scalar) a multiple of 16 bytes (the TMA row
 * pitch; any nx, ny otherwise: partial tiles at the grid edges), with or
 * without a solid mask, whole domains and z slabs; 2-D: D2Q9 whole domains
 * without solids -- else F1). TSLB_EINVAL if M is requested where it is not
 * supported. Same results either way (fused_step, kernels.hpp:209-215). */
int tslb_cuda_set_schedule(tslb_cuda_handle h, int schedule);
int tslb_cuda_get_schedule(tslb_cuda_handle h, int* schedule);
/* Moment storage of the M schedule. TSLB_STORE_NATIVE (default): the
 * storage scalar. TSLB_STORE_F16 (EXTENSION, the paper's mixed-precision
 * outlook): the steps keep the ten moment arrays as scaled
 * IEEE fp16 (40 B per lattice update instead of 80) with fp32 node
 * arithmetic (switched on with it); every other call sees fp32 moments
 * decoded from them. Tolerance mode, not reference-exact. Needs a fp32
 * single-fluid D3Q19/D3Q27 whole domain on M without solids, nx % 8 == 0. */
enum tslb_store { TSLB_STORE_NATIVE = 0, TSLB_STORE_F16 = 1 };
int tslb_cuda_set_moment_storage(tslb_cuda_handle h, int kind);
/* Single-fluid body force F (EXTENSION: the reference has no single-fluid
 * forcing; used for the Poiseuille channel of BASELINE config 3). Velocity
 * shift of the reference's two-fluid prepare_stress (multicomponent.hpp:
 * 286-304) applied in compute_moments: the stored velocity is
 * u_eq = j + tau F, Pi^neq = (sum f cc - cs2 rho) - u_eq u_eq. F = 0 (the
 * default) leaves every result bit-identical to the reference. */
int tslb_cuda_set_body_force(tslb_cuda_handle h, const double* force3);
/* dims[0..4] = nx, ny, nz_local, z0, nz_global; info[0..3] = q, dim, np, scalar bytes */
int tslb_cuda_describe(tslb_cuda_handle h, int* dims, int* info);
int tslb_cuda_memory_bytes(tslb_cuda_handle h, uint64_t* bytes);

/* populations: species 0 = f (or fr), 1 = fb, 2 = the second buffer of
 * reference_step / stream_only (single fluid); q * n_local scalars */
int tslb_cuda_upload_f(tslb_cuda_handle h, int species, const void* host);
int tslb_cuda_download_f(tslb_cuda_handle h, int species, void* host);
int tslb_cuda_upload_field(tslb_cuda_handle h, int field, const void* host);
int tslb_cuda_download_field(tslb_cuda_handle h, int field, void* host);
/* Device-side sampler for the output writers (io.hpp; tslb_main.cpp:137-188):
 * one 2-D slice of a field -- the plane perpendicular to `axis` (0 x, 1 y,
 * 2 z) at local `index` -- without moving the whole field. Output per array
 * of the field: axis 2 -> nx*ny (x fastest), axis 1 -> nx*nz (x fastest),
 * axis 0 -> ny*nz (y fastest). Same host-visible values as download_field. */
int tslb_cuda_download_slice(tslb_cuda_handle h, int field, int axis, int index, void* host);
int tslb_cuda_download_geometry(tslb_cuda_handle h, uint8_t* solid,
                                uint32_t* slow_mask, uint64_t* n_fluid);
int tslb_cuda_init_analytic(tslb_cuda_handle h, int kind, double amplitude,
                            double radius);
/* initialize_regularized (kernels.hpp:296-311; the drop-in's
 * initialize_regularized(FieldSet, NodeGeometry, node_state)) from HOST node
 * states: (1 + D + D(D+1)/2) arrays of n_local storage-type scalars, the
 * prepare_node arguments rho, u[D], Pi[np] per node (solid nodes are
 * skipped). The upload is chunked and overlapped with the device
 * initialisation; pinned host memory gives full PCIe bandwidth. Single fluid
 * only (TSLB_EINVAL otherwise). Same f(0) bits as the host routine. */
int tslb_cuda_init_state(tslb_cuda_handle h, const void* host_state);
/* The same from rho and u alone, Pi^neq = 0 (prepare_node(rho, u, 0, ...): the
 * equilibrium start of the reference driver, tslb_main.cpp:115-122): (1 + D)
 * arrays of n_local storage-type scalars. */
int tslb_cuda_init_equilibrium(tslb_cuda_handle h, const void* host_rho_u);

/* time stepping */
int tslb_cuda_step(tslb_cuda_handle h, long nsteps);
int tslb_cuda_step_async(tslb_cuda_handle h, long nsteps);
int tslb_cuda_synchronize(tslb_cuda_handle h);
int tslb_cuda_steps_done(tslb_cuda_handle h, long* steps);
/* device time (CUDA events on the solver stream) of nsteps steps */
int tslb_cuda_time_steps(tslb_cuda_handle h, long nsteps, double* ms);

/* reference phase functions (single fluid) */
int tslb_cuda_compute_moments(tslb_cuda_handle h);
int tslb_cuda_stream_collide(tslb_cuda_handle h);
int tslb_cuda_reference_step(tslb_cuda_handle h, long nsteps);
int tslb_cuda_stream_only(tslb_cuda_handle h);
/* reference phase functions (two fluid) */
int tslb_cuda_color_moments(tslb_cuda_handle h);
int tslb_cuda_gradient_and_nci(tslb_cuda_handle h);
int tslb_cuda_prepare_stress(tslb_cuda_handle h);
int tslb_cuda_stream_collide_recolor(tslb_cuda_handle h);
int tslb_cuda_refresh_moments(tslb_cuda_handle h);

/* device-side diagnostics (deterministic fp64 reductions) */
int tslb_cuda_totals(tslb_cuda_handle h, double* mass, double* momentum3);
int tslb_cuda_stability(tslb_cuda_handle h, int* finite, double* max_speed,
                        double* min_rho, double* max_rho, int64_t* first_bad);
int tslb_cuda_color_masses(tslb_cuda_handle h, double* red, double* blue);
/* per-plane chunked FNV-1a of the populations: out[a * nz_local + k],
 * a over q (species 0) then q (species 1 for two-fluid). */
int tslb_cuda_plane_digests(tslb_cuda_handle h, uint64_t* out);

/* measurement */
int tslb_cuda_profile(tslb_cuda_handle h, int enable);
int tslb_cuda_profile_read(tslb_cuda_handle h, double* ms_per_class,
                           int64_t* launches_per_class);
int tslb_cuda_launch_count(tslb_cuda_handle h, int64_t* launches);

/* multi-GPU halo exchange (z slabs) */
int tslb_cuda_nccl_unique_id(void* id128);
int tslb_cuda_attach_nccl(tslb_cuda_handle h, const void* id128, int nranks,
                          int rank);
int tslb_cuda_link_local(tslb_cuda_handle* slabs, int count);
int tslb_cuda_group_step(tslb_cuda_handle* slabs, int count, long nsteps);
/* Peer-memory transport for M single-fluid slabs (one process per GPU, no
 * NCCL): each rank exports a block holding its ghost planes (double
 * buffered by exchange parity) and two flag words as a CUDA IPC handle
 * (TSLB_IPC_HANDLE_BYTES), the ranks swap handles over any host channel, and
 * every rank maps its z neighbours' blocks. A step's boundary chunks then
 * store the new boundary planes straight into the neighbours' ghost buffers
 * from the M kernel's epilogue (NVLink peer stores between GPUs) and publish
 * the exchange number in their flag words; the consumer's stream waits for
 * it before the ghost planes are read. A face that wraps onto the rank itself (one rank, periodic) passes
 * the rank's own handle. TSLB_ESTATE for two-fluid or F1 steps. */
#define TSLB_IPC_HANDLE_BYTES 64
int tslb_cuda_ipc_handle(tslb_cuda_handle h, void* handle64);
int tslb_cuda_attach_ipc(tslb_cuda_handle h, const void* below64, const void* above64);

#ifdef __cplusplus
}
#endif
#endif /* TSLB_CUDA_H */
