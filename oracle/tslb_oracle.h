/* Plain-C restatement of the tslb thread-safe lattice-Boltzmann hot path.
 *
 * TEST INFRASTRUCTURE ONLY -- this is the CPU checker the GPU path is compared
 * against (tests/, __graft_entry__.smoke(), bench.py's cpu_baseline leg).
 * The product (paper_2304_06437_b200/libtslb_cuda.so) never links or calls it.
 *
 * Parity pinned: tests/test_oracle_vs_ref.py checks this restatement bit for
 * bit against the UNMODIFIED reference headers compiled into
 * oracle/_ref/libtslb_ref.so (oracle/Makefile), and tests/golden/ holds
 * fixtures generated from that build (tests/golden/make_golden.py).
 * D3Q27 has no reference code: its tables are new and "parity unpinned"
 * beyond lattice invariants.
 *
 * Conventions (reference fields.hpp:16-29): SoA buffers, one array of n
 * scalars per direction / moment, x-fastest index i + nx (j + ny k).
 * Lattice ids: 0 D2Q9, 1 D3Q19, 2 D3Q27.  Scalar ids: 0 double, 1 float.
 * Face kinds (boundary.hpp:18): 0 periodic, 1 no-slip wall, 2 moving wall.
 */
#ifndef TSLB_ORACLE_H
#define TSLB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* tslbo_last_error(void);

int tslbo_lattice_info(int lattice, int* q, int* dim, int* c /*q*3*/,
                       int* opp /*q*/, double* t /*q*/, double* b /*q*/);

int tslbo_classify(int lattice, int nx, int ny, int nz, const int* kinds,
                   const double* uw, const uint8_t* solid, uint8_t* solid_out,
                   uint32_t* slow_out, uint64_t* n_fluid);

/* mode: 0 fused_step, 1 reference_step (two-buffer), 2 compute_moments,
 * 3 stream_collide_fused (moments read from `moments`), 4 stream_only.
 * f: q*n scalars (in/out); moments: (1+D+np)*n scalars (in/out, may be NULL
 * for modes 0/1/4 when not wanted). */
int tslbo_single_run(int lattice, int scalar, int nx, int ny, int nz,
                     double omega, const int* kinds, const double* uw,
                     const uint8_t* solid, void* f, void* moments, long steps,
                     int mode);

/* Two-fluid run; argument meaning identical to tslbref_two_run. */
int tslbo_two_run(int lattice, int scalar, int nx, int ny, int nz,
                  double omega, const double* cp, const int* ip,
                  const int* kinds, const double* uw, const uint8_t* solid,
                  void* fr, void* fb, void* out, uint8_t* flags, long steps,
                  int refresh, int mode, const void* phi_in);

/* initialize_regularized (kernels.hpp:295-311): state = 10*n scalars of T
 * (rho ux uy uz pxx pyy pzz pxy pxz pyz), f = q*n. Solid nodes untouched. */
int tslbo_init_regularized(int lattice, int scalar, int nx, int ny, int nz,
                           const uint8_t* solid, const void* state, void* f);

/* initialize_colors (multicomponent.hpp:427-449): state = 5*n scalars of T
 * (rho_r rho_b ux uy uz). */
int tslbo_init_colors(int lattice, int scalar, int nx, int ny, int nz,
                      const uint8_t* solid, const void* state, void* fr,
                      void* fb);

/* totals (solver.hpp:104-113): serial sums in T over fluid nodes. */
int tslbo_totals(int scalar, int dim, uint64_t n, const uint8_t* solid,
                 const void* rho, const void* mom /*dim*n*/, double* mass,
                 double* momentum /*3*/);

/* scan_stability (solver.hpp:39-65) */
int tslbo_stability(int scalar, int dim, uint64_t n, const uint8_t* solid,
                    const void* rho, const void* mom, int* finite,
                    double* max_speed, double* min_rho, double* max_rho);

/* Single-fluid body force F (EXTENSION: the reference has no single-fluid
 * forcing; parity for F != 0 is unpinned). Velocity-shift convention of the
 * reference's two-fluid prepare_stress (multicomponent.hpp:286-304), in the
 * single-fluid arithmetic: compute_moments stores u_eq = j + tau F and
 * Pi^neq = (sum f cc - cs2 rho) - u_eq u_eq, tau = 1 / double(T(omega)),
 * F rounded to T. F = 0 leaves every result unchanged. */
void tslbo_set_body_force(double fx, double fy, double fz);

uint64_t tslbo_fnv1a(const void* data, size_t n, uint64_t h);

/* count_kernel_cost (bench.hpp:30-66) generalised to D3Q27 */
void tslbo_census(int lattice, int elem_bytes, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif
#endif
