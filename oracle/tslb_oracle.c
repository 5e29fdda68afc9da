/* Plain-C restatement of the tslb hot path -- TEST INFRASTRUCTURE ONLY.
 * See tslb_oracle.h for scope, conventions and how parity is pinned.
 *
 * Compiled with -ffp-contract=off (oracle/Makefile) so no multiply-add is
 * fused: every expression below reproduces the reference's evaluation order
 * exactly (collision.hpp:72-127, kernels.hpp:43-215, multicomponent.hpp).
 * The scalar-generic bodies live in tslb_oracle_impl.inc, included once for
 * double and once for float storage (the reference's template parameter T).
 */
#include "tslb_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

const char* tslbo_last_error(void) { return g_err; }

/* Body force of the single-fluid forcing extension (not in the reference;
 * see tslb_oracle.h). Process-wide, test infrastructure. */
static double g_force[3] = {0.0, 0.0, 0.0};
void tslbo_set_body_force(double fx, double fy, double fz) {
  g_force[0] = fx;
  g_force[1] = fy;
  g_force[2] = fz;
}

static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

/* ---------------------------------------------------------------------- */
/* Lattice tables (reference lattice.hpp:23-75; D3Q27 is new, same         */
/* ordering rules: rest first, axes, then diagonals, opposite pairs        */
/* adjacent).                                                              */
/* ---------------------------------------------------------------------- */
typedef struct {
  int q, dim;
  int c[27][3];
  long t[27][2];
  long b[27][2];
  int opp[27];
} lat_t;

static const lat_t LAT_D2Q9 = {
    9, 2,
    {{0, 0, 0}, {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0},
     {1, 1, 0}, {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0}},
    {{4, 9}, {1, 9}, {1, 9}, {1, 9}, {1, 9}, {1, 36}, {1, 36}, {1, 36}, {1, 36}},
    {{-4, 27}, {2, 27}, {2, 27}, {2, 27}, {2, 27},
     {5, 108}, {5, 108}, {5, 108}, {5, 108}},
    {0, 2, 1, 4, 3, 6, 5, 8, 7}};

#define AX18 {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18}, {1, 18}
#define DG36 {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}, {1, 36}

static const lat_t LAT_D3Q19 = {
    19, 3,
    {{0, 0, 0},
     {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
     {1, 1, 0}, {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0},
     {1, 0, 1}, {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
     {0, 1, 1}, {0, -1, -1}, {0, 1, -1}, {0, -1, 1}},
    {{1, 3}, AX18, DG36, DG36},
    {{-1, 3}, AX18, DG36, DG36},
    {0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17}};

/* D3Q27: t = 8/27, 2/27, 1/54, 1/216. Perturbation weights B are not in the
 * reference; we keep the D3Q19 values on rest/axis/face-diagonals and zero on
 * corners, which satisfies sum B = cs2, sum B c = 0, sum B cc = cs2 I
 * (the conditions stated at lattice.hpp:36-38). */
#define AX27 {2, 27}, {2, 27}, {2, 27}, {2, 27}, {2, 27}, {2, 27}
#define DG54 {1, 54}, {1, 54}, {1, 54}, {1, 54}, {1, 54}, {1, 54}
#define CR216 {1, 216}, {1, 216}, {1, 216}, {1, 216}, \
              {1, 216}, {1, 216}, {1, 216}, {1, 216}
#define CR0 {0, 1}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {0, 1}, {0, 1}

static const lat_t LAT_D3Q27 = {
    27, 3,
    {{0, 0, 0},
     {1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1},
     {1, 1, 0}, {-1, -1, 0}, {1, -1, 0}, {-1, 1, 0},
     {1, 0, 1}, {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
     {0, 1, 1}, {0, -1, -1}, {0, 1, -1}, {0, -1, 1},
     {1, 1, 1}, {-1, -1, -1}, {1, 1, -1}, {-1, -1, 1},
     {1, -1, 1}, {-1, 1, -1}, {-1, 1, 1}, {1, -1, -1}},
    {{8, 27}, AX27, DG54, DG54, CR216},
    {{-1, 3}, AX18, DG36, DG36, CR0},
    {0, 2, 1, 4, 3, 6, 5, 8, 7, 10, 9, 12, 11, 14, 13, 16, 15, 18, 17,
     20, 19, 22, 21, 24, 23, 26, 25}};

static const lat_t* get_lat(int id) {
  switch (id) {
    case 0: return &LAT_D2Q9;
    case 1: return &LAT_D3Q19;
    case 2: return &LAT_D3Q27;
    default: return NULL;
  }
}

int tslbo_lattice_info(int lattice, int* q, int* dim, int* c, int* opp,
                       double* t, double* b) {
  const lat_t* L = get_lat(lattice);
  if (!L) return fail("unknown lattice id");
  *q = L->q;
  *dim = L->dim;
  for (int a = 0; a < L->q; ++a) {
    if (c)
      for (int k = 0; k < 3; ++k) c[3 * a + k] = L->c[a][k];
    if (opp) opp[a] = L->opp[a];
    if (t) t[a] = (double)L->t[a][0] / (double)L->t[a][1];
    if (b) b[a] = (double)L->b[a][0] / (double)L->b[a][1];
  }
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Geometry (boundary.hpp:61-144)                                          */
/* ---------------------------------------------------------------------- */
typedef struct {
  int nx, ny, nz;
  size_t n;
} dims_t;

static inline size_t lin(const dims_t* g, int i, int j, int k) {
  return (size_t)i + (size_t)g->nx * ((size_t)j + (size_t)g->ny * (size_t)k);
}

static inline int wrapi(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

static int check_axes(const int* kinds) {
  for (int ax = 0; ax < 3; ++ax) {
    const int lo = kinds[2 * ax] == 0, hi = kinds[2 * ax + 1] == 0;
    if (lo != hi) {
      snprintf(g_err, sizeof g_err,
               "classify_nodes: axis %d mixes a periodic face with a wall", ax);
      return 1;
    }
  }
  return 0;
}

int tslbo_classify(int lattice, int nx, int ny, int nz, const int* kinds,
                   const double* uw, const uint8_t* solid, uint8_t* solid_out,
                   uint32_t* slow_out, uint64_t* n_fluid) {
  (void)uw;
  const lat_t* L = get_lat(lattice);
  if (!L) return fail("unknown lattice id");
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail("classify: bad dims");
  if (check_axes(kinds)) return 1;
  const dims_t g = {nx, ny, nz, (size_t)nx * ny * nz};
  const int nd[3] = {nx, ny, nz};
  if (solid)
    memcpy(solid_out, solid, g.n);
  else
    memset(solid_out, 0, g.n);
  uint64_t nf = 0;
  for (int k = 0; k < nz; ++k)
    for (int j = 0; j < ny; ++j)
      for (int i = 0; i < nx; ++i) {
        const size_t idx = lin(&g, i, j, k);
        slow_out[idx] = 0;
        if (solid_out[idx]) continue;
        ++nf;
        uint32_t mask = 0;
        for (int a = 1; a < L->q; ++a) {
          const int tc[3] = {i + L->c[a][0], j + L->c[a][1], k + L->c[a][2]};
          int slow = 0, wc[3];
          for (int ax = 0; ax < 3; ++ax) {
            wc[ax] = tc[ax];
            if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
              slow = 1;
              wc[ax] = wrapi(tc[ax], nd[ax]);
            }
          }
          if (!slow && solid_out[lin(&g, wc[0], wc[1], wc[2])]) slow = 1;
          if (slow) mask |= (uint32_t)1 << a;
        }
        slow_out[idx] = mask;
      }
  *n_fluid = nf;
  return 0;
}

/* resolve_push (boundary.hpp:118-144). u_wall accumulates in the storage
 * scalar; callers pass the face velocities already rounded to T and sum
 * with the T-typed helper below. Returns 1 for bounce. */
static inline int resolve_target(const dims_t* g, const int* kinds,
                                 const uint8_t* solid, const int* c, int i,
                                 int j, int k, size_t* target,
                                 int crossed[3] /* face id or -1 */) {
  const int nd[3] = {g->nx, g->ny, g->nz};
  int tc[3] = {i + c[0], j + c[1], k + c[2]};
  int bounce = 0;
  for (int ax = 0; ax < 3; ++ax) {
    crossed[ax] = -1;
    if (tc[ax] < 0 || tc[ax] >= nd[ax]) {
      const int face = 2 * ax + (tc[ax] < 0 ? 0 : 1);
      if (kinds[face] == 0) {
        tc[ax] = wrapi(tc[ax], nd[ax]);
      } else {
        bounce = 1;
        crossed[ax] = face;
      }
    }
  }
  if (bounce) return 1;
  const size_t t = lin(g, tc[0], tc[1], tc[2]);
  if (solid[t]) return 1;
  *target = t;
  return 0;
}

/* ---------------------------------------------------------------------- */
/* Scalar-generic bodies                                                   */
/* ---------------------------------------------------------------------- */
#define T double
#define SUF(x) x##_d
#define SQRT_T sqrt
#include "tslb_oracle_impl.inc"
#undef T
#undef SUF
#undef SQRT_T

#define T float
#define SUF(x) x##_f
#define SQRT_T sqrtf
#include "tslb_oracle_impl.inc"
#undef T
#undef SUF
#undef SQRT_T

/* ---------------------------------------------------------------------- */
/* Dispatch                                                                */
/* ---------------------------------------------------------------------- */
int tslbo_single_run(int lattice, int scalar, int nx, int ny, int nz,
                     double omega, const int* kinds, const double* uw,
                     const uint8_t* solid, void* f, void* moments, long steps,
                     int mode) {
  const lat_t* L = get_lat(lattice);
  if (!L) return fail("unknown lattice id");
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail("allocate_fields: bad dims");
  if (check_axes(kinds)) return 1;
  const dims_t g = {nx, ny, nz, (size_t)nx * ny * nz};
  uint8_t* sol = (uint8_t*)malloc(g.n);
  uint32_t* slow = (uint32_t*)malloc(g.n * 4);
  uint64_t nf;
  int rc = tslbo_classify(lattice, nx, ny, nz, kinds, uw, solid, sol, slow, &nf);
  if (!rc) {
    if (scalar == 0)
      rc = single_run_d(L, &g, omega, kinds, uw, sol, slow, (double*)f,
                        (double*)moments, steps, mode);
    else
      rc = single_run_f(L, &g, omega, kinds, uw, sol, slow, (float*)f,
                        (float*)moments, steps, mode);
  }
  free(sol);
  free(slow);
  return rc;
}

int tslbo_two_run(int lattice, int scalar, int nx, int ny, int nz,
                  double omega, const double* cp, const int* ip,
                  const int* kinds, const double* uw, const uint8_t* solid,
                  void* fr, void* fb, void* out, uint8_t* flags, long steps,
                  int refresh, int mode, const void* phi_in) {
  const lat_t* L = get_lat(lattice);
  if (!L) return fail("unknown lattice id");
  if (nx <= 0 || ny <= 0 || nz <= 0) return fail("allocate_two_fluid: bad dims");
  if (check_axes(kinds)) return 1;
  const dims_t g = {nx, ny, nz, (size_t)nx * ny * nz};
  uint8_t* sol = (uint8_t*)malloc(g.n);
  uint32_t* slow = (uint32_t*)malloc(g.n * 4);
  uint64_t nf;
  int rc = tslbo_classify(lattice, nx, ny, nz, kinds, uw, solid, sol, slow, &nf);
  if (!rc) {
    if (scalar == 0)
      rc = two_run_d(L, &g, omega, cp, ip, kinds, uw, sol, slow, (double*)fr,
                     (double*)fb, (double*)out, flags, steps, refresh, mode,
                     (const double*)phi_in);
    else
      rc = two_run_f(L, &g, omega, cp, ip, kinds, uw, sol, slow, (float*)fr,
                     (float*)fb, (float*)out, flags, steps, refresh, mode,
                     (const float*)phi_in);
  }
  free(sol);
  free(slow);
  return rc;
}

int tslbo_init_regularized(int lattice, int scalar, int nx, int ny, int nz,
                           const uint8_t* solid, const void* state, void* f) {
  const lat_t* L = get_lat(lattice);
  if (!L) return fail("unknown lattice id");
  const dims_t g = {nx, ny, nz, (size_t)nx * ny * nz};
  if (scalar == 0)
    init_regularized_d(L, &g, solid, (const double*)state, (double*)f);
  else
    init_regularized_f(L, &g, solid, (const float*)state, (float*)f);
  return 0;
}

int tslbo_init_colors(int lattice, int scalar, int nx, int ny, int nz,
                      const uint8_t* solid, const void* state, void* fr,
                      void* fb) {
  const lat_t* L = get_lat(lattice);
  if (!L) return fail("unknown lattice id");
  const dims_t g = {nx, ny, nz, (size_t)nx * ny * nz};
  if (scalar == 0)
    init_colors_d(L, &g, solid, (const double*)state, (double*)fr, (double*)fb);
  else
    init_colors_f(L, &g, solid, (const float*)state, (float*)fr, (float*)fb);
  return 0;
}

int tslbo_totals(int scalar, int dim, uint64_t n, const uint8_t* solid,
                 const void* rho, const void* mom, double* mass,
                 double* momentum) {
  if (scalar == 0)
    totals_d(dim, n, solid, (const double*)rho, (const double*)mom, mass,
             momentum);
  else
    totals_f(dim, n, solid, (const float*)rho, (const float*)mom, mass,
             momentum);
  return 0;
}

int tslbo_stability(int scalar, int dim, uint64_t n, const uint8_t* solid,
                    const void* rho, const void* mom, int* finite,
                    double* max_speed, double* min_rho, double* max_rho) {
  if (scalar == 0)
    stability_d(dim, n, solid, (const double*)rho, (const double*)mom, finite,
                max_speed, min_rho, max_rho);
  else
    stability_f(dim, n, solid, (const float*)rho, (const float*)mom, finite,
                max_speed, min_rho, max_rho);
  return 0;
}

/* FNV-1a 64 (bench.hpp:83-91) */
uint64_t tslbo_fnv1a(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = (const unsigned char*)data;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ull;
  }
  return h;
}

/* count_kernel_cost (bench.hpp:30-66), same counting rules, any lattice. */
void tslbo_census(int lattice, int elem_bytes, double* flops, double* bytes) {
  const lat_t* L = get_lat(lattice);
  const int D = L->dim, np = D * (D + 1) / 2;
  double p1 = 0, p2 = 12;
  for (int a = 0; a < L->q; ++a) {
    int nm = 0, pairs = 0;
    for (int ax = 0; ax < 3; ++ax)
      if (L->c[a][ax] != 0) ++nm;
    for (int ax = 0; ax < 3; ++ax)
      for (int bx = ax + 1; bx < 3; ++bx)
        if (L->c[a][ax] != 0 && L->c[a][bx] != 0) ++pairs;
    p1 += 1 + 2 * nm + pairs;
    if (nm == 0)
      p2 += 6;
    else
      p2 += ((nm - 1) + 7) + ((nm + pairs - 1) + 3) + 2;
  }
  p1 += 1 + 3 * D + 2 * (np - D);
  *flops = p1 + p2;
  *bytes = 2.0 * (double)(L->q + 1 + D + np) * (double)elem_bytes;
}
