// Internal launcher declarations shared by the kernel TUs and the C-ABI TU.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tslb_domain.cuh"

namespace tslb_cuda {

enum MathMode : int { kMathDouble = 0, kMathFloat = 1 };

// kInitState: node states (the prepare_node arguments rho, u[D], Pi[np] of
// initialize_regularized, kernels.hpp:296-311) read from device arrays
enum InitKind : int { kInitRest = 0, kInitShear = 1, kInitTaylorGreen = 2, kInitDroplet = 3, kInitState = 4 };

struct InitSpec {
  int kind;
  int nx_g, ny_g, nz_g;  // global extents (for slabs)
  int z0;                // global z of local plane 0
  double amp;            // shear / Taylor-Green velocity amplitude
  double cx, cy, cz, radius, width;  // droplet
  const void* state;     // kInitState: [1 + D (+ np)][sstride] of the storage type
  int64_t sstride;
  int spi;               // kInitState: the states carry Pi^neq (else Pi^neq = 0)
};

struct ColorParamsDev {
  double sigma, beta, nci_strength, eps_bulk, grad_threshold;
  int nci_reach, linear;
};

// ---- single fluid (tslb_single.cu)
template <typename T>
int launch_moments(int lat, int math, const Dom& d, const T* f, T* mo,
                   const uint8_t* solid, cudaStream_t st);
template <typename T>
int launch_streamcoll(int lat, int math, const Dom& d, T* f, const T* mo,
                      const uint8_t* solid, const uint32_t* slow, double omega,
                      cudaStream_t st);
// box geometry (no solid mask), nx % (16 / sizeof(T)) == 0
template <typename T>
int launch_streamcoll_vec(int lat, int math, const Dom& d, T* f, const T* mo,
                          double omega, int vx, int kz, cudaStream_t st);
// moment-resident single-pass step (tslb_mstep.cu): m(t) in `mi` -> m(t+1)
// in `mo` for box geometries, planes [z0, z1) (z1 <= 0: to the end) in
// chunks of lz planes per CTA column; `gm` holds the slab ghost planes
// ([2][NM][plane], below/above) when a z face is a slab interface. Returns
// 1 (nothing launched) when the shape is not supported, -cudaError on a
// launch failure. `maps` caches the TMA tensor maps (opaque, owned by the
// caller, freed with free_mstep_maps).
struct MstepMaps;
void free_mstep_maps(MstepMaps* maps);
bool mstep_supported(int lat, const Dom& d, int esz);
template <typename T>
int launch_mstep(int lat, int math, const Dom& d, const T* mi, const T* gm, T* mo, double omega,
                 int lz, int z0, int z1, MstepMaps*& maps, const uint32_t* sbits, cudaStream_t st,
                 T* peer_lo = nullptr, T* peer_hi = nullptr);
// mixed-precision M step (tslb_mstep.cu, tslb_store16.cuh): fp16 moments,
// fp32 populations and arithmetic, whole domains without solids, nx % 8 == 0
bool mstep16_supported(int lat, const Dom& d);
int launch_mstep16(int lat, const Dom& d, const __half* mi, __half* mo, double omega, int lz, MstepMaps*& maps,
                   cudaStream_t st);
// fp32 moments <-> fp16 storage (to16 = 1: encode m32 into m16)
int launch_moments_codec16(const Dom& d, int nm, float* m32, __half* m16, int to16, cudaStream_t st);
// per-node solid bits of a masked geometry for the 3-D M step (tslb_mstep.cu)
int launch_solid_bits(int lat, const Dom& d, const uint8_t* solid, uint32_t* bits, cudaStream_t st);
// D2Q9 form of the M step (tslb_mstep2d.cu; launched through launch_mstep)
template <typename T>
int launch_mstep2d(int math, const Dom& d, const T* mi, T* mo, double omega, cudaStream_t st);
template <typename T>
int launch_mstep2d_persist(int math, const Dom& d, T* m0, T* m1, double omega, int nsteps, cudaStream_t st);
// slab f materialisation: pushes entering boundary plane `side` (0 below,
// 1 above) rebuilt from the ghost moments
template <typename T>
int launch_ghost_push(int lat, int math, const Dom& d, T* f, const T* gm, double omega, int side,
                      const uint8_t* solid, cudaStream_t st);
template <typename T>
int launch_collide(int lat, const Dom& d, T* f, const T* mo,
                   const uint8_t* solid, double omega, cudaStream_t st);
template <typename T>
int launch_stream_only(int lat, const Dom& d, const T* f, T* dst,
                       const uint8_t* solid, const uint32_t* slow,
                       cudaStream_t st);
int launch_classify(int lat, const Dom& d, const uint8_t* solid,
                    uint32_t* slow, unsigned long long* n_fluid,
                    cudaStream_t st);
template <typename T>
int launch_init_analytic(int lat, const Dom& d, T* f, const uint8_t* solid,
                         const InitSpec& s, cudaStream_t st);
// moments of the analytic f(0) without storing f(0) (M schedule)
template <typename T>
int launch_init_moments(int lat, int math, const Dom& d, T* mo, const InitSpec& s,
                        cudaStream_t st);

// ---- two fluid (tslb_two.cu)
struct TwoFields {
  void *rho_r, *rho_b, *rho, *mom, *pin, *phi, *grad;  // each mstride-strided
  uint8_t* flag;
};
template <typename T>
int launch_cg_moments(int lat, const Dom& d, const T* fr, const T* fb,
                      const TwoFields& s, const uint8_t* solid,
                      cudaStream_t st);
template <typename T>
int launch_cg_gradient(int lat, const Dom& d, const TwoFields& s,
                       const uint8_t* solid, const uint32_t* slow,
                       const ColorParamsDev& cp, cudaStream_t st);
template <typename T>
int launch_cg_prepare_stress(int lat, const Dom& d, const TwoFields& s,
                             const uint8_t* solid, double omega,
                             const ColorParamsDev& cp, cudaStream_t st);
template <typename T>
int launch_cg_streamcoll(int lat, const Dom& d, T* fr, T* fb,
                         const TwoFields& s, const uint8_t* solid,
                         const uint32_t* slow, double omega,
                         const ColorParamsDev& cp, int fold_prepare,
                         cudaStream_t st);
// the whole two-fluid box step in one pass (f_old -> f_new + the colour
// moment arrays; box, NCI off, nx % 32 == ny % 8 == 0); nonzero when not
// applicable
template <typename T>
int launch_cg_fused(int lat, const Dom& d, const T* fr, const T* fb, T* gr, T* gb, const TwoFields& s,
                    double omega, const ColorParamsDev& cp, cudaStream_t st);
bool cg_fused_supported(int lat, const Dom& d, int esz, const ColorParamsDev& cp);
// gradient folded into the recolouring stream-collide (box, NCI off);
// nonzero when not applicable
template <typename T>
int launch_cg_streamcoll_grad(int lat, const Dom& d, T* fr, T* fb, const TwoFields& s,
                              double omega, const ColorParamsDev& cp, cudaStream_t st);
template <typename T>
int launch_init_colors(int lat, const Dom& d, T* fr, T* fb,
                       const uint8_t* solid, const InitSpec& s,
                       cudaStream_t st);
// gradient_and_nci on a box geometry that may be a z slab (phi and the NCI
// flags carry nci_reach ghost planes; hits there are ORed into the
// neighbours' flags with launch_flag_or)
template <typename T>
int launch_cg_gradient_nci_box(int lat, const Dom& d, const TwoFields& s, const ColorParamsDev& cp,
                               cudaStream_t st);
int launch_flag_or(uint8_t* dst, const uint8_t* src, int64_t n, cudaStream_t st);

// ---- reductions / digest (tslb_reduce.cu)
// totals: out[0] = mass, out[1..3] = momentum (fp64 deterministic tree)
template <typename T>
int launch_totals(const Dom& d, int dim, const T* rho, const T* mom,
                  const uint8_t* solid, double* partial, double* out,
                  cudaStream_t st);
// stability: out = {finite(0/1), max_speed, min_rho, max_rho}
template <typename T>
int launch_stability(const Dom& d, int dim, const T* rho, const T* mom,
                     const uint8_t* solid, double* partial, double* out,
                     cudaStream_t st);
// per-plane FNV-1a digests of `narrays` arrays (stride elements apart,
// first owned plane at offset `base`): out[a * nz + k]
int launch_plane_digest(const Dom& d, const void* arr, int narrays,
                        int64_t stride, int64_t base, int elem_bytes,
                        uint64_t* chunk_scratch, uint64_t* out,
                        cudaStream_t st);

size_t reduce_partial_count();

// ---- slab exchange (tslb_exchange.cu)
template <typename T>
int launch_unpack(const Dom& d, T* f, const T* recv, const uint8_t* solid,
                  int ndirs, const int* a, const int* cx, const int* cy,
                  int kdst, int ksrc_ghost, cudaStream_t st);
// peer-memory transport flags: publish / await an exchange number (null
// words are skipped)
int launch_ipc_signal(uint64_t* a, uint64_t* b, uint64_t v, cudaStream_t st);
int launch_ipc_wait(const uint64_t* a, const uint64_t* b, uint64_t v, cudaStream_t st);

}  // namespace tslb_cuda
