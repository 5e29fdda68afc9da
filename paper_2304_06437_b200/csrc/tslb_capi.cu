// C-ABI (include/tslb_cuda.h) over the sm_100a kernels: solver objects,
// device memory, time stepping, slab halo exchange, diagnostics, profiling.
//
// The reference's Sim classes (solver.hpp:70-202) own host Eigen arrays and a
// WorkerPool; here a handle owns device SoA buffers and one CUDA stream. The
// stream order is the phase barrier. Host<->device copies happen only in the
// explicit upload/download calls; the drop-in C++ headers (include/tslb/)
// and the Python mirror keep the reference's host-visible semantics on top.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tslb_cuda.h"
#include "tslb_kernels.h"
#include "tslb_lattice.cuh"

using namespace tslb_cuda;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// (a failed call's error is reported here and cleared, so a later
// cudaGetLastError() does not report it a second time against another call)
#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      cudaGetLastError();                                                     \
      return set_err(TSLB_ECUDA, "%s: %s (%s:%d)", #call,                     \
                     cudaGetErrorString(e_), __FILE__, __LINE__);             \
    }                                                                         \
  } while (0)

// ---- NCCL, loaded at run time (torch's copy if already mapped) -------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrStr)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  auto sym = [&](const char* s) { return dlsym(h, s); };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.Send = (decltype(api.Send))sym("ncclSend");
  api.Recv = (decltype(api.Recv))sym("ncclRecv");
  api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
  api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
  api.ErrStr = (decltype(api.ErrStr))sym("ncclGetErrorString");
  api.ok = api.GetUniqueId && api.CommInitRank && api.Send && api.Recv &&
           api.GroupStart && api.GroupEnd;
  return api;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

template <class F>
void lattice_of(int lat, F&& f) {
  if (lat == kD2Q9) f(D2Q9{});
  else if (lat == kD3Q19) f(D3Q19{});
  else f(D3Q27{});
}

}  // namespace

struct tslb_cuda_sim {
  // configuration
  int lat = 0, scalar = 0, comps = 1, q = 0, dim = 0, np = 0, esz = 8;
  int nx = 0, ny = 0, nzl = 0, z0 = 0, nzg = 0;
  bool decomposed = false;
  int device = 0;
  int math = kMathDouble;
  // box-geometry stream-collide kernel: 0 scalar, 1 vectorised (pipelined
  // if kz > 1) (TSLB_STREAMCOLL=scalar|vec overrides)
  int variant = 1;
  // single-fluid schedule: M (moment-resident single pass, tslb_mstep.cu)
  // where supported, else F1. In M, `fimplicit` means the populations
  // f(t+1) = stream_collide(m(t)) are not stored: `mo` holds m(t) (the
  // reference's lagged moment arrays) and f is materialised on demand.
  int sched = TSLB_SCHED_F1;
  bool fimplicit = false;
  // lazy f under M: `f0_pending` = the current f is the analytic f(0) of
  // `f0_spec` and the buffer does not hold it (yet); `m0_ready` = mo2 holds
  // the moments of the current f (the first step's moments pass, done by the
  // initialiser)
  bool f0_pending = false, m0_ready = false;
  InitSpec f0_spec{};
  int lz = 0;          // planes per CTA of the M kernel (0 = default; TSLB_LZ)
  void* mo2 = nullptr; // second moment buffer of the M schedule (ping-pong)
  void* gm = nullptr;  // M on z slabs: neighbours' boundary-plane moments [2][NM][plane] (below, above)
  void* sx = nullptr;  // M on z slabs: own boundary-plane moments to send [2][NM][plane] (plane 0, nzl - 1)
  int lzb = 0;         // planes of each boundary chunk on slabs (0 = default; TSLB_LZB)
  void* graph_mo = nullptr;  // moment buffer the captured graph starts from
  MstepMaps* mmaps = nullptr;  // TMA tensor maps of the M kernel's inputs
  int vx = 0;          // nodes per thread in the vectorised kernel (0 = default; TSLB_VX)
  int kz = 0;          // planes per block of the pipelined kernel (<= 1: off; TSLB_KZ)
  bool staged = false; // slab halos received into staging + masked unpack
  double omega = 1.0;
  int kinds[6] = {0, 0, 0, 0, 0, 0};
  ColorParamsDev cp{};
  Dom d{};
  // device memory
  void* f[2] = {nullptr, nullptr};
  void* mo = nullptr;     // rho, mom[D], pineq[np]
  void* two = nullptr;    // rho_r, rho_b, phi, grad[D]
  uint8_t* flag = nullptr;
  uint8_t* solid = nullptr;
  uint32_t* slow = nullptr;
  uint32_t* sbits = nullptr;  // M on a masked geometry: per-node solid bits (with ghost planes)
  void* scratch = nullptr;
  void* state_buf = nullptr;  // tslb_cuda_init_state: the node states [state_nm][mstride] (f(0) pending on them)
  int state_nm = 0;            // arrays in state_buf: 1+D+np (init_state) or 1+D (init_equilibrium)
  // mixed-precision moment storage (tslb_cuda_set_moment_storage): the M
  // steps run on fp16 moments mh/mh2 (tslb_store16.cuh); every other API
  // works on the fp32 moments mo, decoded on demand (m32_valid) and encoded
  // again before the next step once an fp32 path changed them (m16_valid)
  // refreshed under M: the moments of the current f(t+1) are in mo2 (one M
  // pass), mo still holds m(t) that f(t+1) is implicit in; the next step is
  // just the swap (tslb_cuda_refresh_moments)
  bool mvis2 = false;
  int store16 = 0;
  void* mh = nullptr;
  void* mh2 = nullptr;
  bool m16_valid = false, m32_valid = true;
  double* red = nullptr;  // partials + outputs
  uint64_t* dig = nullptr;
  size_t dig_bytes = 0;
  uint64_t bytes = 0;
  uint64_t n_fluid = 0;
  cudaStream_t s = nullptr, cs = nullptr;
  cudaEvent_t ev_b = nullptr, ev_c = nullptr, t0 = nullptr, t1 = nullptr;
  // CUDA graph of `graph_steps` fused steps, replayed for small (launch-
  // bound) domains; TSLB_GRAPHS=0 disables
  cudaGraphExec_t graph = nullptr;
  long graph_steps = 0;
  int64_t graph_launches = 0;
  bool graphs_ok = true;
  bool stress_pending = false;
  // two-fluid: the fused step folded the gradient phase into the recolouring
  // kernel; the gradient arrays are filled when something reads them
  bool grad_pending = false;
  bool grad_pending_after_graph = false;
  long steps = 0;
  // profiling
  bool prof = false;
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> rec;
  size_t pool_used = 0;
  int64_t launches = 0;
  // exchange
  void* falt[2] = {nullptr, nullptr};  // two-fluid one-pass step: the other population buffers (ping-pong)
  int xmode = 0;  // 0 none, 1 nccl, 2 local, 3 peer memory (CUDA IPC)
  // peer-memory transport (xmode 3, M steps): the exported block holds two
  // flag words (exchange numbers from below / from above) and the ghost
  // planes [2][NM][plane] twice (exchange parity); the neighbours' blocks
  // are mapped (or, for a face that wraps onto this rank, the own block)
  char* ipc_blk = nullptr;
  size_t ipc_gb = 0;
  char* ipc_up = nullptr;
  char* ipc_down = nullptr;
  bool ipc_up_mapped = false, ipc_down_mapped = false;
  uint64_t xcount = 0;  // exchanges issued
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, up = -1, down = -1;
  tslb_cuda_sim* up_peer = nullptr;
  tslb_cuda_sim* down_peer = nullptr;
  void* recv_lo = nullptr;  // staging (masked geometries), per species
  void* recv_hi = nullptr;
  void* phig = nullptr;     // two-fluid slabs: phi with pgz ghost planes below and above
  int pgz = 1;              // two-fluid slabs: ghost planes of phi (and of the NCI flags): max(1, nci_reach) with NCI
  uint8_t* flagg = nullptr; // two-fluid slabs with NCI: flag allocation with pgz ghost planes each side
  uint8_t* rflag = nullptr; // two-fluid slabs with NCI: received neighbour flag planes [2][pgz plane]
  int zp[9], zm[9], nzp = 0, nzm = 0;  // directions with c_z = +1 / -1
  int zpx[9], zpy[9], zmx[9], zmy[9];

  int64_t n() const { return int64_t(nx) * ny * nzl; }
  int64_t plane() const { return int64_t(nx) * ny; }
  void* fa(int sp, int a) const {
    return static_cast<char*>(f[sp]) + size_t(a) * d.fstride * esz;
  }
  void* m_arr(int c) const {  // the host-visible moment arrays
    return static_cast<char*>(mvis2 ? mo2 : mo) + size_t(c) * d.mstride * esz;
  }
  void* t_arr(int c) const {
    return static_cast<char*>(two) + size_t(c) * d.mstride * esz;
  }
  TwoFields tf() const {
    TwoFields t;
    t.rho = m_arr(0);
    t.mom = m_arr(1);
    t.pin = m_arr(1 + dim);
    t.rho_r = t_arr(0);
    t.rho_b = t_arr(1);
    t.phi = phig ? static_cast<char*>(phig) + size_t(pgz) * size_t(plane()) * esz : t_arr(2);
    t.grad = t_arr(3);
    t.flag = flag;
    return t;
  }
  Dom range(int k0, int k1) const {
    Dom r = d;
    r.k0 = k0;
    r.nzr = k1 - k0;
    return r;
  }
};

namespace {

int alloc(tslb_cuda_sim* h, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e != cudaSuccess)
    return set_err(TSLB_ENOMEM, "cudaMalloc(%zu bytes): %s (device holds %llu already)",
                   bytes, cudaGetErrorString(e), (unsigned long long)h->bytes);
  h->bytes += bytes;
  return 0;
}

// -- profiling helpers --------------------------------------------------------
cudaEvent_t pool_event(tslb_cuda_sim* h) {
  if (h->pool_used == h->pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h->pool.push_back(e);
  }
  return h->pool[h->pool_used++];
}

struct Prof {
  tslb_cuda_sim* h;
  int cls;
  cudaStream_t st;
  cudaEvent_t e0 = nullptr;
  Prof(tslb_cuda_sim* h_, int c, cudaStream_t s_) : h(h_), cls(c), st(s_) {
    if (h->prof) {
      e0 = pool_event(h);
      cudaEventRecord(e0, st);
    }
  }
  ~Prof() {
    if (h->prof) {
      cudaEvent_t e1 = pool_event(h);
      cudaEventRecord(e1, st);
      h->rec.push_back({cls, {e0, e1}});
    }
  }
};

template <class F>
int by_scalar(const tslb_cuda_sim* h, F&& f) {
  if (h->scalar == TSLB_F64) return f(double(0));
  return f(float(0));
}

// the near-contact scan runs (gradient_and_nci: cp.nci_strength != T(0))
bool nci_on(const tslb_cuda_sim* h) {
  return h->scalar == TSLB_F64 ? h->cp.nci_strength != 0.0 : float(h->cp.nci_strength) != 0.0f;
}

// mixed precision: the fp32 moments mo are needed (decode the fp16 state)
int sync32(tslb_cuda_sim* h) {
  if (!h->store16 || h->m32_valid) return 0;
  ++h->launches;
  if (launch_moments_codec16(h->range(0, h->nzl), 1 + h->dim + h->np, static_cast<float*>(h->mo),
                             static_cast<__half*>(h->mh), 0, h->s))
    return set_err(TSLB_ECUDA, "fp16 moment decode launch failed");
  h->m32_valid = true;
  return 0;
}

// leave the refreshed-under-M state for a standard one: f(t+1) stored (from
// m(t)), the moment arrays = m(t+1) (what refresh_moments promised)
int unvis(tslb_cuda_sim* h);

// API prologue: decode fp16 moments if needed; unless the caller only reads
// the host-visible moments, leave the refreshed-under-M state
int settle(tslb_cuda_sim* h, bool visible_ok = false) {
  if (int rc = sync32(h)) return rc;
  if (!visible_ok && h->mvis2) return unvis(h);
  return 0;
}

// -- phases -------------------------------------------------------------------
// the single-fluid population buffer, allocated on first use under M and
// filled with the pending analytic f(0) if there is one
int ensure_f(tslb_cuda_sim* h) {
  // node states of tslb_cuda_init_state that no pending f(0) refers to any
  // more: their memory goes before the populations are allocated
  if (h->state_buf && !h->f0_pending) {
    CK(cudaFree(h->state_buf));
    h->state_buf = nullptr;
    h->bytes -= size_t(h->d.mstride) * h->state_nm * h->esz;
  }
  if (!h->f[0]) {
    const size_t fbytes = size_t(h->d.fstride) * h->q * h->esz;
    if (int rc = alloc(h, &h->f[0], fbytes)) return rc;
    CK(cudaMemsetAsync(h->f[0], 0, fbytes, h->s));
  }
  if (h->f0_pending) {
    h->f0_pending = false;
    ++h->launches;
    return by_scalar(h, [&](auto z) {
      using T = decltype(z);
      return launch_init_analytic<T>(h->lat, h->range(0, h->nzl), static_cast<T*>(h->f[0]), nullptr,
                                     h->f0_spec, h->s);
    });
  }
  return 0;
}

int ph_moments(tslb_cuda_sim* h, cudaStream_t st) {
  if (h->comps == 1)
    if (int rc = ensure_f(h)) return rc;
  h->m16_valid = false;
  h->mvis2 = false;
  Prof p(h, TSLB_K_MOMENTS, st);
  ++h->launches;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_moments<T>(h->lat, h->math, h->range(0, h->nzl),
                             static_cast<const T*>(h->f[0]), static_cast<T*>(h->mo),
                             h->solid, st);
  });
}

int ph_streamcoll(tslb_cuda_sim* h, int k0, int k1, cudaStream_t st) {
  if (k1 <= k0) return 0;
  if (int rc = ensure_f(h)) return rc;
  Prof p(h, TSLB_K_STREAMCOLL, st);
  ++h->launches;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    if (h->variant >= 1 && !h->d.has_solid &&
        launch_streamcoll_vec<T>(h->lat, h->math, h->range(k0, k1), static_cast<T*>(h->f[0]),
                                 static_cast<const T*>(h->mo), h->omega, h->vx, h->kz, st) == 0)
      return 0;
    return launch_streamcoll<T>(h->lat, h->math, h->range(k0, k1),
                                static_cast<T*>(h->f[0]), static_cast<const T*>(h->mo),
                                h->solid, h->slow, h->omega, st);
  });
}

// M schedule: m(t) in h->mo -> m(t+1) in h->mo2 for planes [z0, z1) (z1 <= 0:
// to the end); the caller swaps the buffers once every plane is done.
// peer_lo / peer_hi: where the new planes 0 / nzl-1 also go (the z
// neighbours' ghost buffers, peer-memory transport), or null
int ph_mstep(tslb_cuda_sim* h, cudaStream_t st, int z0 = 0, int z1 = 0, void* peer_lo = nullptr,
             void* peer_hi = nullptr) {
  Prof p(h, TSLB_K_MSTEP, st);
  ++h->launches;
  int rc = by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_mstep<T>(h->lat, h->math, h->range(0, h->nzl), static_cast<const T*>(h->mo),
                           static_cast<const T*>(h->gm), static_cast<T*>(h->mo2), h->omega, h->lz, z0, z1, h->mmaps,
                           h->sbits ? h->sbits + size_t(h->d.ghost) * h->plane() : nullptr, st,
                           static_cast<T*>(peer_lo), static_cast<T*>(peer_hi));
  });
  if (rc < 0) return set_err(TSLB_ECUDA, "k_mstep launch: %s", cudaGetErrorString(cudaError_t(-rc)));
  if (rc) return set_err(TSLB_ESTATE, "M step not supported for this domain");
  return 0;
}

// planes per boundary chunk of a slab step: thin, so the halo exchange
// starts early and overlaps the interior chunks (TSLB_LZB overrides)
constexpr int kBoundaryLz = 16;
int boundary_planes(const tslb_cuda_sim* h) {
  return std::min(h->lzb > 0 ? h->lzb : kBoundaryLz, h->nzl);
}

size_t moment_plane_block(const tslb_cuda_sim* h) {  // bytes of NM planes
  return size_t(1 + h->dim + h->np) * size_t(h->plane()) * h->esz;
}

// the boundary planes of the moment buffer `buf` into the packed send
// buffer h->sx: two strided 2-D copies (NM planes each)
int pack_moments(tslb_cuda_sim* h, const void* buf, cudaStream_t st) {
  const size_t pb = size_t(h->plane()) * h->esz;
  const int nm = 1 + h->dim + h->np;
  for (int side = 0; side < 2; ++side) {
    const int k = side ? h->nzl - 1 : 0;
    const char* src = static_cast<const char*>(buf) + size_t(k) * pb;
    char* dst = static_cast<char*>(h->sx) + size_t(side) * moment_plane_block(h);
    CK(cudaMemcpy2DAsync(dst, pb, src, size_t(h->d.mstride) * h->esz, pb, size_t(nm), cudaMemcpyDeviceToDevice, st));
  }
  return 0;
}

// M on slabs: the packed boundary planes (h->sx, all 1+D+np arrays in one
// block per face) into the neighbours' ghost planes (their `gm`): one send
// and one receive per face. Same grouping as the F1 exchange: +z direction
// first, then -z, so every peer pair matches its sends and receives in order
// (also when up == down).
int exchange_moments_nccl(tslb_cuda_sim* h, cudaStream_t st) {
  NcclApi& N = nccl();
  const ncclDataType_t ty = h->scalar == TSLB_F64 ? ncclFloat64 : ncclFloat32;
  const size_t cnt = size_t(1 + h->dim + h->np) * size_t(h->plane());
  const size_t blk = moment_plane_block(h);
  char* sx = static_cast<char*>(h->sx);
  char* gm = static_cast<char*>(h->gm);
  Prof p(h, TSLB_K_EXCHANGE, st);
  N.GroupStart();
  if (h->up >= 0) N.Send(sx + blk, cnt, ty, h->up, h->comm, st);
  if (h->down >= 0) N.Recv(gm, cnt, ty, h->down, h->comm, st);
  if (h->down >= 0) N.Send(sx, cnt, ty, h->down, h->comm, st);
  if (h->up >= 0) N.Recv(gm + blk, cnt, ty, h->up, h->comm, st);
  ncclResult_t r = N.GroupEnd();
  if (r != ncclSuccess)
    return set_err(TSLB_ECUDA, "NCCL moment halo exchange: %s", N.ErrStr ? N.ErrStr(r) : "error");
  return 0;
}

// local transport of the same (single-device verification)
int exchange_moments_local(tslb_cuda_sim* h, cudaStream_t st) {
  const size_t blk = moment_plane_block(h);
  Prof p(h, TSLB_K_EXCHANGE, st);
  if (h->up_peer)
    CK(cudaMemcpyAsync(h->up_peer->gm, static_cast<char*>(h->sx) + blk, blk, cudaMemcpyDeviceToDevice, st));
  if (h->down_peer)
    CK(cudaMemcpyAsync(static_cast<char*>(h->down_peer->gm) + blk, h->sx, blk, cudaMemcpyDeviceToDevice, st));
  return 0;
}

// peer-memory transport: the new boundary planes of the moment buffer `buf`
// straight into the neighbours' ghost buffers of this exchange's parity (one
// strided 2-D copy per face, over NVLink between GPUs), then the exchange
// number into their flag words. Double buffering by parity makes the flags
// the only synchronisation: a neighbour can only write parity p again after
// it has received this rank's next exchange, which is issued after this
// rank's reads of parity p (stream order).
constexpr size_t kIpcFlags = 256;
// copy = false: the M kernel's boundary chunks already wrote the planes into
// the neighbours' buffers (ipc_targets); only the flags are published
int exchange_moments_ipc(tslb_cuda_sim* h, const void* buf, cudaStream_t st, bool copy = true) {
  const uint64_t e = ++h->xcount;
  const size_t par = size_t(e & 1) * h->ipc_gb;
  const size_t pb = size_t(h->plane()) * h->esz, blk = moment_plane_block(h);
  const int nm = 1 + h->dim + h->np;
  const size_t spitch = size_t(h->d.mstride) * h->esz;
  const char* src = static_cast<const char*>(buf);
  Prof p(h, TSLB_K_EXCHANGE, st);
  if (copy && h->ipc_up)  // top plane -> the up neighbour's "below" ghost planes
    CK(cudaMemcpy2DAsync(h->ipc_up + kIpcFlags + par, pb, src + size_t(h->nzl - 1) * pb, spitch, pb, size_t(nm),
                         cudaMemcpyDeviceToDevice, st));
  if (copy && h->ipc_down)  // bottom plane -> the down neighbour's "above" ghost planes
    CK(cudaMemcpy2DAsync(h->ipc_down + kIpcFlags + par + blk, pb, src, spitch, pb, size_t(nm),
                         cudaMemcpyDeviceToDevice, st));
  ++h->launches;
  if (launch_ipc_signal(h->ipc_up ? reinterpret_cast<uint64_t*>(h->ipc_up) : nullptr,
                        h->ipc_down ? reinterpret_cast<uint64_t*>(h->ipc_down) + 1 : nullptr, e, st))
    return set_err(TSLB_ECUDA, "k_ipc_signal launch failed");
  return 0;
}

// where the M kernel writes this step's boundary planes for the next
// exchange (plane 0 -> the down neighbour's "above" ghost planes, plane
// nzl-1 -> the up neighbour's "below" ones, parity of that exchange)
void ipc_targets(const tslb_cuda_sim* h, void*& lo, void*& hi) {
  lo = hi = nullptr;
  if (h->xmode != 3 || h->d.has_solid) return;  // (masked slabs: copies after the chunks)
  const size_t par = size_t((h->xcount + 1) & 1) * h->ipc_gb;
  if (h->ipc_down) lo = h->ipc_down + kIpcFlags + par + moment_plane_block(h);
  if (h->ipc_up) hi = h->ipc_up + kIpcFlags + par;
}

// before the ghost planes of the current moments are read on `st`: wait for
// the neighbours' latest exchange and point gm at its parity
int ipc_ghosts(tslb_cuda_sim* h, cudaStream_t st) {
  if (h->xmode != 3 || h->xcount == 0) return 0;
  const uint64_t* fl = reinterpret_cast<const uint64_t*>(h->ipc_blk);
  ++h->launches;
  if (launch_ipc_wait(h->ipc_down ? fl : nullptr, h->ipc_up ? fl + 1 : nullptr, h->xcount, st))
    return set_err(TSLB_ECUDA, "k_ipc_wait launch failed");
  h->gm = h->ipc_blk + kIpcFlags + size_t(h->xcount & 1) * h->ipc_gb;
  return 0;
}

// the first step's moments pass: precomputed by the M initialiser, or from f
int first_moments(tslb_cuda_sim* h, cudaStream_t st) {
  h->m16_valid = false;
  h->mvis2 = false;
  if (h->m0_ready) {
    std::swap(h->mo, h->mo2);
    h->m0_ready = false;
    // the current f is now f(1) = stream_collide(m(0)), which overwrites every
    // slot of the buffer when it is materialised: f(0) is no longer owed
    h->f0_pending = false;
    return 0;
  }
  return ph_moments(h, st);
}

// store f(t+1) = stream_collide(m(t)) if the M schedule left it implicit;
// on slabs the pushes entering through the slab faces are rebuilt from the
// ghost moments instead of exchanged
int materialize(tslb_cuda_sim* h) {
  if (!h->fimplicit) return 0;
  if (int rc = sync32(h)) return rc;
  h->fimplicit = false;
  if (int rc = ph_streamcoll(h, 0, h->nzl, h->s)) return rc;
  if (!h->decomposed) return 0;
  if (int rc = ipc_ghosts(h, h->s)) return rc;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    for (int side = 0; side < 2; ++side) {
      if (h->d.mode[side ? ZMax : ZMin] != kGhost) continue;
      ++h->launches;
      if (launch_ghost_push<T>(h->lat, h->math, h->range(0, h->nzl), static_cast<T*>(h->f[0]),
                               static_cast<const T*>(h->gm), h->omega, side,
                               h->d.has_solid ? h->solid : nullptr, h->s))
        return set_err(TSLB_ESTATE, "ghost push: bad lattice");
    }
    return 0;
  });
}

int unvis(tslb_cuda_sim* h) {
  if (!h->mvis2) return 0;
  if (int rc = materialize(h)) return rc;  // f(t+1) from m(t) in mo
  std::swap(h->mo, h->mo2);                // the refreshed m(t+1)
  h->mvis2 = false;
  return 0;
}

int ph_cg_moments(tslb_cuda_sim* h, cudaStream_t st, int k0 = 0, int k1 = -1) {
  if (k1 < 0) k1 = h->nzl;
  if (k1 <= k0) return 0;
  Prof p(h, TSLB_K_CG_MOMENTS, st);
  ++h->launches;
  h->stress_pending = false;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_cg_moments<T>(h->lat, h->range(k0, k1),
                                static_cast<const T*>(h->f[0]),
                                static_cast<const T*>(h->f[1]), h->tf(), h->solid, st);
  });
}

int ph_cg_gradient(tslb_cuda_sim* h, cudaStream_t st) {
  Prof p(h, TSLB_K_CG_GRADIENT, st);
  ++h->launches;
  h->grad_pending = false;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_cg_gradient<T>(h->lat, h->range(0, h->nzl), h->tf(), h->solid,
                                 h->slow, h->cp, st);
  });
}

int ph_cg_prepare(tslb_cuda_sim* h, cudaStream_t st) {
  ++h->launches;
  h->stress_pending = false;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_cg_prepare_stress<T>(h->lat, h->range(0, h->nzl), h->tf(),
                                       h->solid, h->omega, h->cp, st);
  });
}

// the gradient arrays of the last fused two-fluid step, if still owed
int finish_gradient(tslb_cuda_sim* h) {
  if (!h->grad_pending) return 0;
  return ph_cg_gradient(h, h->s);
}

int ph_cg_streamcoll(tslb_cuda_sim* h, int fold, cudaStream_t st) {
  Prof p(h, TSLB_K_CG_STREAMCOLL, st);
  ++h->launches;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_cg_streamcoll<T>(h->lat, h->range(0, h->nzl),
                                   static_cast<T*>(h->f[0]), static_cast<T*>(h->f[1]),
                                   h->tf(), h->solid, h->slow, h->omega, h->cp, fold, st);
  });
}

// -- slab exchange ------------------------------------------------------------
// plane k (-1 .. nzl) of population array a, species 0
void* plane_ptr(const tslb_cuda_sim* h, int a, int k, int sp = 0) {
  return static_cast<char*>(h->fa(sp, a)) +
         size_t((int64_t(k) + h->d.ghost) * h->plane()) * h->esz;
}

// destination for a received plane: in place, or the staging buffer
void* recv_ptr(const tslb_cuda_sim* h, bool from_below, int e, int a, int sp = 0) {
  if (h->staged) {
    void* base = from_below ? h->recv_lo : h->recv_hi;
    return static_cast<char*>(base) + size_t(9 * sp + e) * h->plane() * h->esz;
  }
  return plane_ptr(h, a, from_below ? 0 : h->nzl - 1, sp);
}

int unpack(tslb_cuda_sim* h, cudaStream_t st) {
  if (!h->staged) return 0;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    const size_t sp_off = size_t(9) * h->plane();
    for (int sp = 0; sp < h->comps; ++sp) {
      if (h->d.mode[ZMin] == kGhost) {
        ++h->launches;
        launch_unpack<T>(h->d, static_cast<T*>(h->f[sp]), static_cast<const T*>(h->recv_lo) + sp * sp_off,
                         h->solid, h->nzp, h->zp, h->zpx, h->zpy, 0, -1, st);
      }
      if (h->d.mode[ZMax] == kGhost) {
        ++h->launches;
        launch_unpack<T>(h->d, static_cast<T*>(h->f[sp]), static_cast<const T*>(h->recv_hi) + sp * sp_off,
                         h->solid, h->nzm, h->zm, h->zmx, h->zmy, h->nzl - 1, h->nzl, st);
      }
    }
    return 0;
  });
}

int exchange_nccl(tslb_cuda_sim* h, cudaStream_t st) {
  NcclApi& N = nccl();
  const ncclDataType_t ty = h->scalar == TSLB_F64 ? ncclFloat64 : ncclFloat32;
  const size_t cnt = size_t(h->plane());
  Prof p(h, TSLB_K_EXCHANGE, st);
  N.GroupStart();
  for (int sp = 0; sp < h->comps; ++sp) {
    if (h->up >= 0)
      for (int e = 0; e < h->nzp; ++e) N.Send(plane_ptr(h, h->zp[e], h->nzl, sp), cnt, ty, h->up, h->comm, st);
    if (h->down >= 0)
      for (int e = 0; e < h->nzp; ++e)
        N.Recv(recv_ptr(h, true, e, h->zp[e], sp), cnt, ty, h->down, h->comm, st);
    if (h->down >= 0)
      for (int e = 0; e < h->nzm; ++e) N.Send(plane_ptr(h, h->zm[e], -1, sp), cnt, ty, h->down, h->comm, st);
    if (h->up >= 0)
      for (int e = 0; e < h->nzm; ++e)
        N.Recv(recv_ptr(h, false, e, h->zm[e], sp), cnt, ty, h->up, h->comm, st);
  }
  ncclResult_t r = N.GroupEnd();
  if (r != ncclSuccess)
    return set_err(TSLB_ECUDA, "NCCL halo exchange: %s", N.ErrStr ? N.ErrStr(r) : "error");
  return 0;
}

// local transport: this slab's ghost planes -> neighbours' boundary planes
int exchange_local(tslb_cuda_sim* h, cudaStream_t st) {
  const size_t bytes = size_t(h->plane()) * h->esz;
  Prof p(h, TSLB_K_EXCHANGE, st);
  for (int sp = 0; sp < h->comps; ++sp) {
    if (h->up_peer)
      for (int e = 0; e < h->nzp; ++e)
        CK(cudaMemcpyAsync(recv_ptr(h->up_peer, true, e, h->zp[e], sp),
                           plane_ptr(h, h->zp[e], h->nzl, sp), bytes,
                           cudaMemcpyDeviceToDevice, st));
    if (h->down_peer)
      for (int e = 0; e < h->nzm; ++e)
        CK(cudaMemcpyAsync(recv_ptr(h->down_peer, false, e, h->zm[e], sp),
                           plane_ptr(h, h->zm[e], -1, sp), bytes,
                           cudaMemcpyDeviceToDevice, st));
  }
  return 0;
}

// two-fluid slabs: phi's pgz boundary planes -> the neighbours' phi ghost
// planes (the gradient stencil and the near-contact probes), same grouping
// as above
int exchange_phi_nccl(tslb_cuda_sim* h, cudaStream_t st) {
  NcclApi& N = nccl();
  const ncclDataType_t ty = h->scalar == TSLB_F64 ? ncclFloat64 : ncclFloat32;
  const int g = h->pgz;
  const size_t cnt = size_t(g) * size_t(h->plane());
  char* phi = static_cast<char*>(h->tf().phi);
  auto pl = [&](int k) { return phi + (int64_t(k) * h->plane()) * h->esz; };
  Prof p(h, TSLB_K_EXCHANGE, st);
  N.GroupStart();
  if (h->up >= 0) N.Send(pl(h->nzl - g), cnt, ty, h->up, h->comm, st);
  if (h->down >= 0) N.Recv(pl(-g), cnt, ty, h->down, h->comm, st);
  if (h->down >= 0) N.Send(pl(0), cnt, ty, h->down, h->comm, st);
  if (h->up >= 0) N.Recv(pl(h->nzl), cnt, ty, h->up, h->comm, st);
  ncclResult_t r = N.GroupEnd();
  if (r != ncclSuccess)
    return set_err(TSLB_ECUDA, "NCCL phi halo exchange: %s", N.ErrStr ? N.ErrStr(r) : "error");
  return 0;
}

int exchange_phi_local(tslb_cuda_sim* h, cudaStream_t st) {
  const int g = h->pgz;
  const size_t bytes = size_t(g) * size_t(h->plane()) * h->esz;
  auto pl = [&](const tslb_cuda_sim* x, int k) {
    return static_cast<char*>(x->tf().phi) + (int64_t(k) * x->plane()) * x->esz;
  };
  Prof p(h, TSLB_K_EXCHANGE, st);
  if (h->up_peer) CK(cudaMemcpyAsync(pl(h->up_peer, -g), pl(h, h->nzl - g), bytes, cudaMemcpyDeviceToDevice, st));
  if (h->down_peer)
    CK(cudaMemcpyAsync(pl(h->down_peer, h->down_peer->nzl), pl(h, 0), bytes, cudaMemcpyDeviceToDevice, st));
  return 0;
}

// two-fluid slabs with NCI: flags the scan set in the ghost planes belong
// to the neighbours' nodes -- ship them (lower ghosts to the slab below,
// upper to the slab above) into the receiver's staging planes, which
// fold_flags ORs into its own boundary planes
int exchange_flags_nccl(tslb_cuda_sim* h, cudaStream_t st) {
  NcclApi& N = nccl();
  const size_t gp = size_t(h->pgz) * size_t(h->plane());
  Prof p(h, TSLB_K_EXCHANGE, st);
  N.GroupStart();
  if (h->up >= 0) N.Send(h->flag + int64_t(h->nzl) * h->plane(), gp, ncclUint8, h->up, h->comm, st);
  if (h->down >= 0) N.Recv(h->rflag, gp, ncclUint8, h->down, h->comm, st);
  if (h->down >= 0) N.Send(h->flagg, gp, ncclUint8, h->down, h->comm, st);
  if (h->up >= 0) N.Recv(h->rflag + gp, gp, ncclUint8, h->up, h->comm, st);
  ncclResult_t r = N.GroupEnd();
  if (r != ncclSuccess)
    return set_err(TSLB_ECUDA, "NCCL NCI flag exchange: %s", N.ErrStr ? N.ErrStr(r) : "error");
  return 0;
}

int exchange_flags_local(tslb_cuda_sim* h, cudaStream_t st) {
  const size_t gp = size_t(h->pgz) * size_t(h->plane());
  Prof p(h, TSLB_K_EXCHANGE, st);
  if (h->up_peer)
    CK(cudaMemcpyAsync(h->up_peer->rflag, h->flag + int64_t(h->nzl) * h->plane(), gp, cudaMemcpyDeviceToDevice, st));
  if (h->down_peer) CK(cudaMemcpyAsync(h->down_peer->rflag + gp, h->flagg, gp, cudaMemcpyDeviceToDevice, st));
  return 0;
}

// received flags -> OR into the boundary planes they describe (from below:
// planes [0, pgz); from above: [nzl - pgz, nzl)); then clear the ghost flags
// for the next scan
int fold_flags(tslb_cuda_sim* h, cudaStream_t st) {
  const int64_t gp = int64_t(h->pgz) * h->plane();
  h->launches += 2;
  if (h->down >= 0 || h->down_peer)
    if (launch_flag_or(h->flag, h->rflag, gp, st)) return set_err(TSLB_ECUDA, "k_flag_or launch failed");
  if (h->up >= 0 || h->up_peer)
    if (launch_flag_or(h->flag + int64_t(h->nzl) * h->plane() - gp, h->rflag + gp, gp, st))
      return set_err(TSLB_ECUDA, "k_flag_or launch failed");
  CK(cudaMemsetAsync(h->flagg, 0, size_t(gp), st));
  CK(cudaMemsetAsync(h->flag + int64_t(h->nzl) * h->plane(), 0, size_t(gp), st));
  return 0;
}

// gradient + near-contact scan of a slab (box geometry, ghost planes)
int ph_cg_gradient_slab(tslb_cuda_sim* h, cudaStream_t st) {
  Prof p(h, TSLB_K_CG_GRADIENT, st);
  h->launches += nci_on(h) ? 2 : 1;
  h->grad_pending = false;
  const int rc = by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_cg_gradient_nci_box<T>(h->lat, h->range(0, h->nzl), h->tf(), h->cp, st);
  });
  return rc ? set_err(TSLB_ESTATE, "two-fluid slab step needs a box geometry") : 0;
}

// the recolouring stream-collide of planes [k0, k1) from the stored
// gradient arrays and flags (prepare_stress folded in)
int ph_cg_streamcoll_range(tslb_cuda_sim* h, int k0, int k1, cudaStream_t st) {
  if (k1 <= k0) return 0;
  Prof p(h, TSLB_K_CG_STREAMCOLL, st);
  ++h->launches;
  return by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_cg_streamcoll<T>(h->lat, h->range(k0, k1), static_cast<T*>(h->f[0]), static_cast<T*>(h->f[1]),
                                   h->tf(), h->solid, h->slow, h->omega, h->cp, 1, st);
  });
}

// One fused step (fused_step / two_fluid_step) enqueued on h->s.
// the two-fluid one-pass step (k_cg_fused) is opt-in, TSLB_CG_FUSED=1: it
// is bit-exact but measured slower than the two-kernel step (droplet 512^3:
// 7.4 vs 14.3 GLUPS -- the staging costs twice the instructions per node and
// the ring re-reads 1.5x the population bytes; profiles/r02_droplet_fused_ncu_full.txt)
bool cg_fused_on(const tslb_cuda_sim* h) {
  if (h->comps != 2 || h->decomposed) return false;
  const char* e = std::getenv("TSLB_CG_FUSED");
  if (!e || std::atoi(e) != 1) return false;
  return cg_fused_supported(h->lat, h->d, int(h->esz), h->cp);
}

int enqueue_step(tslb_cuda_sim* h) {
  if (h->xmode == 3 && !(h->comps == 1 && h->sched == TSLB_SCHED_M && !h->store16))
    return set_err(TSLB_ESTATE, "peer-memory (IPC) slab transport: single-fluid M steps only");
  int rc;
  if (h->comps == 2 && h->xmode == 1 && nci_on(h)) {
    // two-fluid slab with the near-contact scan: colour moments, phi's
    // nci_reach boundary planes to the neighbours, gradient + scan (probes
    // run into the ghost planes and may flag the neighbours' nodes), the
    // ghost flags ORed into their owners' planes, then the recolouring
    // stream-collide from the stored gradient and flags -- boundary planes
    // first, population exchange overlapped with the interior as below
    if ((rc = ph_cg_moments(h, h->s))) return rc;
    if ((rc = exchange_phi_nccl(h, h->s))) return rc;
    if ((rc = ph_cg_gradient_slab(h, h->s))) return rc;
    if ((rc = exchange_flags_nccl(h, h->s))) return rc;
    if ((rc = fold_flags(h, h->s))) return rc;
    if ((rc = ph_cg_streamcoll_range(h, 0, 1, h->s))) return rc;
    if (h->nzl > 1 && (rc = ph_cg_streamcoll_range(h, h->nzl - 1, h->nzl, h->s))) return rc;
    CK(cudaEventRecord(h->ev_b, h->s));
    CK(cudaStreamWaitEvent(h->cs, h->ev_b, 0));
    if ((rc = exchange_nccl(h, h->cs))) return rc;
    CK(cudaEventRecord(h->ev_c, h->cs));
    if ((rc = ph_cg_streamcoll_range(h, 1, h->nzl - 1, h->s))) return rc;
    CK(cudaStreamWaitEvent(h->s, h->ev_c, 0));
    if ((rc = unpack(h, h->s))) return rc;
    h->stress_pending = true;
    ++h->steps;
    return 0;
  }
  if (h->comps == 2 && h->xmode == 1) {
    // two-fluid slab: colour moments, phi ghost planes, folded recolouring
    // stream-collide, population halos of both species. As in F1, the two
    // boundary planes go first and the population exchange on the comm
    // stream overlaps the interior planes: the interior stream-collide
    // reads phi of owned planes only and writes no slot the exchange
    // sends or receives (one writer per slot)
    // colour moments of the two boundary planes first: their phi goes to
    // the neighbours on the comm stream while the interior planes' colour
    // moments run (they neither read nor write phi's boundary/ghost planes)
    if ((rc = ph_cg_moments(h, h->s, 0, 1))) return rc;
    if (h->nzl > 1 && (rc = ph_cg_moments(h, h->s, h->nzl - 1, h->nzl))) return rc;
    CK(cudaEventRecord(h->ev_b, h->s));
    CK(cudaStreamWaitEvent(h->cs, h->ev_b, 0));
    if ((rc = exchange_phi_nccl(h, h->cs))) return rc;
    CK(cudaEventRecord(h->ev_c, h->cs));
    if ((rc = ph_cg_moments(h, h->s, 1, h->nzl - 1))) return rc;
    CK(cudaStreamWaitEvent(h->s, h->ev_c, 0));
    auto scr = [&](int k0, int k1) {
      if (k1 <= k0) return 0;
      Prof p(h, TSLB_K_CG_STREAMCOLL, h->s);
      ++h->launches;
      const int r = by_scalar(h, [&](auto z) {
        using T = decltype(z);
        return launch_cg_streamcoll_grad<T>(h->lat, h->range(k0, k1), static_cast<T*>(h->f[0]),
                                            static_cast<T*>(h->f[1]), h->tf(), h->omega, h->cp, h->s);
      });
      return r ? set_err(TSLB_ESTATE, "two-fluid slab step needs a box geometry without NCI") : 0;
    };
    if ((rc = scr(0, 1))) return rc;
    if (h->nzl > 1 && (rc = scr(h->nzl - 1, h->nzl))) return rc;
    CK(cudaEventRecord(h->ev_b, h->s));
    CK(cudaStreamWaitEvent(h->cs, h->ev_b, 0));
    if ((rc = exchange_nccl(h, h->cs))) return rc;
    CK(cudaEventRecord(h->ev_c, h->cs));
    if ((rc = scr(1, h->nzl - 1))) return rc;
    CK(cudaStreamWaitEvent(h->s, h->ev_c, 0));
    if ((rc = unpack(h, h->s))) return rc;
    h->grad_pending = true;
    h->stress_pending = true;
    ++h->steps;
    return 0;
  }
  if (h->comps == 2 && cg_fused_on(h)) {
    // box geometry without NCI: the whole step in one pass into the other
    // population buffers (k_cg_fused), which then become the current ones
    if (!h->falt[0]) {
      const size_t fbytes = size_t(h->d.fstride) * h->q * h->esz;
      for (int sp = 0; sp < 2; ++sp)
        if ((rc = alloc(h, &h->falt[sp], fbytes))) return rc;
    }
    {
      Prof p(h, TSLB_K_CG_STREAMCOLL, h->s);
      rc = by_scalar(h, [&](auto z) {
        using T = decltype(z);
        return launch_cg_fused<T>(h->lat, h->range(0, h->nzl), static_cast<const T*>(h->f[0]),
                                  static_cast<const T*>(h->f[1]), static_cast<T*>(h->falt[0]),
                                  static_cast<T*>(h->falt[1]), h->tf(), h->omega, h->cp, h->s);
      });
    }
    if (rc < 0) return set_err(TSLB_ECUDA, "k_cg_fused launch: %s", cudaGetErrorString(cudaError_t(-rc)));
    if (rc == 0) {
      ++h->launches;
      std::swap(h->f[0], h->falt[0]);
      std::swap(h->f[1], h->falt[1]);
      h->grad_pending = true;
      h->stress_pending = true;
      ++h->steps;
      return 0;
    }
  }
  if (h->comps == 2) {
    if ((rc = ph_cg_moments(h, h->s))) return rc;
    // box geometry without NCI: gradient folded into the stream-collide
    int folded = 1;
    {
      Prof p(h, TSLB_K_CG_STREAMCOLL, h->s);
      folded = by_scalar(h, [&](auto z) {
        using T = decltype(z);
        return launch_cg_streamcoll_grad<T>(h->lat, h->range(0, h->nzl), static_cast<T*>(h->f[0]),
                                            static_cast<T*>(h->f[1]), h->tf(), h->omega, h->cp, h->s);
      });
    }
    if (folded == 0) {
      ++h->launches;
      h->grad_pending = true;
    } else {
      if ((rc = ph_cg_gradient(h, h->s))) return rc;
      if ((rc = ph_cg_streamcoll(h, 1, h->s))) return rc;
    }
    h->stress_pending = true;
    ++h->steps;
    return 0;
  }
  if (h->sched == TSLB_SCHED_M) {
    if (!h->fimplicit) {
      // first step from stored populations: the moments pass (and, on
      // slabs, the ghost planes of m(t)); the stream-collide is deferred
      if ((rc = first_moments(h, h->s))) return rc;
      if (h->xmode == 1) {
        if ((rc = pack_moments(h, h->mo, h->s))) return rc;
        if ((rc = exchange_moments_nccl(h, h->s))) return rc;
      } else if (h->xmode == 3) {
        if ((rc = exchange_moments_ipc(h, h->mo, h->s))) return rc;
      }
      h->fimplicit = true;
    } else if (h->xmode == 1 || h->xmode == 3) {
      // slab: the two thin boundary chunks run on the (high-priority) comm
      // stream and write the new boundary planes into the send buffer; the
      // exchange follows them there, while the interior chunk runs on the
      // solver stream at the same time. The boundary chunks start once the
      // previous step is complete on both streams; the solver stream joins
      // the exchange before the next step.
      const int b = boundary_planes(h);
      // peer memory: the boundary chunks write their new boundary planes into
      // the neighbours' ghost buffers themselves, the exchange only
      // publishes the flags; NCCL: packed send / receive
      auto exchange = [&](cudaStream_t st) {
        if (h->xmode == 3) return exchange_moments_ipc(h, h->mo2, st, h->d.has_solid);
        if (int r = pack_moments(h, h->mo2, st)) return r;
        return exchange_moments_nccl(h, st);
      };
      void *plo = nullptr, *phi = nullptr;
      if (h->nzl <= 2 * b) {
        if ((rc = ipc_ghosts(h, h->s))) return rc;
        ipc_targets(h, plo, phi);
        if ((rc = ph_mstep(h, h->s, 0, 0, plo, phi))) return rc;
        if ((rc = exchange(h->s))) return rc;
      } else {
        CK(cudaEventRecord(h->ev_b, h->s));
        CK(cudaStreamWaitEvent(h->cs, h->ev_b, 0));
        if ((rc = ipc_ghosts(h, h->cs))) return rc;
        ipc_targets(h, plo, phi);
        if ((rc = ph_mstep(h, h->cs, 0, b, plo, nullptr))) return rc;
        if ((rc = ph_mstep(h, h->cs, h->nzl - b, h->nzl, nullptr, phi))) return rc;
        if ((rc = exchange(h->cs))) return rc;
        CK(cudaEventRecord(h->ev_c, h->cs));
        if ((rc = ph_mstep(h, h->s, b, h->nzl - b))) return rc;
        CK(cudaStreamWaitEvent(h->s, h->ev_c, 0));
      }
      std::swap(h->mo, h->mo2);
    } else if (h->store16) {
      // mixed precision: fp16 moments in and out (40 B per update)
      if (!h->m16_valid) {
        ++h->launches;
        if (launch_moments_codec16(h->range(0, h->nzl), 1 + h->dim + h->np, static_cast<float*>(h->mo),
                                   static_cast<__half*>(h->mh), 1, h->s))
          return set_err(TSLB_ECUDA, "fp16 moment encode launch failed");
        h->m16_valid = true;
      }
      {
        Prof p(h, TSLB_K_MSTEP, h->s);
        ++h->launches;
        const int r = launch_mstep16(h->lat, h->range(0, h->nzl), static_cast<const __half*>(h->mh),
                                     static_cast<__half*>(h->mh2), h->omega, h->lz, h->mmaps, h->s);
        if (r < 0) return set_err(TSLB_ECUDA, "k_mstep (fp16) launch: %s", cudaGetErrorString(cudaError_t(-r)));
        if (r) return set_err(TSLB_ESTATE, "fp16 M step not supported for this domain");
      }
      std::swap(h->mh, h->mh2);
      h->m32_valid = false;
    } else {
      if ((rc = ph_mstep(h, h->s))) return rc;
      std::swap(h->mo, h->mo2);
    }
    ++h->steps;
    return 0;
  }
  if ((rc = ph_moments(h, h->s))) return rc;
  if (h->xmode != 1) {
    if ((rc = ph_streamcoll(h, 0, h->nzl, h->s))) return rc;
  } else {
    // boundary planes first, halo exchange on the comm stream overlapped
    // with the interior planes, then join before the next moments pass
    if ((rc = ph_streamcoll(h, 0, 1, h->s))) return rc;
    if (h->nzl > 1 && (rc = ph_streamcoll(h, h->nzl - 1, h->nzl, h->s))) return rc;
    CK(cudaEventRecord(h->ev_b, h->s));
    CK(cudaStreamWaitEvent(h->cs, h->ev_b, 0));
    if ((rc = exchange_nccl(h, h->cs))) return rc;
    CK(cudaEventRecord(h->ev_c, h->cs));
    if ((rc = ph_streamcoll(h, 1, h->nzl - 1, h->s))) return rc;
    CK(cudaStreamWaitEvent(h->s, h->ev_c, 0));
    if ((rc = unpack(h, h->s))) return rc;
  }
  ++h->steps;
  return 0;
}

int check_axes(const int* kinds) {
  for (int ax = 0; ax < 3; ++ax) {
    const bool lo = kinds[2 * ax] == TSLB_FACE_PERIODIC;
    const bool hi = kinds[2 * ax + 1] == TSLB_FACE_PERIODIC;
    if (lo != hi)
      return set_err(TSLB_EINVAL,
                     "classify_nodes: axis %d mixes a periodic face with a wall", ax);
  }
  return 0;
}

int run_classify(tslb_cuda_sim* h, uint32_t* slow_dst) {
  unsigned long long* cnt;
  CK(cudaMallocAsync(&cnt, sizeof(unsigned long long), h->s));
  CK(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), h->s));
  ++h->launches;
  if (launch_classify(h->lat, h->range(0, h->nzl), h->solid, slow_dst, cnt, h->s))
    return set_err(TSLB_EINVAL, "classify: bad lattice");
  unsigned long long v = 0;
  CK(cudaMemcpyAsync(&v, cnt, sizeof v, cudaMemcpyDeviceToHost, h->s));
  CK(cudaFreeAsync(cnt, h->s));
  CK(cudaStreamSynchronize(h->s));
  h->n_fluid = v;
  return 0;
}

int create_impl(int lattice, int scalar, int components, int nx, int ny,
                int nz, int z0, int nzl, double omega, const int* kinds,
                const double* uw, const uint8_t* solid, const double* color,
                const int* color_i, int device, tslb_cuda_handle* out) {
  if (!out) return set_err(TSLB_EINVAL, "null output handle");
  *out = nullptr;
  if (lattice < 0 || lattice > 2) return set_err(TSLB_EINVAL, "unknown lattice %d", lattice);
  if (scalar != TSLB_F64 && scalar != TSLB_F32) return set_err(TSLB_EINVAL, "unknown scalar %d", scalar);
  if (components != 1 && components != 2)
    return set_err(TSLB_EINVAL, "components must be 1 or 2");
  if (nx <= 0 || ny <= 0 || nz <= 0 || nzl <= 0 || z0 < 0 || z0 + nzl > nz)
    return set_err(TSLB_EINVAL, "allocate_fields: bad dims");
  if (lattice == kD2Q9 && nz != 1) return set_err(TSLB_EINVAL, "allocate_fields: d2q9 needs nz = 1");
  if (!kinds || !uw) return set_err(TSLB_EINVAL, "face arrays are required");
  if (int rc = check_axes(kinds)) return rc;
  const bool decomposed = nzl != nz;
  CK(cudaSetDevice(device));

  auto* h = new tslb_cuda_sim();
  h->lat = lattice;
  h->scalar = scalar;
  h->comps = components;
  h->esz = scalar == TSLB_F64 ? 8 : 4;
  lattice_of(lattice, [&](auto L) {
    using Lat = decltype(L);
    h->q = Lat::q;
    h->dim = Lat::dim;
    for (int a = 0; a < Lat::q; ++a) {
      if (Lat::c[a][2] == 1) {
        h->zpx[h->nzp] = Lat::c[a][0];
        h->zpy[h->nzp] = Lat::c[a][1];
        h->zp[h->nzp++] = a;
      }
      if (Lat::c[a][2] == -1) {
        h->zmx[h->nzm] = Lat::c[a][0];
        h->zmy[h->nzm] = Lat::c[a][1];
        h->zm[h->nzm++] = a;
      }
    }
  });
  h->np = h->dim * (h->dim + 1) / 2;
  h->nx = nx;
  h->ny = ny;
  h->nzl = nzl;
  h->z0 = z0;
  h->nzg = nz;
  h->decomposed = decomposed;
  h->device = device;
  h->omega = omega;
  if (const char* e = std::getenv("TSLB_STREAMCOLL"))
    h->variant = !std::strcmp(e, "scalar") ? 0 : 1;
  if (const char* e = std::getenv("TSLB_VX")) h->vx = std::atoi(e);
  if (const char* e = std::getenv("TSLB_KZ")) h->kz = std::atoi(e);
  if (const char* e = std::getenv("TSLB_GRAPHS")) h->graphs_ok = std::atoi(e) != 0;
  if (const char* e = std::getenv("TSLB_LZ")) h->lz = std::atoi(e);
  if (const char* e = std::getenv("TSLB_LZB")) h->lzb = std::atoi(e);
  std::memcpy(h->kinds, kinds, sizeof h->kinds);
  if (color) {
    h->cp.sigma = color[0];
    h->cp.beta = color[1];
    h->cp.nci_strength = color[2];
    h->cp.eps_bulk = color[3];
    h->cp.grad_threshold = color[4];
  } else {
    h->cp.sigma = 0.01;
    h->cp.beta = 0.7;
    h->cp.nci_strength = 0;
    h->cp.eps_bulk = 0.02;
    h->cp.grad_threshold = 1e-6;
  }
  h->cp.nci_reach = color_i ? color_i[0] : 3;
  h->cp.linear = color_i ? color_i[1] : 0;

  Dom& d = h->d;
  d.nx = nx;
  d.ny = ny;
  d.nz = nzl;
  d.ghost = decomposed ? 1 : 0;
  d.plane = h->plane();
  d.n = h->n();
  d.fstride = round_up(d.plane * (nzl + 2 * d.ghost), 64);
  d.mstride = round_up(d.n, 64);
  for (int fc = 0; fc < 6; ++fc) {
    d.mode[fc] = kinds[fc] == TSLB_FACE_PERIODIC ? kWrap : kWall;
    for (int c = 0; c < 3; ++c)
      d.uw[fc][c] = scalar == TSLB_F32 ? double(float(uw[3 * fc + c])) : uw[3 * fc + c];
  }
  if (decomposed) {
    if (!(z0 == 0 && kinds[ZMin] != TSLB_FACE_PERIODIC)) d.mode[ZMin] = kGhost;
    if (!(z0 + nzl == nz && kinds[ZMax] != TSLB_FACE_PERIODIC)) d.mode[ZMax] = kGhost;
  }
  d.has_solid = 0;
  if (solid)
    for (int64_t t = 0, N = int64_t(nx) * ny * nz; t < N; ++t)
      if (solid[t]) {
        d.has_solid = 1;
        break;
      }
  if (decomposed && components == 2 && d.has_solid) {
    delete h;
    return set_err(TSLB_EINVAL, "two-fluid slabs: box geometries only (no solid mask)");
  }
  d.xblocks = (nx + 127) / 128;
  d.k0 = 0;
  d.nzr = nzl;

  int rc = 0;
  auto fail = [&](int r) {
    tslb_cuda_destroy(h);
    return r;
  };
  CK(cudaStreamCreateWithFlags(&h->s, cudaStreamNonBlocking));
  // the halo stream runs at the highest priority: its NCCL kernels get SMs
  // ahead of the queued CTAs of the interior chunks they overlap with
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CK(cudaStreamCreateWithPriority(&h->cs, cudaStreamNonBlocking, prio_hi));
  CK(cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_c, cudaEventDisableTiming));
  CK(cudaEventCreate(&h->t0));
  CK(cudaEventCreate(&h->t1));

  const size_t mbytes = size_t(d.mstride) * (1 + h->dim + h->np) * h->esz;
  if ((rc = alloc(h, &h->mo, mbytes))) return fail(rc);
  CK(cudaMemsetAsync(h->mo, 0, mbytes, h->s));
  if (components == 2) {
    const size_t tb = size_t(d.mstride) * (3 + h->dim) * h->esz;
    if ((rc = alloc(h, &h->two, tb))) return fail(rc);
    CK(cudaMemsetAsync(h->two, 0, tb, h->s));
    const bool nci = nci_on(h);
    if (decomposed) {
      // the near-contact scan probes nci_reach nodes along +-c: phi (and the
      // flags it may set) need that many ghost planes on each side
      h->pgz = nci ? std::max(1, h->cp.nci_reach) : 1;
      if (nzl < h->pgz)
        return fail(set_err(TSLB_EINVAL, "two-fluid slab of %d planes is thinner than nci_reach = %d", nzl, h->pgz));
      const size_t pg = size_t(d.plane) * (nzl + 2 * h->pgz) * h->esz;
      if ((rc = alloc(h, &h->phig, pg))) return fail(rc);
      CK(cudaMemsetAsync(h->phig, 0, pg, h->s));
    }
    if (decomposed && nci) {
      const size_t gp = size_t(h->pgz) * size_t(d.plane);
      const size_t fb = 2 * gp + size_t(d.mstride);
      if ((rc = alloc(h, reinterpret_cast<void**>(&h->flagg), fb))) return fail(rc);
      CK(cudaMemsetAsync(h->flagg, 0, fb, h->s));
      h->flag = h->flagg + gp;
      if ((rc = alloc(h, reinterpret_cast<void**>(&h->rflag), 2 * gp))) return fail(rc);
    } else {
      if ((rc = alloc(h, reinterpret_cast<void**>(&h->flag), size_t(d.mstride)))) return fail(rc);
      CK(cudaMemsetAsync(h->flag, 0, size_t(d.mstride), h->s));
    }
  }
  // solid mask with ghost planes (always present: 1 B/node)
  const size_t sbytes = size_t(d.fstride);
  if ((rc = alloc(h, reinterpret_cast<void**>(&h->solid), sbytes))) return fail(rc);
  CK(cudaMemsetAsync(h->solid, 0, sbytes, h->s));
  if (d.has_solid) {
    // owned planes + ghost planes (z wraps for periodic global boundaries)
    std::vector<uint8_t> hs(size_t(d.plane) * (nzl + 2 * d.ghost), 0);
    for (int k = -d.ghost; k < nzl + d.ghost; ++k) {
      int kg = z0 + k;
      if (kg < 0 || kg >= nz) {
        if (kinds[ZMin] != TSLB_FACE_PERIODIC) continue;
        kg = (kg + nz) % nz;
      }
      std::memcpy(hs.data() + size_t(k + d.ghost) * d.plane,
                  solid + size_t(kg) * d.plane, size_t(d.plane));
    }
    CK(cudaMemcpyAsync(h->solid, hs.data(), hs.size(), cudaMemcpyHostToDevice, h->s));
    CK(cudaStreamSynchronize(h->s));
  }
  if (d.has_solid || components == 2) {
    if ((rc = alloc(h, reinterpret_cast<void**>(&h->slow), size_t(d.mstride) * 4))) return fail(rc);
    if ((rc = run_classify(h, h->slow))) return fail(rc);
  } else {
    // box geometry: every non-solid node is fluid
    h->n_fluid = uint64_t(d.n);
  }
  // A ghost-plane slot is written by the neighbour only if its source node is
  // fluid and the push did not cross an x/y wall; with solids or x/y walls
  // the received planes are staged and unpacked under that mask.
  h->staged = decomposed && (d.has_solid || d.mode[XMin] == kWall || d.mode[YMin] == kWall);
  if (h->staged) {
    const size_t pb = size_t(d.plane) * 9 * components * h->esz;
    if ((rc = alloc(h, &h->recv_lo, pb))) return fail(rc);
    if ((rc = alloc(h, &h->recv_hi, pb))) return fail(rc);
  }
  if (components == 1 && mstep_supported(lattice, d, h->esz)) {
    const char* e = std::getenv("TSLB_SCHEDULE");
    // M needs a second moment buffer (and ghost planes on slabs); where HBM
    // cannot hold it (e.g. D3Q27 1024^3 fp32) the solver stays on F1
    if (!(e && !std::strcmp(e, "f1"))) {
      // (slabs: the ghost planes and the packed send buffer, [2][NM][plane] each)
      const size_t gb = decomposed ? size_t(d.plane) * 2 * (1 + h->dim + h->np) * h->esz : 0;
      // masked geometries: 4 B of solid bits per node (+ the ghost planes)
      const size_t sb = d.has_solid ? size_t(d.plane) * (nzl + 2 * d.ghost) * 4 : 0;
      if (cudaMalloc(&h->mo2, mbytes) == cudaSuccess &&
          (!gb || cudaMalloc(&h->gm, gb) == cudaSuccess) && (!gb || cudaMalloc(&h->sx, gb) == cudaSuccess) &&
          (!sb || cudaMalloc(reinterpret_cast<void**>(&h->sbits), sb) == cudaSuccess)) {
        h->bytes += mbytes + 2 * gb + sb;
        CK(cudaMemsetAsync(h->mo2, 0, mbytes, h->s));
        if (gb) CK(cudaMemsetAsync(h->gm, 0, gb, h->s));
        if (gb) CK(cudaMemsetAsync(h->sx, 0, gb, h->s));
        if (sb && launch_solid_bits(lattice, d, h->solid, h->sbits, h->s))
          return fail(set_err(TSLB_ECUDA, "solid bits: launch failed"));
        h->sched = TSLB_SCHED_M;
      } else {
        cudaGetLastError();  // clear the allocation failure
        if (h->mo2) cudaFree(h->mo2);
        if (h->gm) cudaFree(h->gm);
        if (h->sx) cudaFree(h->sx);
        h->mo2 = nullptr;
        h->gm = nullptr;
        h->sx = nullptr;
      }
    }
  }
  // populations: always for two-fluid and F1; under M the single-fluid f is
  // only allocated when something needs it (ensure_f)
  if (components == 2 || h->sched != TSLB_SCHED_M) {
    const size_t fbytes = size_t(d.fstride) * h->q * h->esz;
    for (int sp = 0; sp < components; ++sp) {
      if ((rc = alloc(h, &h->f[sp], fbytes))) return fail(rc);
      CK(cudaMemsetAsync(h->f[sp], 0, fbytes, h->s));
    }
  }
  if ((rc = alloc(h, reinterpret_cast<void**>(&h->red),
                  (reduce_partial_count() + 16) * sizeof(double))))
    return fail(rc);
  CK(cudaStreamSynchronize(h->s));
  *out = h;
  return 0;
}

int sync(tslb_cuda_sim* h) {
  CK(cudaStreamSynchronize(h->s));
  CK(cudaGetLastError());
  return 0;
}

void drop_graph(tslb_cuda_sim* h) {
  if (h->graph) cudaGraphExecDestroy(h->graph);
  h->graph = nullptr;
}

// Second population buffer of the two-buffer reference step / stream_only
// (the reference's `scratch`, kernels.hpp:219-291). Created on first use as a
// copy of f, like `auto scratch = b.f` in the reference tests.
int ensure_scratch(tslb_cuda_sim* h) {
  if (h->scratch) return 0;
  if (int rc = materialize(h)) return rc;
  if (int rc = ensure_f(h)) return rc;
  const size_t fbytes = size_t(h->d.fstride) * h->q * h->esz;
  if (int rc = alloc(h, &h->scratch, fbytes)) return rc;
  CK(cudaMemcpyAsync(h->scratch, h->f[0], fbytes, cudaMemcpyDeviceToDevice, h->s));
  return 0;
}

// base of population species 0/1 (f / fr, fb) or 2 (scratch buffer)
int species_base(tslb_cuda_sim* h, int species, char** base, bool overwrite = false) {
  if (species == 0 && h->comps == 1) {
    if (overwrite) {
      // every owned slot is about to be replaced: no pending f(0) to fill
      h->f0_pending = false;
      h->m0_ready = false;
    }
    if (int rc = ensure_f(h)) return rc;
  }
  if (species == 2 && h->comps == 1 && !h->decomposed) {
    if (int rc = ensure_scratch(h)) return rc;
    *base = static_cast<char*>(h->scratch);
    return 0;
  }
  if (species < 0 || species >= h->comps) return set_err(TSLB_EINVAL, "bad species %d", species);
  *base = static_cast<char*>(h->f[species]);
  return 0;
}

}  // namespace

// ============================================================================
extern "C" {

int tslb_cuda_abi_version(void) { return TSLB_CUDA_ABI_VERSION; }
const char* tslb_cuda_last_error(void) { return g_err.c_str(); }

int tslb_cuda_device_count(int* count) {
  CK(cudaGetDeviceCount(count));
  return 0;
}

int tslb_cuda_create(int lattice, int scalar, int components, int nx, int ny,
                     int nz, double omega, const int* face_kind,
                     const double* face_uwall, const uint8_t* solid,
                     const double* color, const int* color_i, int device,
                     tslb_cuda_handle* out) {
  return create_impl(lattice, scalar, components, nx, ny, nz, 0, nz, omega,
                     face_kind, face_uwall, solid, color, color_i, device, out);
}

int tslb_cuda_create_slab(int lattice, int scalar, int components, int nx,
                          int ny, int nz, int z0, int nz_local, double omega,
                          const int* face_kind, const double* face_uwall,
                          const uint8_t* solid, const double* color,
                          const int* color_i, int device,
                          tslb_cuda_handle* out) {
  return create_impl(lattice, scalar, components, nx, ny, nz, z0, nz_local,
                     omega, face_kind, face_uwall, solid, color, color_i,
                     device, out);
}

int tslb_cuda_destroy(tslb_cuda_handle h) {
  if (!h) return 0;
  cudaSetDevice(h->device);
  if (h->s) cudaStreamSynchronize(h->s);
  if (h->cs) cudaStreamSynchronize(h->cs);
  if (h->comm && nccl().CommDestroy) nccl().CommDestroy(h->comm);
  if (h->ipc_up_mapped) cudaIpcCloseMemHandle(h->ipc_up);
  if (h->ipc_down_mapped && h->ipc_down != h->ipc_up) cudaIpcCloseMemHandle(h->ipc_down);
  if (h->ipc_blk) {
    const char* g = static_cast<const char*>(h->gm);
    if (g >= h->ipc_blk && g < h->ipc_blk + kIpcFlags + 2 * h->ipc_gb) h->gm = nullptr;  // (inside the block)
    cudaFree(h->ipc_blk);
  }
  void* bufs[] = {h->f[0], h->f[1], h->falt[0], h->falt[1], h->mo, h->mo2, h->gm, h->sx, h->phig, h->two,
                  h->flagg ? h->flagg : h->flag, h->rflag, h->solid, h->slow,
                  h->sbits, h->scratch, h->state_buf, h->mh, h->mh2, h->red, h->dig, h->recv_lo, h->recv_hi};
  for (void* b : bufs)
    if (b) cudaFree(b);
  if (h->graph) cudaGraphExecDestroy(h->graph);
  free_mstep_maps(h->mmaps);
  for (auto e : h->pool) cudaEventDestroy(e);
  cudaEvent_t evs[] = {h->ev_b, h->ev_c, h->t0, h->t1};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  if (h->s) cudaStreamDestroy(h->s);
  if (h->cs) cudaStreamDestroy(h->cs);
  delete h;
  return 0;
}

int tslb_cuda_set_math(tslb_cuda_handle h, int math) {
  if (int rc = settle(h)) return rc;
  if (math != kMathDouble && math != kMathFloat) return set_err(TSLB_EINVAL, "bad math mode");
  CK(cudaSetDevice(h->device));
  // a pending f(t+1) belongs to the step that was taken with the old mode
  if (int rc = materialize(h)) return rc;
  h->m0_ready = false;  // the initialiser's moments used the old arithmetic
  h->math = math;
  drop_graph(h);
  return 0;
}

int tslb_cuda_set_schedule(tslb_cuda_handle h, int schedule) {
  if (int rc = settle(h)) return rc;
  if (schedule != TSLB_SCHED_F1 && schedule != TSLB_SCHED_M)
    return set_err(TSLB_EINVAL, "bad schedule %d", schedule);
  if (schedule == h->sched) return 0;
  CK(cudaSetDevice(h->device));
  if (schedule == TSLB_SCHED_M) {
    if (h->comps != 1 || !mstep_supported(h->lat, h->d, h->esz))
      return set_err(TSLB_EINVAL,
                     "M schedule needs a single-fluid D3Q19/D3Q27 domain whose x rows are a multiple of "
                     "16 bytes (or D2Q9 whole domains without solids)");
    if (!h->mo2) {
      const size_t mbytes = size_t(h->d.mstride) * (1 + h->dim + h->np) * h->esz;
      if (int rc = alloc(h, &h->mo2, mbytes)) return rc;
    }
    if (h->decomposed && !h->gm) {
      const size_t gb = size_t(h->plane()) * 2 * (1 + h->dim + h->np) * h->esz;
      if (int rc = alloc(h, &h->gm, gb)) return rc;
      if (int rc = alloc(h, &h->sx, gb)) return rc;
      CK(cudaMemsetAsync(h->gm, 0, gb, h->s));
      CK(cudaMemsetAsync(h->sx, 0, gb, h->s));
    }
    if (h->d.has_solid && !h->sbits) {
      if (int rc = alloc(h, reinterpret_cast<void**>(&h->sbits),
                         size_t(h->plane()) * (h->nzl + 2 * h->d.ghost) * 4))
        return rc;
      if (launch_solid_bits(h->lat, h->d, h->solid, h->sbits, h->s))
        return set_err(TSLB_ECUDA, "solid bits: launch failed");
    }
  } else {
    if (int rc = materialize(h)) return rc;
    h->m0_ready = false;
  }
  h->sched = schedule;
  drop_graph(h);
  return sync(h);
}

int tslb_cuda_set_body_force(tslb_cuda_handle h, const double* force) {
  if (int rc = settle(h)) return rc;
  if (!force) return set_err(TSLB_EINVAL, "null force");
  if (h->comps != 1) return set_err(TSLB_EINVAL, "the body force is a single-fluid extension");
  CK(cudaSetDevice(h->device));
  // a pending f(t+1) = stream_collide(m(t)) does not depend on F; the
  // initialiser's precomputed moments do
  h->m0_ready = false;
  Dom& d = h->d;
  d.forced = force[0] != 0.0 || force[1] != 0.0 || force[2] != 0.0;
  // tau = 1 / omega with omega stored as T; F rounded to T (the
  // CollisionParams<T> convention); products in double as on the host
  const double omega_t = h->scalar == TSLB_F32 ? double(float(h->omega)) : h->omega;
  const double tau = 1.0 / omega_t;
  for (int c = 0; c < 3; ++c) {
    const double fc = h->scalar == TSLB_F32 ? double(float(force[c])) : force[c];
    d.tf[c] = (c < h->dim) ? tau * fc : 0.0;
  }
  drop_graph(h);
  return 0;
}

int tslb_cuda_get_schedule(tslb_cuda_handle h, int* schedule) {
  *schedule = h->sched;
  return 0;
}

int tslb_cuda_describe(tslb_cuda_handle h, int* dims, int* info) {
  if (dims) {
    dims[0] = h->nx;
    dims[1] = h->ny;
    dims[2] = h->nzl;
    dims[3] = h->z0;
    dims[4] = h->nzg;
  }
  if (info) {
    info[0] = h->q;
    info[1] = h->dim;
    info[2] = h->np;
    info[3] = h->esz;
  }
  return 0;
}

int tslb_cuda_memory_bytes(tslb_cuda_handle h, uint64_t* bytes) {
  *bytes = h->bytes;
  return 0;
}

int tslb_cuda_upload_f(tslb_cuda_handle h, int species, const void* host) {
  if (int rc = settle(h)) return rc;
  h->m16_valid = false;
  CK(cudaSetDevice(h->device));
  char* base;
  if (species == 0) h->fimplicit = false;  // every owned slot is overwritten
  if (int rc = species_base(h, species, &base, true)) return rc;
  const size_t pb = size_t(h->n()) * h->esz;
  const size_t off = size_t(h->d.ghost * h->plane()) * h->esz;
  for (int a = 0; a < h->q; ++a)
    CK(cudaMemcpyAsync(base + size_t(a) * h->d.fstride * h->esz + off,
                       static_cast<const char*>(host) + a * pb, pb,
                       cudaMemcpyHostToDevice, h->s));
  return sync(h);
}

int tslb_cuda_download_f(tslb_cuda_handle h, int species, void* host) {
  CK(cudaSetDevice(h->device));
  if (species == 0)
    if (int rc = materialize(h)) return rc;
  char* base;
  if (int rc = species_base(h, species, &base)) return rc;
  const size_t pb = size_t(h->n()) * h->esz;
  const size_t off = size_t(h->d.ghost * h->plane()) * h->esz;
  for (int a = 0; a < h->q; ++a)
    CK(cudaMemcpyAsync(static_cast<char*>(host) + a * pb,
                       base + size_t(a) * h->d.fstride * h->esz + off, pb,
                       cudaMemcpyDeviceToHost, h->s));
  return sync(h);
}

namespace {
// (device base, number of arrays, element bytes) for a field id
int field_desc(tslb_cuda_sim* h, int field, void** base, int* count, int* eb,
               int64_t* stride, bool upload) {
  *eb = h->esz;
  *stride = h->d.mstride;
  const bool two = h->comps == 2;
  switch (field) {
    case TSLB_FIELD_RHO: *base = h->m_arr(0); *count = 1; return 0;
    case TSLB_FIELD_MOM: *base = h->m_arr(1); *count = h->dim; return 0;
    case TSLB_FIELD_PINEQ: *base = h->m_arr(1 + h->dim); *count = h->np; return 0;
    case TSLB_FIELD_RHO_R: if (!two) break; *base = h->t_arr(0); *count = 1; return 0;
    case TSLB_FIELD_RHO_B: if (!two) break; *base = h->t_arr(1); *count = 1; return 0;
    case TSLB_FIELD_PHI: if (!two) break; *base = h->tf().phi; *count = 1; return 0;
    case TSLB_FIELD_GRADPHI: if (!two) break; *base = h->t_arr(3); *count = h->dim; return 0;
    case TSLB_FIELD_NCI_FLAG: if (!two) break; *base = h->flag; *count = 1; *eb = 1; return 0;
    case TSLB_FIELD_SOLID:
      if (upload) break;
      *base = static_cast<char*>(static_cast<void*>(h->solid)) + h->d.ghost * h->plane();
      *count = 1; *eb = 1; return 0;
    case TSLB_FIELD_SLOW_MASK:
      if (upload || !h->slow) break;
      *base = h->slow; *count = 1; *eb = 4; return 0;
    default: break;
  }
  return set_err(TSLB_EINVAL, "field %d not available for this solver%s", field,
                 upload ? " (or read-only)" : "");
}
}  // namespace

int tslb_cuda_upload_field(tslb_cuda_handle h, int field, const void* host) {
  if (int rc = settle(h)) return rc;
  h->m16_valid = false;
  void* base; int cnt, eb; int64_t stride;
  if (int rc = field_desc(h, field, &base, &cnt, &eb, &stride, true)) return rc;
  CK(cudaSetDevice(h->device));
  if (int rc = finish_gradient(h)) return rc;
  // the implicit f(t+1) is a function of the moment arrays being replaced
  if (int rc = materialize(h)) return rc;
  const size_t pb = size_t(h->n()) * eb;
  for (int c = 0; c < cnt; ++c)
    CK(cudaMemcpyAsync(static_cast<char*>(base) + size_t(c) * stride * eb,
                       static_cast<const char*>(host) + c * pb, pb,
                       cudaMemcpyHostToDevice, h->s));
  if (field == TSLB_FIELD_MOM || field == TSLB_FIELD_PINEQ) h->stress_pending = false;
  return sync(h);
}

int tslb_cuda_download_field(tslb_cuda_handle h, int field, void* host) {
  if (int rc = settle(h, true)) return rc;
  CK(cudaSetDevice(h->device));
  if (int rc = finish_gradient(h)) return rc;
  // two-fluid: after a step the host-visible mom/pineq are u_eq / Pi^neq
  // (prepare_stress output, multicomponent.hpp:271-309); the fused step keeps
  // the raw values on the device, so finish the phase lazily here.
  if (h->comps == 2 && h->stress_pending &&
      (field == TSLB_FIELD_MOM || field == TSLB_FIELD_PINEQ)) {
    if (int rc = ph_cg_prepare(h, h->s)) return rc;
  }
  if (field == TSLB_FIELD_SLOW_MASK && !h->slow) {
    uint32_t* tmp;
    CK(cudaMalloc(&tmp, size_t(h->d.mstride) * 4));
    if (int rc = run_classify(h, tmp)) { cudaFree(tmp); return rc; }
    CK(cudaMemcpy(host, tmp, size_t(h->n()) * 4, cudaMemcpyDeviceToHost));
    cudaFree(tmp);
    return 0;
  }
  void* base; int cnt, eb; int64_t stride;
  if (int rc = field_desc(h, field, &base, &cnt, &eb, &stride, false)) return rc;
  const size_t pb = size_t(h->n()) * eb;
  for (int c = 0; c < cnt; ++c)
    CK(cudaMemcpyAsync(static_cast<char*>(host) + c * pb,
                       static_cast<const char*>(base) + size_t(c) * stride * eb, pb,
                       cudaMemcpyDeviceToHost, h->s));
  return sync(h);
}

int tslb_cuda_download_slice(tslb_cuda_handle h, int field, int axis, int index, void* host) {
  if (int rc = settle(h, true)) return rc;
  if (axis < 0 || axis > 2) return set_err(TSLB_EINVAL, "slice axis must be 0, 1 or 2");
  const int ext[3] = {h->nx, h->ny, h->nzl};
  if (index < 0 || index >= ext[axis]) return set_err(TSLB_EINVAL, "slice index %d outside [0, %d)", index, ext[axis]);
  if (field == TSLB_FIELD_SLOW_MASK) return set_err(TSLB_EINVAL, "slices of the slow mask are not provided");
  CK(cudaSetDevice(h->device));
  if (int rc = finish_gradient(h)) return rc;
  if (h->comps == 2 && h->stress_pending && (field == TSLB_FIELD_MOM || field == TSLB_FIELD_PINEQ))
    if (int rc = ph_cg_prepare(h, h->s)) return rc;
  void* base; int cnt, eb; int64_t stride;
  if (int rc = field_desc(h, field, &base, &cnt, &eb, &stride, false)) return rc;
  // one strided 2-D copy per array: rows of `width` bytes, `rows` of them,
  // `spitch` apart in device memory, packed on the host
  const size_t nx = size_t(h->nx), ny = size_t(h->ny), nz = size_t(h->nzl);
  size_t off, width, spitch, rows;
  if (axis == 2) {         // x-y plane: contiguous
    off = size_t(index) * nx * ny; width = nx * ny * eb; spitch = width; rows = 1;
  } else if (axis == 1) {  // x-z plane: nz rows of nx, one plane apart
    off = size_t(index) * nx; width = nx * eb; spitch = nx * ny * eb; rows = nz;
  } else {                 // y-z plane: ny * nz single elements, one row apart
    off = size_t(index); width = eb; spitch = nx * eb; rows = ny * nz;
  }
  const size_t plane_bytes = width * rows;
  for (int c = 0; c < cnt; ++c)
    CK(cudaMemcpy2DAsync(static_cast<char*>(host) + c * plane_bytes, width,
                         static_cast<const char*>(base) + (size_t(c) * stride + off) * eb, spitch, width, rows,
                         cudaMemcpyDeviceToHost, h->s));
  return sync(h);
}

int tslb_cuda_download_geometry(tslb_cuda_handle h, uint8_t* solid,
                                uint32_t* slow_mask, uint64_t* n_fluid) {
  if (solid)
    if (int rc = tslb_cuda_download_field(h, TSLB_FIELD_SOLID, solid)) return rc;
  if (slow_mask)
    if (int rc = tslb_cuda_download_field(h, TSLB_FIELD_SLOW_MASK, slow_mask)) return rc;
  if (n_fluid) *n_fluid = h->n_fluid;
  return 0;
}

int tslb_cuda_init_analytic(tslb_cuda_handle h, int kind, double amplitude,
                            double radius) {
  if (int rc = settle(h)) return rc;
  h->m16_valid = false;
  CK(cudaSetDevice(h->device));
  InitSpec s{};
  s.kind = kind;
  s.nx_g = h->nx;
  s.ny_g = h->ny;
  s.nz_g = h->nzg;
  s.z0 = h->z0;
  s.amp = amplitude;
  s.cx = 0.5 * h->nx - 0.5;
  s.cy = 0.5 * h->ny - 0.5;
  s.cz = 0.5 * h->nzg - 0.5;
  s.radius = radius;
  s.width = 1.0;
  ++h->launches;
  int rc = by_scalar(h, [&](auto z) {
    using T = decltype(z);
    if (kind == TSLB_INIT_DROPLET) {
      if (h->comps != 2) return set_err(TSLB_EINVAL, "droplet init needs two components");
      return launch_init_colors<T>(h->lat, h->range(0, h->nzl), static_cast<T*>(h->f[0]),
                                   static_cast<T*>(h->f[1]), h->solid, s, h->s);
    }
    if (h->comps != 1) return set_err(TSLB_EINVAL, "analytic init %d needs one component", kind);
    h->fimplicit = false;
    if (h->sched == TSLB_SCHED_M && !h->d.has_solid) {
      // M: f(0) is not stored; the first step's moments pass is done here
      h->f0_spec = s;
      h->f0_pending = true;
      h->m0_ready = true;
      return launch_init_moments<T>(h->lat, h->math, h->range(0, h->nzl), static_cast<T*>(h->mo2), s, h->s);
    }
    h->f0_pending = false;
    h->m0_ready = false;
    if (int rc = ensure_f(h)) return rc;
    return launch_init_analytic<T>(h->lat, h->range(0, h->nzl), static_cast<T*>(h->f[0]),
                                   h->d.has_solid ? h->solid : nullptr, s, h->s);
  });
  if (rc) return rc;
  return sync(h);
}

// initialize_regularized (kernels.hpp:296-311) on the device from HOST node
// states: the state planes travel in z chunks on the copy (comm) stream and
// each chunk's kernel runs as soon as its planes have landed, so the PCIe
// transfer overlaps the initialisation. Under M (box geometry) the kernel
// writes the first step's moments directly and f(0) stays pending on the
// uploaded states (materialised only if read); otherwise f(0) is stored.
// with_pi: the host states carry Pi^neq (1+D+np arrays); without, they are
// rho and u only and Pi^neq = 0 (1+D arrays).
static int init_state(tslb_cuda_sim* h, const void* host, bool with_pi) {
  if (int rc = settle(h)) return rc;
  h->m16_valid = false;
  if (!host) return set_err(TSLB_EINVAL, "init_state: null state");
  if (h->comps != 1)
    return set_err(TSLB_EINVAL, "init_state: single-fluid node states (two-fluid: initialize_colors + upload_f)");
  CK(cudaSetDevice(h->device));
  const int nm = 1 + h->dim + (with_pi ? h->np : 0);
  const bool m_path = h->sched == TSLB_SCHED_M && !h->d.has_solid;
  h->fimplicit = false;
  h->f0_pending = false;
  h->m0_ready = false;
  // (ensure_f releases an earlier state buffer: allocate this one after it)
  if (!m_path)
    if (int rc = ensure_f(h)) return rc;
  if (h->state_buf && h->state_nm != nm) {
    CK(cudaFree(h->state_buf));
    h->state_buf = nullptr;
    h->bytes -= size_t(h->d.mstride) * h->state_nm * h->esz;
  }
  if (!h->state_buf) {
    if (int rc = alloc(h, &h->state_buf, size_t(h->d.mstride) * nm * h->esz)) return rc;
    h->state_nm = nm;
  }
  InitSpec sp{};
  sp.kind = kInitState;
  sp.nx_g = h->nx;
  sp.ny_g = h->ny;
  sp.nz_g = h->nzg;
  sp.z0 = h->z0;
  sp.state = h->state_buf;
  sp.sstride = h->d.mstride;
  sp.spi = with_pi ? 1 : 0;
  // ~32 MB of each state array per chunk
  const int64_t plane = h->plane();
  const int cz = int(std::max<int64_t>(1, (int64_t(32) << 20) / (plane * h->esz)));
  const size_t pitch_h = size_t(h->n()) * h->esz, pitch_d = size_t(h->d.mstride) * h->esz;
  CK(cudaEventRecord(h->ev_b, h->s));  // (the buffers are free once earlier work is done)
  CK(cudaStreamWaitEvent(h->cs, h->ev_b, 0));
  for (int k0 = 0; k0 < h->nzl; k0 += cz) {
    const int k1 = std::min(h->nzl, k0 + cz);
    const size_t off = size_t(k0) * plane * h->esz;
    CK(cudaMemcpy2DAsync(static_cast<char*>(h->state_buf) + off, pitch_d, static_cast<const char*>(host) + off,
                         pitch_h, size_t(k1 - k0) * plane * h->esz, size_t(nm), cudaMemcpyHostToDevice, h->cs));
    CK(cudaEventRecord(h->ev_c, h->cs));
    CK(cudaStreamWaitEvent(h->s, h->ev_c, 0));
    ++h->launches;
    const int rc = by_scalar(h, [&](auto z) {
      using T = decltype(z);
      if (m_path)
        return launch_init_moments<T>(h->lat, h->math, h->range(k0, k1), static_cast<T*>(h->mo2), sp, h->s);
      return launch_init_analytic<T>(h->lat, h->range(k0, k1), static_cast<T*>(h->f[0]),
                                     h->d.has_solid ? h->solid : nullptr, sp, h->s);
    });
    if (rc) return set_err(TSLB_EINVAL, "init_state: bad lattice");
  }
  if (m_path) {
    h->f0_spec = sp;
    h->f0_pending = true;
    h->m0_ready = true;
    return sync(h);
  }
  // f(0) is stored: the states are no longer needed
  if (int rc = sync(h)) return rc;
  CK(cudaFree(h->state_buf));
  h->state_buf = nullptr;
  h->bytes -= size_t(h->d.mstride) * nm * h->esz;
  return 0;
}

int tslb_cuda_init_state(tslb_cuda_handle h, const void* host) { return init_state(h, host, true); }

int tslb_cuda_init_equilibrium(tslb_cuda_handle h, const void* host) { return init_state(h, host, false); }

int tslb_cuda_set_moment_storage(tslb_cuda_handle h, int kind) {
  if (kind != TSLB_STORE_NATIVE && kind != TSLB_STORE_F16) return set_err(TSLB_EINVAL, "bad moment storage %d", kind);
  CK(cudaSetDevice(h->device));
  if (kind == h->store16) return 0;
  if (kind == TSLB_STORE_NATIVE) {
    if (int rc = sync32(h)) return rc;
    CK(cudaStreamSynchronize(h->s));
    const size_t hb = size_t(h->d.mstride) * (1 + h->dim + h->np) * sizeof(__half);
    CK(cudaFree(h->mh));
    CK(cudaFree(h->mh2));
    h->mh = h->mh2 = nullptr;
    h->bytes -= 2 * hb;
    h->store16 = 0;
    return 0;
  }
  if (h->comps != 1 || h->scalar != TSLB_F32 || h->sched != TSLB_SCHED_M || h->decomposed ||
      !mstep16_supported(h->lat, h->d))
    return set_err(TSLB_EINVAL,
                   "fp16 moment storage needs a single-fluid fp32 D3Q19/D3Q27 whole domain on the M schedule, "
                   "without solids, nx %% 8 == 0");
  // fp16 storage is paired with fp32 node arithmetic
  if (h->math != kMathFloat)
    if (int rc = tslb_cuda_set_math(h, kMathFloat)) return rc;
  const size_t hb = size_t(h->d.mstride) * (1 + h->dim + h->np) * sizeof(__half);
  if (int rc = alloc(h, &h->mh, hb)) return rc;
  if (int rc = alloc(h, &h->mh2, hb)) return rc;
  drop_graph(h);
  h->graphs_ok = false;  // (the encode of the first fp16 step must not be replayed)
  h->store16 = 1;
  h->m16_valid = false;
  h->m32_valid = true;
  return 0;
}

int tslb_cuda_step_async(tslb_cuda_handle h, long nsteps) {
  if (h->xmode == 2) return set_err(TSLB_ESTATE, "locally linked slabs step with tslb_cuda_group_step");
  if (h->decomposed && h->xmode == 0)
    return set_err(TSLB_ESTATE, "slab solver has no halo transport attached");
  CK(cudaSetDevice(h->device));
  long done = 0;
  if (h->mvis2 && nsteps > 0) {
    // refreshed under M: the next step's moment pass already ran (mo2 =
    // m(t+1)); afterwards f(t+2) is implicit in it, whether or not f(t+1)
    // was materialised meanwhile
    std::swap(h->mo, h->mo2);
    h->mvis2 = false;
    h->fimplicit = true;
    ++h->steps;
    ++done;
  }
  // small 2-D domains under M: the whole run in persistent cooperative
  // launches (temporal blocking: a grid barrier every four passes) -- per-
  // pass launch overhead is most of their step time; TSLB_PERSIST=0 selects
  // the graph path instead. Up to 512^2 nodes: measured r02
  // (tools/micro/tb2d_sizes.py), 256^2 29.0 / 24.0 GLUPS (periodic / lid)
  // persistent vs 17.5 / 16.1 from graphs, 512^2 36.7 / 30.9 vs 36.8 / 28.7,
  // 640^2 39.3 / 33.1 vs 42.7 / 33.5
  const char* pmx = std::getenv("TSLB_PERSIST_MAX");  // (nodes; measurements)
  const int64_t kPersistMaxNodes = pmx ? std::atoll(pmx) : int64_t(1) << 18;
  const char* pe = std::getenv("TSLB_PERSIST");
  const bool persist = !(pe && std::atoi(pe) == 0);
  if (persist && h->sched == TSLB_SCHED_M && h->dim == 2 && h->comps == 1 && h->xmode == 0 && !h->decomposed &&
      !h->d.has_solid && h->n() <= kPersistMaxNodes && nsteps >= 3) {
    if (!h->fimplicit) {
      if (int rc = enqueue_step(h)) return rc;
      ++done;
    }
    while (nsteps - done >= 2) {
      const int n = int(std::min<long>(nsteps - done, 1L << 20));
      int rc;
      {
        Prof p(h, TSLB_K_MSTEP, h->s);
        rc = by_scalar(h, [&](auto z) {
          using T = decltype(z);
          return launch_mstep2d_persist<T>(h->math, h->range(0, h->nzl), static_cast<T*>(h->mo),
                                           static_cast<T*>(h->mo2), h->omega, n, h->s);
        });
      }
      if (rc < 0) return set_err(TSLB_ECUDA, "k_mstep2d_persist launch: %s", cudaGetErrorString(cudaError_t(-rc)));
      if (rc) break;  // not co-resident: the regular launches below
      ++h->launches;
      if (n & 1) std::swap(h->mo, h->mo2);
      h->steps += n;
      done += n;
    }
  }
  // small domains are launch bound: replay a captured graph of G steps
  constexpr int64_t kGraphMaxNodes = int64_t(8) << 20;
  constexpr long kGraphSteps = 32;  // even: an M graph ends on the buffer it starts from
  // (steps still owed only: the persistent path above may have run them all)
  // (not for the two-fluid one-pass step: its population buffers alternate)
  if (h->graphs_ok && !h->prof && h->xmode == 0 && h->n() <= kGraphMaxNodes && nsteps - done >= kGraphSteps &&
      !cg_fused_on(h)) {
    // an M graph replays M passes only: leave the stored-f state first, and
    // start from the moment buffer the graph was captured on
    if (h->sched == TSLB_SCHED_M) {
      if (!h->fimplicit && done < nsteps) {
        if (int rc = enqueue_step(h)) return rc;
        ++done;
      }
      if (h->graph && h->graph_mo != h->mo && done < nsteps) {
        if (int rc = enqueue_step(h)) return rc;
        ++done;
      }
    }
    if (!h->graph && nsteps - done >= kGraphSteps) {
      h->graph_mo = h->mo;
      const long steps0 = h->steps;
      const int64_t l0 = h->launches;
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
      int rc = 0;
      for (long k = 0; k < kGraphSteps && !rc; ++k) rc = enqueue_step(h);
      cudaError_t ce = cudaStreamEndCapture(h->s, &g);
      h->steps = steps0;
      h->grad_pending_after_graph = h->grad_pending;
      h->graph_launches = h->launches - l0;
      h->launches = l0;
      if (rc) return rc;
      if (ce != cudaSuccess) return set_err(TSLB_ECUDA, "graph capture: %s", cudaGetErrorString(ce));
      ce = cudaGraphInstantiate(&h->graph, g, 0);
      cudaGraphDestroy(g);
      if (ce != cudaSuccess) return set_err(TSLB_ECUDA, "graph instantiate: %s", cudaGetErrorString(ce));
      h->graph_steps = kGraphSteps;
    }
    for (; h->graph && done + h->graph_steps <= nsteps; done += h->graph_steps) {
      CK(cudaGraphLaunch(h->graph, h->s));
      h->steps += h->graph_steps;
      h->launches += h->graph_launches;
      if (h->comps == 2) {
        h->stress_pending = true;
        h->grad_pending = h->grad_pending_after_graph;
      }
    }
  }
  for (long k = done; k < nsteps; ++k)
    if (int rc = enqueue_step(h)) return rc;
  CK(cudaGetLastError());
  return 0;
}

int tslb_cuda_step(tslb_cuda_handle h, long nsteps) {
  if (int rc = tslb_cuda_step_async(h, nsteps)) return rc;
  return sync(h);
}

int tslb_cuda_synchronize(tslb_cuda_handle h) {
  CK(cudaSetDevice(h->device));
  return sync(h);
}

int tslb_cuda_steps_done(tslb_cuda_handle h, long* steps) {
  *steps = h->steps;
  return 0;
}

int tslb_cuda_time_steps(tslb_cuda_handle h, long nsteps, double* ms) {
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->s));
  CK(cudaEventRecord(h->t0, h->s));
  if (int rc = tslb_cuda_step_async(h, nsteps)) return rc;
  CK(cudaEventRecord(h->t1, h->s));
  CK(cudaEventSynchronize(h->t1));
  float f = 0;
  CK(cudaEventElapsedTime(&f, h->t0, h->t1));
  *ms = f;
  return sync(h);
}

int tslb_cuda_compute_moments(tslb_cuda_handle h) {
  if (int rc = settle(h)) return rc;
  if (h->comps != 1) return set_err(TSLB_EINVAL, "compute_moments is single-fluid");
  CK(cudaSetDevice(h->device));
  if (int rc = materialize(h)) return rc;
  if (int rc = ph_moments(h, h->s)) return rc;
  return sync(h);
}

int tslb_cuda_stream_collide(tslb_cuda_handle h) {
  if (int rc = settle(h)) return rc;
  if (h->comps != 1) return set_err(TSLB_EINVAL, "stream_collide_fused is single-fluid");
  if (h->decomposed) return set_err(TSLB_ESTATE, "use step() on slab solvers");
  CK(cudaSetDevice(h->device));
  if (int rc = materialize(h)) return rc;
  h->m0_ready = false;
  if (int rc = ph_streamcoll(h, 0, h->nzl, h->s)) return rc;
  return sync(h);
}

int tslb_cuda_reference_step(tslb_cuda_handle h, long nsteps) {
  if (int rc = settle(h)) return rc;
  if (h->comps != 1 || h->decomposed)
    return set_err(TSLB_EINVAL, "reference_step: single-fluid, single domain only");
  CK(cudaSetDevice(h->device));
  if (int rc = materialize(h)) return rc;
  h->m0_ready = false;
  if (int rc = ensure_scratch(h)) return rc;
  for (long s = 0; s < nsteps; ++s) {
    if (int rc = ph_moments(h, h->s)) return rc;
    h->launches += 2;
    int rc = by_scalar(h, [&](auto z) {
      using T = decltype(z);
      launch_collide<T>(h->lat, h->range(0, h->nzl), static_cast<T*>(h->f[0]),
                        static_cast<const T*>(h->mo), h->solid, h->omega, h->s);
      return launch_stream_only<T>(h->lat, h->range(0, h->nzl),
                                   static_cast<const T*>(h->f[0]),
                                   static_cast<T*>(h->scratch), h->solid, h->slow, h->s);
    });
    if (rc) return rc;
    std::swap(h->f[0], h->scratch);
    drop_graph(h);  // the captured graph addresses the old f buffer
    ++h->steps;
  }
  return sync(h);
}

int tslb_cuda_stream_only(tslb_cuda_handle h) {
  if (int rc = settle(h)) return rc;
  if (h->comps != 1 || h->decomposed)
    return set_err(TSLB_EINVAL, "stream_only: single-fluid, single domain only");
  CK(cudaSetDevice(h->device));
  if (int rc = materialize(h)) return rc;
  h->m0_ready = false;
  // pushes f into the second buffer (its slots not reached by any push keep
  // their contents, as in the reference), then swaps the two
  if (int rc = ensure_scratch(h)) return rc;
  ++h->launches;
  int rc = by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_stream_only<T>(h->lat, h->range(0, h->nzl),
                                 static_cast<const T*>(h->f[0]),
                                 static_cast<T*>(h->scratch), h->solid, h->slow, h->s);
  });
  if (rc) return rc;
  std::swap(h->f[0], h->scratch);
  drop_graph(h);
  return sync(h);
}

int tslb_cuda_color_moments(tslb_cuda_handle h) {
  if (h->comps != 2) return set_err(TSLB_EINVAL, "color_moments is two-fluid");
  CK(cudaSetDevice(h->device));
  if (int rc = finish_gradient(h)) return rc;
  if (int rc = ph_cg_moments(h, h->s)) return rc;
  return sync(h);
}

int tslb_cuda_gradient_and_nci(tslb_cuda_handle h) {
  if (h->comps != 2) return set_err(TSLB_EINVAL, "gradient_and_nci is two-fluid");
  CK(cudaSetDevice(h->device));
  if (int rc = ph_cg_gradient(h, h->s)) return rc;
  return sync(h);
}

int tslb_cuda_prepare_stress(tslb_cuda_handle h) {
  if (h->comps != 2) return set_err(TSLB_EINVAL, "prepare_stress is two-fluid");
  CK(cudaSetDevice(h->device));
  if (int rc = finish_gradient(h)) return rc;
  if (int rc = ph_cg_prepare(h, h->s)) return rc;
  return sync(h);
}

int tslb_cuda_stream_collide_recolor(tslb_cuda_handle h) {
  if (h->comps != 2) return set_err(TSLB_EINVAL, "stream_collide_recolor is two-fluid");
  CK(cudaSetDevice(h->device));
  if (int rc = finish_gradient(h)) return rc;
  if (int rc = ph_cg_streamcoll(h, 0, h->s)) return rc;
  return sync(h);
}

int tslb_cuda_refresh_moments(tslb_cuda_handle h) {
  if (int rc = sync32(h)) return rc;
  CK(cudaSetDevice(h->device));
  if (h->mvis2) return 0;  // (already refreshed)
  if (h->comps == 1 && h->sched == TSLB_SCHED_M && h->fimplicit && !h->decomposed && !h->store16) {
    // M: the moments of f(t+1) are one more moment-resident pass from m(t)
    // (80 B per node instead of storing f and re-reading it); mo keeps m(t)
    // for f(t+1), the host sees mo2 until the next step takes it over
    if (int rc = ph_mstep(h, h->s)) return rc;
    h->mvis2 = true;
    return sync(h);
  }
  if (h->comps == 1) {
    if (int rc = materialize(h)) return rc;
    if (int rc = ph_moments(h, h->s)) return rc;
  } else {
    if (int rc = ph_cg_moments(h, h->s)) return rc;
    if (int rc = ph_cg_gradient(h, h->s)) return rc;
  }
  return sync(h);
}

int tslb_cuda_totals(tslb_cuda_handle h, double* mass, double* momentum3) {
  if (int rc = settle(h, true)) return rc;
  CK(cudaSetDevice(h->device));
  double* part = h->red;
  double* out = h->red + reduce_partial_count();
  h->launches += 2;
  by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_totals<T>(h->range(0, h->nzl), h->dim, static_cast<const T*>(h->m_arr(0)),
                            static_cast<const T*>(h->m_arr(1)), h->solid, part, out, h->s);
  });
  double v[4];
  CK(cudaMemcpyAsync(v, out, sizeof v, cudaMemcpyDeviceToHost, h->s));
  if (int rc = sync(h)) return rc;
  *mass = v[0];
  for (int c = 0; c < 3; ++c) momentum3[c] = c < h->dim ? v[1 + c] : 0.0;
  return 0;
}

int tslb_cuda_stability(tslb_cuda_handle h, int* finite, double* max_speed,
                        double* min_rho, double* max_rho, int64_t* first_bad) {
  if (int rc = settle(h, true)) return rc;
  CK(cudaSetDevice(h->device));
  if (int rc = finish_gradient(h)) return rc;
  if (h->comps == 2 && h->stress_pending)
    if (int rc = ph_cg_prepare(h, h->s)) return rc;
  double* part = h->red;
  double* out = h->red + reduce_partial_count();
  h->launches += 2;
  by_scalar(h, [&](auto z) {
    using T = decltype(z);
    return launch_stability<T>(h->range(0, h->nzl), h->dim, static_cast<const T*>(h->m_arr(0)),
                               static_cast<const T*>(h->m_arr(1)), h->solid, part, out, h->s);
  });
  double v[5];
  CK(cudaMemcpyAsync(v, out, sizeof v, cudaMemcpyDeviceToHost, h->s));
  if (int rc = sync(h)) return rc;
  if (finite) *finite = v[0] > 0.5;
  if (max_speed) *max_speed = v[1];
  if (min_rho) *min_rho = v[2];
  if (max_rho) *max_rho = v[3];
  if (first_bad) *first_bad = int64_t(v[4]);
  return 0;
}

int tslb_cuda_color_masses(tslb_cuda_handle h, double* red, double* blue) {
  if (h->comps != 2) return set_err(TSLB_EINVAL, "color_masses is two-fluid");
  CK(cudaSetDevice(h->device));
  double* part = h->red;
  double* out = h->red + reduce_partial_count();
  h->launches += 2;
  by_scalar(h, [&](auto z) {
    using T = decltype(z);
    // rho_r as "rho", rho_b as a one-component "mom"
    return launch_totals<T>(h->range(0, h->nzl), 1, static_cast<const T*>(h->t_arr(0)),
                            static_cast<const T*>(h->t_arr(1)), h->solid, part, out, h->s);
  });
  double v[4];
  CK(cudaMemcpyAsync(v, out, sizeof v, cudaMemcpyDeviceToHost, h->s));
  if (int rc = sync(h)) return rc;
  *red = v[0];
  *blue = v[1];
  return 0;
}

int tslb_cuda_plane_digests(tslb_cuda_handle h, uint64_t* out) {
  if (int rc = settle(h)) return rc;
  CK(cudaSetDevice(h->device));
  if (int rc = materialize(h)) return rc;
  if (h->comps == 1)
    if (int rc = ensure_f(h)) return rc;
  const int64_t plane_bytes = h->plane() * h->esz;
  const int64_t cpp = (plane_bytes + 16383) / 16384;
  const size_t need = size_t(h->q) * h->nzl * (cpp + 1) * sizeof(uint64_t);
  if (h->dig_bytes < need) {
    if (h->dig) cudaFree(h->dig);
    CK(cudaMalloc(&h->dig, need));
    h->dig_bytes = need;
  }
  uint64_t* chunk = h->dig;
  uint64_t* planes = h->dig + size_t(h->q) * h->nzl * cpp;
  for (int sp = 0; sp < h->comps; ++sp) {
    h->launches += 2;
    launch_plane_digest(h->range(0, h->nzl), h->f[sp], h->q, h->d.fstride,
                        int64_t(h->d.ghost) * h->plane(), h->esz, chunk, planes, h->s);
    CK(cudaMemcpyAsync(out + size_t(sp) * h->q * h->nzl, planes,
                       size_t(h->q) * h->nzl * sizeof(uint64_t),
                       cudaMemcpyDeviceToHost, h->s));
    if (int rc = sync(h)) return rc;
  }
  return 0;
}

int tslb_cuda_profile(tslb_cuda_handle h, int enable) {
  h->prof = enable != 0;
  h->rec.clear();
  h->pool_used = 0;
  return 0;
}

int tslb_cuda_profile_read(tslb_cuda_handle h, double* ms, int64_t* launches) {
  CK(cudaSetDevice(h->device));
  CK(cudaStreamSynchronize(h->s));
  CK(cudaStreamSynchronize(h->cs));
  for (int c = 0; c < TSLB_K_COUNT; ++c) {
    if (ms) ms[c] = 0;
    if (launches) launches[c] = 0;
  }
  for (auto& r : h->rec) {
    float t = 0;
    CK(cudaEventElapsedTime(&t, r.second.first, r.second.second));
    if (ms) ms[r.first] += t;
    if (launches) launches[r.first] += 1;
  }
  h->rec.clear();
  h->pool_used = 0;
  return 0;
}

int tslb_cuda_launch_count(tslb_cuda_handle h, int64_t* launches) {
  *launches = h->launches;
  return 0;
}

int tslb_cuda_nccl_unique_id(void* id128) {
  NcclApi& N = nccl();
  if (!N.ok) return set_err(TSLB_ECUDA, "libnccl.so.2 could not be loaded");
  ncclUniqueId id;
  ncclResult_t r = N.GetUniqueId(&id);
  if (r != ncclSuccess) return set_err(TSLB_ECUDA, "ncclGetUniqueId: %s", N.ErrStr(r));
  std::memcpy(id128, &id, sizeof id);
  return 0;
}

int tslb_cuda_attach_nccl(tslb_cuda_handle h, const void* id128, int nranks,
                          int rank) {
  NcclApi& N = nccl();
  if (!N.ok) return set_err(TSLB_ECUDA, "libnccl.so.2 could not be loaded");
  if (!h->decomposed) return set_err(TSLB_ESTATE, "attach_nccl needs a slab solver");
  CK(cudaSetDevice(h->device));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclResult_t r = N.CommInitRank(&h->comm, nranks, id, rank);
  if (r != ncclSuccess) return set_err(TSLB_ECUDA, "ncclCommInitRank: %s", N.ErrStr(r));
  h->rank = rank;
  h->nranks = nranks;
  h->up = h->d.mode[ZMax] == kGhost ? (rank + 1) % nranks : -1;
  h->down = h->d.mode[ZMin] == kGhost ? (rank - 1 + nranks) % nranks : -1;
  h->xmode = 1;
  return 0;
}

// peer-memory transport (CUDA IPC): export this slab's block of flag words
// and ghost planes ...
static int ipc_block(tslb_cuda_sim* h) {
  if (h->ipc_blk) return 0;
  const size_t gb = size_t(h->plane()) * 2 * (1 + h->dim + h->np) * h->esz;
  void* p = nullptr;
  if (cudaMalloc(&p, kIpcFlags + 2 * gb) != cudaSuccess) {
    cudaGetLastError();
    return set_err(TSLB_ENOMEM, "peer-memory transport block (%zu bytes)", kIpcFlags + 2 * gb);
  }
  CK(cudaMemset(p, 0, kIpcFlags + 2 * gb));
  h->ipc_blk = static_cast<char*>(p);
  h->ipc_gb = gb;
  h->bytes += kIpcFlags + 2 * gb;
  return 0;
}

int tslb_cuda_ipc_handle(tslb_cuda_handle h, void* handle64) {
  if (!handle64) return set_err(TSLB_EINVAL, "ipc_handle: null output");
  if (!h->decomposed || h->comps != 1) return set_err(TSLB_ESTATE, "ipc_handle needs a single-fluid slab solver");
  CK(cudaSetDevice(h->device));
  if (int rc = ipc_block(h)) return rc;
  cudaIpcMemHandle_t hd;
  CK(cudaIpcGetMemHandle(&hd, h->ipc_blk));
  static_assert(sizeof hd == TSLB_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  std::memcpy(handle64, &hd, sizeof hd);
  return 0;
}

// ... and map the neighbours' (a face whose neighbour is this rank itself --
// one rank, periodic -- uses the own block)
int tslb_cuda_attach_ipc(tslb_cuda_handle h, const void* below64, const void* above64) {
  if (!h->decomposed || h->comps != 1) return set_err(TSLB_ESTATE, "attach_ipc needs a single-fluid slab solver");
  if (h->xmode != 0) return set_err(TSLB_ESTATE, "attach_ipc: the slab already has a transport");
  const bool has_dn = h->d.mode[ZMin] == kGhost, has_up = h->d.mode[ZMax] == kGhost;
  if ((has_dn && !below64) || (has_up && !above64)) return set_err(TSLB_EINVAL, "attach_ipc: missing neighbour handle");
  CK(cudaSetDevice(h->device));
  if (int rc = ipc_block(h)) return rc;
  cudaIpcMemHandle_t own;
  CK(cudaIpcGetMemHandle(&own, h->ipc_blk));
  auto open = [&](const void* hb, char*& ptr, bool& mapped) -> int {
    if (std::memcmp(hb, &own, sizeof own) == 0) {
      ptr = h->ipc_blk;
      return 0;
    }
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, hb, sizeof hd);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return set_err(TSLB_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    }
    ptr = static_cast<char*>(p);
    mapped = true;
    return 0;
  };
  if (has_up)
    if (int rc = open(above64, h->ipc_up, h->ipc_up_mapped)) return rc;
  if (has_dn) {
    if (has_up && std::memcmp(below64, above64, sizeof own) == 0) {
      h->ipc_down = h->ipc_up;  // (two ranks: the same neighbour on both faces)
    } else if (int rc = open(below64, h->ipc_down, h->ipc_down_mapped)) {
      return rc;
    }
  }
  // the ghost planes now live in the exported block
  if (h->gm) {
    CK(cudaFree(h->gm));
    h->bytes -= h->ipc_gb;
  }
  h->gm = h->ipc_blk + kIpcFlags;
  h->xcount = 0;
  h->xmode = 3;
  return 0;
}

int tslb_cuda_link_local(tslb_cuda_handle* slabs, int count) {
  if (count < 2) return set_err(TSLB_EINVAL, "link_local needs at least two slabs");
  for (int r = 0; r < count; ++r) {
    tslb_cuda_sim* h = slabs[r];
    if (!h->decomposed) return set_err(TSLB_ESTATE, "link_local needs slab solvers");
    h->up_peer = h->d.mode[ZMax] == kGhost ? slabs[(r + 1) % count] : nullptr;
    h->down_peer = h->d.mode[ZMin] == kGhost ? slabs[(r - 1 + count) % count] : nullptr;
    h->xmode = 2;
  }
  return 0;
}

int tslb_cuda_group_step(tslb_cuda_handle* slabs, int count, long nsteps) {
  // Same schedule as the NCCL path, serialised on the first slab's stream
  // (single-device verification transport).
  cudaStream_t st = slabs[0]->s;
  CK(cudaSetDevice(slabs[0]->device));
  bool all_m = true, any_m = false;
  for (int r = 0; r < count; ++r) {
    all_m = all_m && slabs[r]->sched == TSLB_SCHED_M;
    any_m = any_m || slabs[r]->sched == TSLB_SCHED_M;
  }
  if (any_m && !all_m) return set_err(TSLB_ESTATE, "linked slabs must share one step schedule");
  if (slabs[0]->comps == 2 && nci_on(slabs[0])) {
    // the NCCL path's phases (NCI), serialised
    for (long s = 0; s < nsteps; ++s) {
      for (int r = 0; r < count; ++r)
        if (int rc = ph_cg_moments(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r)
        if (int rc = exchange_phi_local(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r)
        if (int rc = ph_cg_gradient_slab(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r)
        if (int rc = exchange_flags_local(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r)
        if (int rc = fold_flags(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r)
        if (int rc = ph_cg_streamcoll_range(slabs[r], 0, slabs[r]->nzl, st)) return rc;
      for (int r = 0; r < count; ++r)
        if (int rc = exchange_local(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r) {
        if (int rc = unpack(slabs[r], st)) return rc;
        slabs[r]->stress_pending = true;
        ++slabs[r]->steps;
      }
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return 0;
  }
  if (slabs[0]->comps == 2) {
    for (long s = 0; s < nsteps; ++s) {
      for (int r = 0; r < count; ++r)
        if (int rc = ph_cg_moments(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r)
        if (int rc = exchange_phi_local(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r) {
        tslb_cuda_sim* h = slabs[r];
        ++h->launches;
        const int rc = by_scalar(h, [&](auto z) {
          using T = decltype(z);
          return launch_cg_streamcoll_grad<T>(h->lat, h->range(0, h->nzl), static_cast<T*>(h->f[0]),
                                              static_cast<T*>(h->f[1]), h->tf(), h->omega, h->cp, st);
        });
        if (rc) return set_err(TSLB_ESTATE, "two-fluid slab step needs a box geometry without NCI");
      }
      for (int r = 0; r < count; ++r)
        if (int rc = exchange_local(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r) {
        if (int rc = unpack(slabs[r], st)) return rc;
        slabs[r]->grad_pending = true;
        slabs[r]->stress_pending = true;
        ++slabs[r]->steps;
      }
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return 0;
  }
  for (long s = 0; s < nsteps; ++s) {
    if (all_m) {
      // the NCCL path's order: boundary chunks (writing the send buffers),
      // exchange, interior chunks, swap (first step: moments, pack, exchange)
      const bool first = !slabs[0]->fimplicit;
      for (int r = 0; r < count; ++r) {
        tslb_cuda_sim* h = slabs[r];
        const int b = boundary_planes(h);
        int rc = 0;
        if (first) {
          if (!(rc = first_moments(h, st))) rc = pack_moments(h, h->mo, st);
        } else if (h->nzl <= 2 * b) {
          rc = ph_mstep(h, st);
        } else if (!(rc = ph_mstep(h, st, 0, b))) {
          rc = ph_mstep(h, st, h->nzl - b, h->nzl);
        }
        if (!rc && !first) rc = pack_moments(h, h->mo2, st);
        if (rc) return rc;
      }
      for (int r = 0; r < count; ++r)
        if (int rc = exchange_moments_local(slabs[r], st)) return rc;
      for (int r = 0; r < count; ++r) {
        tslb_cuda_sim* h = slabs[r];
        if (!first) {
          const int b = boundary_planes(h);
          if (h->nzl > 2 * b)
            if (int rc = ph_mstep(h, st, b, h->nzl - b)) return rc;
          std::swap(h->mo, h->mo2);
        }
        h->fimplicit = true;
        ++h->steps;
      }
      continue;
    }
    for (int r = 0; r < count; ++r)
      if (int rc = ph_moments(slabs[r], st)) return rc;
    for (int r = 0; r < count; ++r)
      if (int rc = ph_streamcoll(slabs[r], 0, slabs[r]->nzl, st)) return rc;
    for (int r = 0; r < count; ++r)
      if (int rc = exchange_local(slabs[r], st)) return rc;
    for (int r = 0; r < count; ++r) {
      if (int rc = unpack(slabs[r], st)) return rc;
      ++slabs[r]->steps;
    }
  }
  CK(cudaStreamSynchronize(st));
  CK(cudaGetLastError());
  return 0;
}

}  // extern "C"
