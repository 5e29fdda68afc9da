// tslb_b200/tslb.hpp -- C++ drop-in for the tslb solver interface, backed by
// the B200 kernels through the C-ABI (include/tslb_cuda.h,
// libtslb_cuda.so).
//
// A caller of the reference library (proj/include/tslb/*.hpp) switches by
// putting this repo's include/ first on the include path: include/tslb/*.hpp
// forward here. Names, template parameters, signatures, host-visible state
// and exception types follow the reference headers; the time stepping runs
// on the GPU. Cited reference lines are relative to proj/include/tslb/.
//
//   lattice.hpp      -> D2Q9, D3Q19 (+ new D3Q27), LatticeDescriptor, ...
//   fields.hpp       -> GridDims, FieldSet, TwoFluidFieldSet, allocate_*
//   boundary.hpp     -> FaceKind, BoundarySpec, NodeGeometry, classify_nodes
//   collision.hpp    -> CollisionParams, NodeMoments, per-direction algebra
//   parallel.hpp     -> WorkerPool (accepted for signature compatibility)
//   kernels.hpp      -> compute_moments, stream_collide_fused, fused_step, ...
//   multicomponent.hpp -> colour-gradient phases, two_fluid_step
//   solver.hpp       -> SingleFluidSim, TwoFluidSim, dispatch_lattice
//   bench.hpp        -> count_kernel_cost, fnv1a, state_digest, run_benchmark
//
// Device-state model: a Sim keeps its fields resident on the GPU and a host
// mirror (FieldSet with Eigen arrays). Non-const fields() synchronises the
// mirror and marks it dirty; the next device operation uploads it. const
// fields() only synchronises. Free functions on a caller-owned FieldSet
// upload, run one device phase and download (tests and drivers use them on
// small grids, as the reference tests do). There is no host fallback for
// any time-stepping phase: a missing device or library throws.
#pragma once

#include <Eigen/Core>

#include <array>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <istream>
#include <memory>
#include <numbers>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "../tslb_cuda.h"

namespace tslb {

// ===========================================================================
// lattices
// ===========================================================================
enum class LatticeKind { D2Q9 = TSLB_D2Q9, D3Q19 = TSLB_D3Q19, D3Q27 = TSLB_D3Q27 };

namespace tables {
using V = std::array<int, 3>;
using R = std::array<long, 2>;
}  // namespace tables

struct D2Q9 {
  static constexpr LatticeKind kind = LatticeKind::D2Q9;
  static constexpr int dim = 2, q = 9;
  static constexpr std::array<tables::V, q> c{{{0, 0, 0},
                                               {1, 0, 0},
                                               {-1, 0, 0},
                                               {0, 1, 0},
                                               {0, -1, 0},
                                               {1, 1, 0},
                                               {-1, -1, 0},
                                               {1, -1, 0},
                                               {-1, 1, 0}}};
  static constexpr std::array<tables::R, q> t_rat{
      {{4, 9}, {1, 9}, {1, 9}, {1, 9}, {1, 9}, {1, 36}, {1, 36}, {1, 36}, {1, 36}}};
  static constexpr std::array<tables::R, q> b_rat{
      {{-4, 27}, {2, 27}, {2, 27}, {2, 27}, {2, 27}, {5, 108}, {5, 108}, {5, 108}, {5, 108}}};
  static constexpr std::array<int, q> opp{0, 2, 1, 4, 3, 6, 5, 8, 7};
};

namespace detail {
template <std::size_t Q>
constexpr std::array<int, Q> pair_opposites() {
  std::array<int, Q> o{};
  for (std::size_t a = 1; a < Q; ++a) o[a] = int((a % 2) ? a + 1 : a - 1);
  return o;
}
constexpr tables::R kR18{1, 18}, kR36{1, 36}, kR3{1, 3}, kRm3{-1, 3};
}  // namespace detail

struct D3Q19 {
  static constexpr LatticeKind kind = LatticeKind::D3Q19;
  static constexpr int dim = 3, q = 19;
  static constexpr std::array<tables::V, q> c{
      {{0, 0, 0},  {1, 0, 0},   {-1, 0, 0}, {0, 1, 0},  {0, -1, 0},
       {0, 0, 1},  {0, 0, -1},  {1, 1, 0},  {-1, -1, 0}, {1, -1, 0},
       {-1, 1, 0}, {1, 0, 1},   {-1, 0, -1}, {1, 0, -1}, {-1, 0, 1},
       {0, 1, 1},  {0, -1, -1}, {0, 1, -1}, {0, -1, 1}}};
  static constexpr std::array<tables::R, q> t_rat = [] {
    std::array<tables::R, q> t{};
    t[0] = detail::kR3;
    for (int a = 1; a < q; ++a) t[a] = a <= 6 ? detail::kR18 : detail::kR36;
    return t;
  }();
  static constexpr std::array<tables::R, q> b_rat = [] {
    std::array<tables::R, q> b{};
    b[0] = detail::kRm3;
    for (int a = 1; a < q; ++a) b[a] = a <= 6 ? detail::kR18 : detail::kR36;
    return b;
  }();
  static constexpr std::array<int, q> opp = detail::pair_opposites<q>();
};

/// New: D3Q27 (no reference code). D3Q19 order for the first 19 vectors,
/// corners appended in opposite pairs; t = 8/27, 2/27, 1/54, 1/216.
struct D3Q27 {
  static constexpr LatticeKind kind = LatticeKind::D3Q27;
  static constexpr int dim = 3, q = 27;
  static constexpr std::array<tables::V, q> c = [] {
    std::array<tables::V, q> v{};
    for (int a = 0; a < 19; ++a) v[a] = D3Q19::c[a];
    const tables::V corners[8] = {{1, 1, 1},  {-1, -1, -1}, {1, 1, -1},  {-1, -1, 1},
                                  {1, -1, 1}, {-1, 1, -1},  {-1, 1, 1}, {1, -1, -1}};
    for (int e = 0; e < 8; ++e) v[19 + e] = corners[e];
    return v;
  }();
  static constexpr std::array<tables::R, q> t_rat = [] {
    std::array<tables::R, q> t{};
    t[0] = {8, 27};
    for (int a = 1; a < q; ++a) t[a] = a <= 6 ? tables::R{2, 27} : a <= 18 ? tables::R{1, 54} : tables::R{1, 216};
    return t;
  }();
  static constexpr std::array<tables::R, q> b_rat = [] {
    std::array<tables::R, q> b{};
    for (int a = 0; a < 19; ++a) b[a] = D3Q19::b_rat[a];
    for (int a = 19; a < q; ++a) b[a] = {0, 1};
    return b;
  }();
  static constexpr std::array<int, q> opp = detail::pair_opposites<q>();
};

template <typename T>
constexpr T cs2_v = T(1) / T(3);

template <typename T>
struct LatticeDescriptor {
  LatticeKind kind{};
  int dim = 0;
  int q = 0;
  T cs2 = cs2_v<T>;
  Eigen::Matrix<int, 3, Eigen::Dynamic> c;
  Eigen::VectorX<T> t;
  Eigen::VectorX<T> b;
  Eigen::VectorXi opp;
  Eigen::Matrix<T, 6, Eigen::Dynamic> q2;
};

template <class Lat, typename T>
LatticeDescriptor<T> descriptor_of() {
  LatticeDescriptor<T> d;
  d.kind = Lat::kind;
  d.dim = Lat::dim;
  d.q = Lat::q;
  d.c.resize(3, Lat::q);
  d.t.resize(Lat::q);
  d.b.resize(Lat::q);
  d.opp.resize(Lat::q);
  d.q2.resize(6, Lat::q);
  for (int a = 0; a < Lat::q; ++a) {
    const auto& v = Lat::c[std::size_t(a)];
    for (int k = 0; k < 3; ++k) d.c(k, a) = v[std::size_t(k)];
    d.t(a) = T(Lat::t_rat[std::size_t(a)][0]) / T(Lat::t_rat[std::size_t(a)][1]);
    d.b(a) = T(Lat::b_rat[std::size_t(a)][0]) / T(Lat::b_rat[std::size_t(a)][1]);
    d.opp(a) = Lat::opp[std::size_t(a)];
    const T x = T(v[0]), y = T(v[1]), z = T(v[2]);
    d.q2(0, a) = x * x - d.cs2;
    d.q2(1, a) = y * y - d.cs2;
    d.q2(2, a) = z * z - (Lat::dim == 3 ? d.cs2 : T(0));
    d.q2(3, a) = x * y;
    d.q2(4, a) = x * z;
    d.q2(5, a) = y * z;
  }
  return d;
}

template <typename T = double>
LatticeDescriptor<T> make_descriptor(LatticeKind kind) {
  if (kind == LatticeKind::D2Q9) return descriptor_of<D2Q9, T>();
  if (kind == LatticeKind::D3Q27) return descriptor_of<D3Q27, T>();
  return descriptor_of<D3Q19, T>();
}

struct ValidationReport {
  struct Check {
    std::string name;
    double violation = 0.0;
    bool pass = false;
  };
  std::vector<Check> checks;
  double tolerance = 1e-14;
  bool all_pass() const {
    for (const auto& c : checks)
      if (!c.pass) return false;
    return true;
  }
};

/// validate_moments (lattice.hpp:155-244): discrete moment and isotropy
/// conditions of t and B, opposite map, trace of Q; failures reported.
template <typename T>
ValidationReport validate_moments(const LatticeDescriptor<T>& d, double tol = 1e-14) {
  ValidationReport rep;
  rep.tolerance = tol;
  const int D = d.dim;
  const double cs2 = double(d.cs2), cs4 = cs2 * cs2;
  auto cc = [&](int a, int al) { return double(d.c(al, a)); };
  // weighted moment of weights w over the product of the listed axes
  auto moment = [&](const auto& w, std::initializer_list<int> axes) {
    double s = 0.0;
    for (int a = 0; a < d.q; ++a) {
      double term = double(w(a));
      for (int ax : axes) term *= cc(a, ax);
      s += term;
    }
    return s;
  };
  auto add = [&](const char* name, double v) { rep.checks.push_back({name, v, v <= tol}); };
  auto delta = [](int x, int y) { return x == y ? 1.0 : 0.0; };

  add("sum t = 1", std::abs(moment(d.t, {}) - 1.0));
  double v1 = 0, v2 = 0, v4 = 0, b1 = 0;
  for (int al = 0; al < D; ++al) {
    v1 = std::max(v1, std::abs(moment(d.t, {al})));
    b1 = std::max(b1, std::abs(moment(d.b, {al})));
    for (int be = 0; be < D; ++be) {
      v2 = std::max(v2, std::abs(moment(d.t, {al, be}) - cs2 * delta(al, be)));
      for (int ga = 0; ga < D; ++ga)
        for (int de = 0; de < D; ++de) {
          const double want = cs4 * (delta(al, be) * delta(ga, de) + delta(al, ga) * delta(be, de) +
                                     delta(al, de) * delta(be, ga));
          v4 = std::max(v4, std::abs(moment(d.t, {al, be, ga, de}) - want));
        }
    }
  }
  add("sum t c = 0", v1);
  add("sum t cc = cs2 I", v2);
  add("4th-order isotropy", v4);
  double vo = 0;
  for (int a = 0; a < d.q; ++a) {
    const int o = d.opp(a);
    if (o < 0 || o >= d.q || d.opp(o) != a) vo = 1.0;
    else
      for (int al = 0; al < 3; ++al) vo = std::max(vo, std::abs(cc(o, al) + cc(a, al)));
  }
  add("opp involution, c[opp] = -c", vo);
  add("sum B = cs2", std::abs(moment(d.b, {}) - cs2));
  add("sum B c = 0", b1);
  double vq = 0;
  for (int a = 0; a < d.q; ++a) {
    const double tr = double(d.q2(0, a)) + double(d.q2(1, a)) + double(d.q2(2, a));
    vq = std::max(vq, std::abs(tr - (cc(a, 0) * cc(a, 0) + cc(a, 1) * cc(a, 1) + cc(a, 2) * cc(a, 2) - D * cs2)));
  }
  add("trace Q = |c|^2 - D cs2", vq);
  return rep;
}

inline const char* lattice_name(LatticeKind k) {
  return k == LatticeKind::D2Q9 ? "d2q9" : k == LatticeKind::D3Q19 ? "d3q19" : "d3q27";
}

/// Compile-time direction loop: f(std::integral_constant<int, a>) for each a.
template <class Lat, class F>
inline void for_each_dir(F&& f) {
  [&]<int... A>(std::integer_sequence<int, A...>) {
    (f(std::integral_constant<int, A>{}), ...);
  }(std::make_integer_sequence<int, Lat::q>{});
}

// ===========================================================================
// grid and fields (host mirror types)
// ===========================================================================
struct GridDims {
  int nx = 0, ny = 0, nz = 1;
  std::size_t n() const { return std::size_t(nx) * std::size_t(ny) * std::size_t(nz); }
  bool valid() const { return nx > 0 && ny > 0 && nz > 0; }
};

inline std::size_t linear_index(const GridDims& g, int i, int j, int k) {
  return std::size_t(i) + std::size_t(g.nx) * (std::size_t(j) + std::size_t(g.ny) * std::size_t(k));
}

inline int wrap(int i, int n) {
  const int r = i % n;
  return r < 0 ? r + n : r;
}

template <typename T>
using FieldArray = Eigen::ArrayX<T>;

template <typename T>
struct FieldSet {
  GridDims dims;
  int q = 0;
  int dim = 0;
  std::vector<FieldArray<T>> f;
  FieldArray<T> rho;
  std::vector<FieldArray<T>> mom;
  std::vector<FieldArray<T>> pineq;
  std::size_t n() const { return dims.n(); }
  int npineq() const { return dim * (dim + 1) / 2; }
};

template <typename T>
struct TwoFluidFieldSet {
  GridDims dims;
  int q = 0;
  int dim = 0;
  std::vector<FieldArray<T>> fr, fb;
  FieldArray<T> rho_r, rho_b, rho;
  std::vector<FieldArray<T>> mom, pineq;
  FieldArray<T> phi;
  std::vector<FieldArray<T>> gradphi;
  std::vector<std::uint8_t> nci_flag;
  std::size_t n() const { return dims.n(); }
  int npineq() const { return dim * (dim + 1) / 2; }
};

namespace detail {
template <typename T>
std::vector<FieldArray<T>> zero_arrays(int count, Eigen::Index n) {
  std::vector<FieldArray<T>> v(static_cast<std::size_t>(count));
  for (auto& a : v) a = FieldArray<T>::Zero(n);
  return v;
}
}  // namespace detail

template <typename T>
FieldSet<T> allocate_fields(const GridDims& g, const LatticeDescriptor<T>& d) {
  if (!g.valid()) throw std::invalid_argument("allocate_fields: bad dims");
  FieldSet<T> s;
  s.dims = g;
  s.q = d.q;
  s.dim = d.dim;
  const auto n = Eigen::Index(g.n());
  s.f = detail::zero_arrays<T>(d.q, n);
  s.rho = FieldArray<T>::Zero(n);
  s.mom = detail::zero_arrays<T>(d.dim, n);
  s.pineq = detail::zero_arrays<T>(s.npineq(), n);
  return s;
}

template <typename T>
TwoFluidFieldSet<T> allocate_two_fluid(const GridDims& g, const LatticeDescriptor<T>& d) {
  if (!g.valid()) throw std::invalid_argument("allocate_two_fluid: bad dims");
  TwoFluidFieldSet<T> s;
  s.dims = g;
  s.q = d.q;
  s.dim = d.dim;
  const auto n = Eigen::Index(g.n());
  s.fr = detail::zero_arrays<T>(d.q, n);
  s.fb = detail::zero_arrays<T>(d.q, n);
  s.rho_r = FieldArray<T>::Zero(n);
  s.rho_b = FieldArray<T>::Zero(n);
  s.rho = FieldArray<T>::Zero(n);
  s.mom = detail::zero_arrays<T>(d.dim, n);
  s.pineq = detail::zero_arrays<T>(s.npineq(), n);
  s.phi = FieldArray<T>::Zero(n);
  s.gradphi = detail::zero_arrays<T>(d.dim, n);
  s.nci_flag.assign(g.n(), 0);
  return s;
}

struct ArrayLedger {
  LatticeKind kind{};
  int q = 0, dim = 0, fused_arrays = 0, flipflop_arrays = 0;
  std::size_t elem_bytes = 0, fused_bytes_per_node = 0, flipflop_bytes_per_node = 0,
              saved_bytes_per_node = 0;
};

inline ArrayLedger memory_report(LatticeKind kind, std::size_t elem_bytes) {
  const auto d = make_descriptor<double>(kind);
  ArrayLedger l;
  l.kind = kind;
  l.q = d.q;
  l.dim = d.dim;
  l.fused_arrays = d.q + 1 + d.dim + d.dim * (d.dim + 1) / 2;
  l.flipflop_arrays = 2 * d.q + 1 + d.dim;
  l.elem_bytes = elem_bytes;
  l.fused_bytes_per_node = std::size_t(l.fused_arrays) * elem_bytes;
  l.flipflop_bytes_per_node = std::size_t(l.flipflop_arrays) * elem_bytes;
  l.saved_bytes_per_node = l.flipflop_bytes_per_node - l.fused_bytes_per_node;
  return l;
}

// ===========================================================================
// boundaries and geometry
// ===========================================================================
enum class FaceKind { Periodic = TSLB_FACE_PERIODIC, NoSlipWall = TSLB_FACE_WALL, MovingWall = TSLB_FACE_MOVING };
enum FaceId { XMin = 0, XMax = 1, YMin = 2, YMax = 3, ZMin = 4, ZMax = 5 };

template <typename T>
struct Face {
  FaceKind kind = FaceKind::Periodic;
  std::array<T, 3> u_wall = {T(0), T(0), T(0)};
};

template <typename T>
struct BoundarySpec {
  std::array<Face<T>, 6> faces;
  static BoundarySpec all_periodic() { return BoundarySpec{}; }
  static BoundarySpec closed_box() {
    BoundarySpec s;
    for (auto& f : s.faces) f.kind = FaceKind::NoSlipWall;
    return s;
  }
  static BoundarySpec lid_cavity(T u_lid) {
    BoundarySpec s = closed_box();
    s.faces[YMax].kind = FaceKind::MovingWall;
    s.faces[YMax].u_wall = {u_lid, T(0), T(0)};
    return s;
  }
};

struct NodeGeometry {
  GridDims dims;
  std::vector<std::uint8_t> solid;
  std::vector<std::uint32_t> slow_mask;
  std::size_t n_fluid = 0;
};

// ---- C-ABI plumbing --------------------------------------------------------
namespace detail {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int rc) {
  if (rc == TSLB_OK) return;
  const std::string msg = tslb_cuda_last_error();
  if (rc == TSLB_EINVAL) throw std::invalid_argument(msg);
  throw CudaError(msg);
}

template <typename T>
constexpr int scalar_id() {
  static_assert(std::is_same_v<T, double> || std::is_same_v<T, float>, "double or float storage");
  return std::is_same_v<T, double> ? TSLB_F64 : TSLB_F32;
}

inline int device_id() {
  if (const char* e = std::getenv("TSLB_DEVICE")) return std::atoi(e);
  return 0;
}

template <typename T>
void face_arrays(const BoundarySpec<T>& spec, int kinds[6], double uw[18]) {
  for (int f = 0; f < 6; ++f) {
    kinds[f] = int(spec.faces[std::size_t(f)].kind);
    for (int c = 0; c < 3; ++c) uw[3 * f + c] = double(spec.faces[std::size_t(f)].u_wall[std::size_t(c)]);
  }
}

/// RAII owner of one C-ABI solver handle.
class Device {
 public:
  Device() = default;
  template <class Lat, typename T>
  static Device make(const GridDims& g, double omega, const BoundarySpec<T>& spec,
                     const std::vector<std::uint8_t>& solid, int components,
                     const double* color = nullptr, const int* color_i = nullptr) {
    if (!solid.empty() && solid.size() != g.n())
      throw std::invalid_argument("classify_nodes: mask size mismatch");
    int kinds[6];
    double uw[18];
    face_arrays(spec, kinds, uw);
    Device d;
    tslb_cuda_handle h = nullptr;
    check(tslb_cuda_create(int(Lat::kind), scalar_id<T>(), components, g.nx, g.ny, g.nz, omega, kinds, uw,
                           solid.empty() ? nullptr : solid.data(), color, color_i, device_id(), &h));
    d.h_.reset(h);
    return d;
  }
  tslb_cuda_handle get() const { return h_.get(); }
  explicit operator bool() const { return bool(h_); }

 private:
  struct Del {
    void operator()(tslb_cuda_sim* h) const { tslb_cuda_destroy(h); }
  };
  std::unique_ptr<tslb_cuda_sim, Del> h_;
};

template <typename T>
void upload_arrays(tslb_cuda_handle h, int species, const std::vector<FieldArray<T>>& a, std::size_t n) {
  std::vector<T> buf(a.size() * n);
  for (std::size_t k = 0; k < a.size(); ++k) std::memcpy(buf.data() + k * n, a[k].data(), n * sizeof(T));
  check(tslb_cuda_upload_f(h, species, buf.data()));
}

template <typename T>
void download_arrays(tslb_cuda_handle h, int species, std::vector<FieldArray<T>>& a, std::size_t n) {
  std::vector<T> buf(a.size() * n);
  check(tslb_cuda_download_f(h, species, buf.data()));
  for (std::size_t k = 0; k < a.size(); ++k) std::memcpy(a[k].data(), buf.data() + k * n, n * sizeof(T));
}

template <typename T>
void upload_field(tslb_cuda_handle h, int field, const std::vector<FieldArray<T>>& a, std::size_t n) {
  std::vector<T> buf(a.size() * n);
  for (std::size_t k = 0; k < a.size(); ++k) std::memcpy(buf.data() + k * n, a[k].data(), n * sizeof(T));
  check(tslb_cuda_upload_field(h, field, buf.data()));
}

template <typename T>
void download_field(tslb_cuda_handle h, int field, std::vector<FieldArray<T>>& a, std::size_t n) {
  std::vector<T> buf(a.size() * n);
  check(tslb_cuda_download_field(h, field, buf.data()));
  for (std::size_t k = 0; k < a.size(); ++k) std::memcpy(a[k].data(), buf.data() + k * n, n * sizeof(T));
}

template <typename T>
void upload_one(tslb_cuda_handle h, int field, const FieldArray<T>& a) {
  check(tslb_cuda_upload_field(h, field, a.data()));
}
template <typename T>
void download_one(tslb_cuda_handle h, int field, FieldArray<T>& a) {
  check(tslb_cuda_download_field(h, field, a.data()));
}

template <typename T>
void upload_single(tslb_cuda_handle h, const FieldSet<T>& s) {
  upload_arrays(h, 0, s.f, s.n());
  upload_one(h, TSLB_FIELD_RHO, s.rho);
  upload_field(h, TSLB_FIELD_MOM, s.mom, s.n());
  upload_field(h, TSLB_FIELD_PINEQ, s.pineq, s.n());
}

template <typename T>
void download_single(tslb_cuda_handle h, FieldSet<T>& s) {
  download_arrays(h, 0, s.f, s.n());
  download_one(h, TSLB_FIELD_RHO, s.rho);
  download_field(h, TSLB_FIELD_MOM, s.mom, s.n());
  download_field(h, TSLB_FIELD_PINEQ, s.pineq, s.n());
}

template <typename T>
void upload_two(tslb_cuda_handle h, const TwoFluidFieldSet<T>& s) {
  const std::size_t n = s.n();
  upload_arrays(h, 0, s.fr, n);
  upload_arrays(h, 1, s.fb, n);
  upload_one(h, TSLB_FIELD_RHO_R, s.rho_r);
  upload_one(h, TSLB_FIELD_RHO_B, s.rho_b);
  upload_one(h, TSLB_FIELD_RHO, s.rho);
  upload_field(h, TSLB_FIELD_MOM, s.mom, n);
  upload_field(h, TSLB_FIELD_PINEQ, s.pineq, n);
  upload_one(h, TSLB_FIELD_PHI, s.phi);
  upload_field(h, TSLB_FIELD_GRADPHI, s.gradphi, n);
  check(tslb_cuda_upload_field(h, TSLB_FIELD_NCI_FLAG, s.nci_flag.data()));
}

template <typename T>
void download_two(tslb_cuda_handle h, TwoFluidFieldSet<T>& s) {
  const std::size_t n = s.n();
  download_arrays(h, 0, s.fr, n);
  download_arrays(h, 1, s.fb, n);
  download_one(h, TSLB_FIELD_RHO_R, s.rho_r);
  download_one(h, TSLB_FIELD_RHO_B, s.rho_b);
  download_one(h, TSLB_FIELD_RHO, s.rho);
  download_field(h, TSLB_FIELD_MOM, s.mom, n);
  download_field(h, TSLB_FIELD_PINEQ, s.pineq, n);
  download_one(h, TSLB_FIELD_PHI, s.phi);
  download_field(h, TSLB_FIELD_GRADPHI, s.gradphi, n);
  check(tslb_cuda_download_field(h, TSLB_FIELD_NCI_FLAG, s.nci_flag.data()));
}

inline NodeGeometry geometry_of(tslb_cuda_handle h, const GridDims& g) {
  NodeGeometry geo;
  geo.dims = g;
  geo.solid.resize(g.n());
  geo.slow_mask.resize(g.n());
  std::uint64_t nf = 0;
  check(tslb_cuda_download_geometry(h, geo.solid.data(), geo.slow_mask.data(), &nf));
  geo.n_fluid = std::size_t(nf);
  return geo;
}

inline bool any_solid(const NodeGeometry& geo) {
  for (auto v : geo.solid)
    if (v) return true;
  return false;
}

}  // namespace detail

/// classify_nodes (boundary.hpp:61-111) on the device; bit-identical masks.
template <typename T, class Lat>
NodeGeometry classify_nodes(const GridDims& g, const BoundarySpec<T>& spec,
                            const std::vector<std::uint8_t>& solid = {}) {
  static_assert(Lat::q <= 32, "slow_mask holds one bit per direction");
  auto dev = detail::Device::make<Lat, T>(g, 1.0, spec, solid, 1);
  return detail::geometry_of(dev.get(), g);
}

/// resolve_push (boundary.hpp:118-144): index logic of one slow-path push,
/// used by drivers and tests to reason about targets (no field arithmetic).
template <typename T, class Lat>
inline bool resolve_push(const GridDims& g, const BoundarySpec<T>& spec, const std::vector<std::uint8_t>& solid,
                         int i, int j, int k, int a, std::size_t& target_idx, std::array<T, 3>& u_wall) {
  const auto& cv = Lat::c[std::size_t(a)];
  const int ext[3] = {g.nx, g.ny, g.nz};
  int p[3] = {i + cv[0], j + cv[1], k + cv[2]};
  u_wall = {T(0), T(0), T(0)};
  bool hits_wall = false;
  for (int ax = 0; ax < 3; ++ax) {
    if (p[ax] >= 0 && p[ax] < ext[ax]) continue;
    const Face<T>& face = spec.faces[std::size_t(2 * ax + (p[ax] < 0 ? 0 : 1))];
    if (face.kind == FaceKind::Periodic) {
      p[ax] = wrap(p[ax], ext[ax]);
      continue;
    }
    hits_wall = true;
    for (int c = 0; c < 3; ++c) u_wall[std::size_t(c)] += face.u_wall[std::size_t(c)];
  }
  if (hits_wall) return true;
  const std::size_t t = linear_index(g, p[0], p[1], p[2]);
  if (solid[t]) return true;
  target_idx = t;
  return false;
}

/// load_mask (boundary.hpp:149-189): '.' fluid, '#' solid, top row = y max,
/// z slabs separated by blank lines.
inline std::vector<std::uint8_t> load_mask(std::istream& in, const GridDims& g) {
  std::vector<std::uint8_t> solid(g.n(), 0);
  std::vector<std::string> slab;
  int k = 0;
  auto flush = [&] {
    if (slab.empty()) return;
    if (int(slab.size()) != g.ny)
      throw std::runtime_error("mask: slab has " + std::to_string(slab.size()) + " rows, expected " +
                               std::to_string(g.ny));
    if (k >= g.nz) throw std::runtime_error("mask: too many rows");
    for (int r = 0; r < g.ny; ++r)
      for (int i = 0; i < g.nx; ++i)
        solid[linear_index(g, i, g.ny - 1 - r, k)] = slab[std::size_t(r)][std::size_t(i)] == '#';
    ++k;
    slab.clear();
  };
  std::string line;
  while (std::getline(in, line)) {
    while (!line.empty() && (line.back() == '\r' || line.back() == ' ')) line.pop_back();
    if (line.empty()) {
      flush();
      continue;
    }
    if (int(line.size()) != g.nx)
      throw std::runtime_error("mask: row width " + std::to_string(line.size()) + ", expected " +
                               std::to_string(g.nx));
    for (char ch : line)
      if (ch != '.' && ch != '#') throw std::runtime_error(std::string("mask: bad character '") + ch + "'");
    if (int(slab.size()) >= g.ny || k >= g.nz) throw std::runtime_error("mask: too many rows");
    slab.push_back(line);
  }
  if (!slab.empty() && int(slab.size()) != g.ny) throw std::runtime_error("mask: final slab incomplete");
  flush();
  if (k != g.nz)
    throw std::runtime_error("mask: " + std::to_string(k) + " slabs, expected " + std::to_string(g.nz));
  return solid;
}

// ===========================================================================
// node algebra (host forms for initialisers, tests and analysis; the device
// kernels carry their own bit-identical copies)
// ===========================================================================
template <typename T>
struct CollisionParams {
  T omega = T(1);
  T rho0 = T(1);
  // EXTENSION (not in the reference): single-fluid body force, applied as the
  // velocity shift u_eq = j + tau F of the moments pass (tslb_cuda.h,
  // tslb_cuda_set_body_force). Zero leaves every result unchanged.
  std::array<T, 3> force{};
  T tau() const { return T(1) / omega; }
  T nu() const { return cs2_v<T> * (tau() - T(0.5)); }
};

template <typename T>
T omega_from_nu(T nu) {
  return T(1) / (nu / cs2_v<T> + T(0.5));
}
template <typename T>
T omega_from_tau(T tau) {
  return T(1) / tau;
}
template <typename T>
T nu_from_omega(T omega) {
  return cs2_v<T> * (T(1) / omega - T(0.5));
}

template <class Lat, int A, typename T>
constexpr T weight() {
  return T(Lat::t_rat[A][0]) / T(Lat::t_rat[A][1]);
}
template <class Lat, int A, typename T>
constexpr T bweight() {
  return T(Lat::b_rat[A][0]) / T(Lat::b_rat[A][1]);
}

template <int CX, int CY, int CZ, typename T>
inline T dot_c(T x, T y, T z) {
  T s = T(0);
  if constexpr (CX != 0) s = CX > 0 ? s + x : s - x;
  if constexpr (CY != 0) s = CY > 0 ? s + y : s - y;
  if constexpr (CZ != 0) s = CZ > 0 ? s + z : s - z;
  return s;
}

template <typename T>
struct NodeMoments {
  T rho{}, ux{}, uy{}, uz{};
  T usq15{};
  T pxx{}, pyy{}, pzz{};
  T pxy2{}, pxz2{}, pyz2{};
  T trcs2{};
};

template <typename T>
inline NodeMoments<T> prepare_node(T rho, T ux, T uy, T uz, T pxx, T pyy, T pzz, T pxy, T pxz, T pyz) {
  NodeMoments<T> m;
  m.rho = rho;
  m.ux = ux;
  m.uy = uy;
  m.uz = uz;
  m.usq15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
  m.pxx = pxx;
  m.pyy = pyy;
  m.pzz = pzz;
  m.pxy2 = pxy + pxy;
  m.pxz2 = pxz + pxz;
  m.pyz2 = pyz + pyz;
  m.trcs2 = cs2_v<T> * (pxx + pyy + pzz);
  return m;
}

template <class Lat, int A, typename T>
inline T equilibrium_dir(const NodeMoments<T>& m) {
  constexpr auto v = Lat::c[A];
  const T cu = dot_c<v[0], v[1], v[2]>(m.ux, m.uy, m.uz);
  return weight<Lat, A, T>() * (m.rho + T(3) * cu + T(4.5) * cu * cu - m.usq15);
}

template <class Lat, int A, typename T>
inline T regularized_dir(const NodeMoments<T>& m) {
  constexpr auto v = Lat::c[A];
  T s = T(0);
  if constexpr (v[0] != 0) s += m.pxx;
  if constexpr (v[1] != 0) s += m.pyy;
  if constexpr (v[2] != 0) s += m.pzz;
  if constexpr (v[0] * v[1] != 0) s = v[0] * v[1] > 0 ? s + m.pxy2 : s - m.pxy2;
  if constexpr (v[0] * v[2] != 0) s = v[0] * v[2] > 0 ? s + m.pxz2 : s - m.pxz2;
  if constexpr (v[1] * v[2] != 0) s = v[1] * v[2] > 0 ? s + m.pyz2 : s - m.pyz2;
  return weight<Lat, A, T>() * T(4.5) * (s - m.trcs2);
}

template <class Lat, int A, typename T>
inline T post_collision_dir(const NodeMoments<T>& m, T one_minus_omega) {
  return equilibrium_dir<Lat, A, T>(m) + one_minus_omega * regularized_dir<Lat, A, T>(m);
}

template <typename T>
Eigen::VectorX<T> equilibrium_all(const LatticeDescriptor<T>& d, T rho, T ux, T uy, T uz) {
  Eigen::VectorX<T> fe(d.q);
  const T usq15 = T(1.5) * (ux * ux + uy * uy + uz * uz);
  for (int a = 0; a < d.q; ++a) {
    const T cu = T(d.c(0, a)) * ux + T(d.c(1, a)) * uy + T(d.c(2, a)) * uz;
    fe(a) = d.t(a) * (rho + T(3) * cu + T(4.5) * cu * cu - usq15);
  }
  return fe;
}

template <typename T>
Eigen::Matrix<T, 3, 3> pineq_from_f(const LatticeDescriptor<T>& d, const Eigen::VectorX<T>& f, T rho, T ux, T uy,
                                    T uz) {
  const auto fe = equilibrium_all(d, rho, ux, uy, uz);
  Eigen::Matrix<T, 3, 3> p = Eigen::Matrix<T, 3, 3>::Zero();
  for (int a = 0; a < d.q; ++a)
    for (int al = 0; al < 3; ++al)
      for (int be = 0; be < 3; ++be) p(al, be) += (f(a) - fe(a)) * T(d.c(al, a)) * T(d.c(be, a));
  return p;
}

// ===========================================================================
// parallel substrate: the GPU grid replaces the thread team. WorkerPool keeps
// the reference API (parallel.hpp:38-92) so drivers compile unchanged; work
// submitted through run() executes on the calling thread per worker id.
// ===========================================================================
struct Range {
  std::size_t begin = 0, end = 0;
  std::size_t size() const { return end - begin; }
};

inline Range partition_range(std::size_t total, int parts, int part) {
  const std::size_t p = std::size_t(parts);
  return {total * std::size_t(part) / p, total * (std::size_t(part) + 1) / p};
}

inline int default_worker_count() {
  if (const char* env = std::getenv("TSLB_WORKERS")) {
    const int w = std::atoi(env);
    if (w > 0) return w;
  }
  const unsigned hw = std::thread::hardware_concurrency();
  return hw > 0 ? int(hw) : 1;
}

class WorkerPool {
 public:
  explicit WorkerPool(int workers = default_worker_count()) : nw_(workers < 1 ? 1 : workers) {}
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;
  int size() const { return nw_; }
  void run(const std::function<void(int)>& fn) {
    for (int w = 0; w < nw_; ++w) fn(w);
  }

 private:
  int nw_;
};

// ===========================================================================
// single-fluid phases on a caller-owned FieldSet (kernels.hpp)
// ===========================================================================
namespace detail {
template <class Lat, typename T, class Op>
void single_phase(FieldSet<T>& s, const NodeGeometry& geo, const BoundarySpec<T>& spec, T omega, Op&& op) {
  auto dev = Device::make<Lat, T>(s.dims, double(omega), spec, any_solid(geo) ? geo.solid : std::vector<std::uint8_t>{},
                                  1);
  upload_single(dev.get(), s);
  op(dev.get());
  download_single(dev.get(), s);
}
}  // namespace detail

template <class Lat, typename T>
void compute_moments(FieldSet<T>& s, const NodeGeometry& geo, WorkerPool* = nullptr) {
  detail::single_phase<Lat, T>(s, geo, BoundarySpec<T>::all_periodic(), T(1),
                               [](tslb_cuda_handle h) { detail::check(tslb_cuda_compute_moments(h)); });
}

template <class Lat, typename T>
void stream_collide_fused(FieldSet<T>& s, const NodeGeometry& geo, const BoundarySpec<T>& spec,
                          const CollisionParams<T>& prm, WorkerPool* = nullptr) {
  detail::single_phase<Lat, T>(s, geo, spec, prm.omega,
                               [](tslb_cuda_handle h) { detail::check(tslb_cuda_stream_collide(h)); });
}

template <class Lat, typename T>
void fused_step(FieldSet<T>& s, const NodeGeometry& geo, const BoundarySpec<T>& spec, const CollisionParams<T>& prm,
                WorkerPool* = nullptr) {
  detail::single_phase<Lat, T>(s, geo, spec, prm.omega,
                               [](tslb_cuda_handle h) { detail::check(tslb_cuda_step(h, 1)); });
}

/// stream_only (kernels.hpp:219-256): push the current f into dst.
template <class Lat, typename T>
void stream_only(FieldSet<T>& s, std::vector<FieldArray<T>>& dst, const NodeGeometry& geo,
                 const BoundarySpec<T>& spec, WorkerPool* = nullptr) {
  auto dev = detail::Device::make<Lat, T>(s.dims, 1.0, spec,
                                          detail::any_solid(geo) ? geo.solid : std::vector<std::uint8_t>{}, 1);
  detail::upload_arrays(dev.get(), 0, s.f, s.n());
  detail::upload_arrays(dev.get(), 2, dst, s.n());  // species 2 = second buffer
  detail::check(tslb_cuda_stream_only(dev.get()));
  detail::download_arrays(dev.get(), 0, dst, s.n());
}

/// reference_step (kernels.hpp:262-291): moments, collide in place, stream
/// into `scratch`, swap.
template <class Lat, typename T>
void reference_step(FieldSet<T>& s, std::vector<FieldArray<T>>& scratch, const NodeGeometry& geo,
                    const BoundarySpec<T>& spec, const CollisionParams<T>& prm, WorkerPool* = nullptr) {
  auto dev = detail::Device::make<Lat, T>(s.dims, double(prm.omega), spec,
                                          detail::any_solid(geo) ? geo.solid : std::vector<std::uint8_t>{}, 1);
  detail::upload_single(dev.get(), s);
  detail::upload_arrays(dev.get(), 2, scratch, s.n());
  detail::check(tslb_cuda_reference_step(dev.get(), 1));
  detail::download_single(dev.get(), s);
  detail::download_arrays(dev.get(), 2, scratch, s.n());
}

template <class Lat, int A, typename T>
inline T bounce_correction(const std::array<T, 3>& u_wall) {
  constexpr auto v = Lat::c[A];
  return T(6) * weight<Lat, A, T>() * dot_c<v[0], v[1], v[2]>(u_wall[0], u_wall[1], u_wall[2]);
}

template <class Lat>
inline std::array<std::ptrdiff_t, Lat::q> push_offsets(const GridDims& g) {
  std::array<std::ptrdiff_t, Lat::q> off{};
  for (int a = 0; a < Lat::q; ++a) {
    const auto& v = Lat::c[std::size_t(a)];
    off[std::size_t(a)] = std::ptrdiff_t(v[0]) + std::ptrdiff_t(g.nx) * (std::ptrdiff_t(v[1]) +
                                                                          std::ptrdiff_t(g.ny) * std::ptrdiff_t(v[2]));
  }
  return off;
}

/// initialize_regularized (kernels.hpp:295-311): host initialiser.
template <class Lat, typename T, class F>
void initialize_regularized(FieldSet<T>& s, const NodeGeometry& geo, F&& node_state) {
  const GridDims g = s.dims;
  for (int k = 0; k < g.nz; ++k)
    for (int j = 0; j < g.ny; ++j)
      for (int i = 0; i < g.nx; ++i) {
        const std::size_t idx = linear_index(g, i, j, k);
        if (geo.solid[idx]) continue;
        const NodeMoments<T> m = node_state(i, j, k);
        for_each_dir<Lat>([&](auto A) {
          constexpr int a = decltype(A)::value;
          s.f[std::size_t(a)][Eigen::Index(idx)] = equilibrium_dir<Lat, a, T>(m) + regularized_dir<Lat, a, T>(m);
        });
      }
}

// ===========================================================================
// two-fluid (multicomponent.hpp)
// ===========================================================================
enum class PerturbationForm { Squared, Linear };

template <typename T>
struct ColorParams {
  T sigma = T(0.01);
  T beta = T(0.7);
  T nci_strength = T(0);
  int nci_reach = 3;
  T eps_bulk = T(0.02);
  T grad_threshold = T(1e-6);
  PerturbationForm form = PerturbationForm::Squared;
};

template <class Lat, int A, typename T>
constexpr T inv_cnorm() {
  constexpr auto v = Lat::c[A];
  constexpr int c2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  if constexpr (c2 == 0) return T(0);
  else if constexpr (c2 == 1) return T(1);
  else if constexpr (c2 == 2) return T(0.70710678118654752440084436210485L);
  else return T(0.57735026918962576450914878050196L);
}

namespace detail {
template <typename T>
void color_arrays(const ColorParams<T>& cp, double c[5], int ci[2]) {
  c[0] = double(cp.sigma);
  c[1] = double(cp.beta);
  c[2] = double(cp.nci_strength);
  c[3] = double(cp.eps_bulk);
  c[4] = double(cp.grad_threshold);
  ci[0] = cp.nci_reach;
  ci[1] = cp.form == PerturbationForm::Linear ? 1 : 0;
}

template <class Lat, typename T, class Op>
void two_phase(TwoFluidFieldSet<T>& s, const NodeGeometry& geo, const BoundarySpec<T>& spec, T omega,
               const ColorParams<T>& cp, Op&& op) {
  double c[5];
  int ci[2];
  color_arrays(cp, c, ci);
  auto dev = Device::make<Lat, T>(s.dims, double(omega), spec,
                                  any_solid(geo) ? geo.solid : std::vector<std::uint8_t>{}, 2, c, ci);
  upload_two(dev.get(), s);
  op(dev.get());
  download_two(dev.get(), s);
}
}  // namespace detail

template <class Lat, typename T>
void color_moments(TwoFluidFieldSet<T>& s, const NodeGeometry& geo, WorkerPool* = nullptr) {
  detail::two_phase<Lat, T>(s, geo, BoundarySpec<T>::all_periodic(), T(1), ColorParams<T>{},
                            [](tslb_cuda_handle h) { detail::check(tslb_cuda_color_moments(h)); });
}

template <class Lat, typename T>
void gradient_and_nci(TwoFluidFieldSet<T>& s, const NodeGeometry& geo, const BoundarySpec<T>& spec,
                      const ColorParams<T>& cp, WorkerPool* = nullptr) {
  detail::two_phase<Lat, T>(s, geo, spec, T(1), cp,
                            [](tslb_cuda_handle h) { detail::check(tslb_cuda_gradient_and_nci(h)); });
}

template <class Lat, typename T>
void prepare_stress(TwoFluidFieldSet<T>& s, const NodeGeometry& geo, const CollisionParams<T>& prm,
                    const ColorParams<T>& cp, WorkerPool* = nullptr) {
  detail::two_phase<Lat, T>(s, geo, BoundarySpec<T>::all_periodic(), prm.omega, cp,
                            [](tslb_cuda_handle h) { detail::check(tslb_cuda_prepare_stress(h)); });
}

template <class Lat, typename T>
void stream_collide_recolor(TwoFluidFieldSet<T>& s, const NodeGeometry& geo, const BoundarySpec<T>& spec,
                            const CollisionParams<T>& prm, const ColorParams<T>& cp, WorkerPool* = nullptr) {
  detail::two_phase<Lat, T>(s, geo, spec, prm.omega, cp,
                            [](tslb_cuda_handle h) { detail::check(tslb_cuda_stream_collide_recolor(h)); });
}

template <class Lat, typename T>
void two_fluid_step(TwoFluidFieldSet<T>& s, const NodeGeometry& geo, const BoundarySpec<T>& spec,
                    const CollisionParams<T>& prm, const ColorParams<T>& cp, WorkerPool* = nullptr) {
  detail::two_phase<Lat, T>(s, geo, spec, prm.omega, cp,
                            [](tslb_cuda_handle h) { detail::check(tslb_cuda_step(h, 1)); });
}

/// nci_force_at (multicomponent.hpp:249-266): per-node force helper on
/// host fields (the device folds the same expression into its step).
template <class Lat, typename T>
inline std::array<T, 3> nci_force_at(const TwoFluidFieldSet<T>& s, const ColorParams<T>& cp, std::size_t idx) {
  std::array<T, 3> F = {T(0), T(0), T(0)};
  if (!s.nci_flag[idx]) return F;
  const auto e = Eigen::Index(idx);
  const T gx = s.gradphi[0][e], gy = s.gradphi[1][e];
  const T gz = Lat::dim == 3 ? s.gradphi[2][e] : T(0);
  const T gn = std::sqrt(gx * gx + gy * gy + gz * gz);
  if (gn <= cp.grad_threshold) return F;
  const T scale = cp.nci_strength * s.rho_r[e] / gn;
  F = {scale * gx, scale * gy, scale * gz};
  return F;
}

template <typename T>
struct ColorInit {
  T rho_r{}, rho_b{};
  T ux{}, uy{}, uz{};
};

/// initialize_colors (multicomponent.hpp:427-449): host initialiser.
template <class Lat, typename T, class F>
void initialize_colors(TwoFluidFieldSet<T>& s, const NodeGeometry& geo, F&& node_state) {
  const GridDims g = s.dims;
  for (int k = 0; k < g.nz; ++k)
    for (int j = 0; j < g.ny; ++j)
      for (int i = 0; i < g.nx; ++i) {
        const std::size_t idx = linear_index(g, i, j, k);
        if (geo.solid[idx]) continue;
        const ColorInit<T> ci = node_state(i, j, k);
        const T r = ci.rho_r + ci.rho_b;
        const NodeMoments<T> m = prepare_node(r, ci.ux, ci.uy, ci.uz, T(0), T(0), T(0), T(0), T(0), T(0));
        const T frac = ci.rho_r / r;
        for_each_dir<Lat>([&](auto A) {
          constexpr int a = decltype(A)::value;
          const T fe = equilibrium_dir<Lat, a, T>(m);
          s.fr[std::size_t(a)][Eigen::Index(idx)] = frac * fe;
          s.fb[std::size_t(a)][Eigen::Index(idx)] = fe - frac * fe;
        });
      }
}

// ===========================================================================
// solvers (solver.hpp)
// ===========================================================================
template <class F>
decltype(auto) dispatch_lattice(LatticeKind k, F&& f) {
  if (k == LatticeKind::D2Q9) return f(std::type_identity<D2Q9>{});
  if (k == LatticeKind::D3Q27) return f(std::type_identity<D3Q27>{});
  return f(std::type_identity<D3Q19>{});
}

template <typename T>
struct StabilityReport {
  bool finite = true;
  T max_speed = T(0);
  T min_rho = T(0);
  T max_rho = T(0);
  std::int64_t first_bad = -1;  // new: first non-finite node (device scan)
  bool stable() const { return finite && max_speed < T(0.3) * T(0.57735026918962576L); }
};

namespace detail {
template <typename T>
StabilityReport<T> stability_of(tslb_cuda_handle h) {
  int fin = 1;
  double ms = 0, lo = 0, hi = 0;
  std::int64_t bad = -1;
  check(tslb_cuda_stability(h, &fin, &ms, &lo, &hi, &bad));
  StabilityReport<T> r;
  r.finite = fin != 0;
  r.max_speed = T(ms);
  r.min_rho = T(lo);
  r.max_rho = T(hi);
  r.first_bad = bad;
  return r;
}
}  // namespace detail

/// scan_stability (solver.hpp:39-65) on host arrays, evaluated on the device.
template <typename T>
StabilityReport<T> scan_stability(const GridDims& g, const std::vector<std::uint8_t>& solid, const FieldArray<T>& rho,
                                  const std::vector<FieldArray<T>>& mom) {
  const bool three = mom.size() == 3;
  auto dev = three ? detail::Device::make<D3Q19, T>(g, 1.0, BoundarySpec<T>::all_periodic(), solid, 1)
                   : detail::Device::make<D2Q9, T>(g, 1.0, BoundarySpec<T>::all_periodic(), solid, 1);
  detail::upload_one(dev.get(), TSLB_FIELD_RHO, rho);
  detail::upload_field(dev.get(), TSLB_FIELD_MOM, mom, g.n());
  return detail::stability_of<T>(dev.get());
}

/// Shared Sim machinery: device residency + host mirror bookkeeping.
template <class Lat, typename T, class Fields>
class SimCore {
 public:
  using Lattice = Lat;
  using Scalar = T;

  GridDims dims() const { return dims_; }
  const CollisionParams<T>& params() const { return prm_; }
  const BoundarySpec<T>& boundary() const { return spec_; }
  const NodeGeometry& geometry() const { return geo_; }
  long steps() const { return steps_; }
  WorkerPool* pool() const { return pool_; }

  /// Mutable host view: synchronised, and uploaded before the next device op.
  Fields& fields() {
    pull();
    host_dirty_ = true;
    return host_;
  }
  /// Read-only host view.
  const Fields& fields() const {
    pull();
    return host_;
  }

  void run(long n) {
    push();
    detail::check(tslb_cuda_step(dev_.get(), n));
    steps_ += n;
    device_newer_ = true;
  }
  void step() { run(1); }

  void refresh_moments() {
    push();
    detail::check(tslb_cuda_refresh_moments(dev_.get()));
    device_newer_ = true;
  }

  StabilityReport<T> stability() const {
    const_cast<SimCore*>(this)->push();
    return detail::stability_of<T>(dev_.get());
  }

  /// Device handle, for callers that want the C-ABI directly.
  tslb_cuda_handle handle() const { return dev_.get(); }

 protected:
  SimCore(const GridDims& g, const CollisionParams<T>& prm, const BoundarySpec<T>& spec,
          const std::vector<std::uint8_t>& solid, WorkerPool* pool, int components, const double* color,
          const int* color_i)
      : dims_(g), prm_(prm), spec_(spec), pool_(pool) {
    dev_ = detail::Device::make<Lat, T>(g, double(prm.omega), spec, solid, components, color, color_i);
    if (components == 1 && (prm.force[0] != T(0) || prm.force[1] != T(0) || prm.force[2] != T(0))) {
      const double f3[3] = {double(prm.force[0]), double(prm.force[1]), double(prm.force[2])};
      detail::check(tslb_cuda_set_body_force(dev_.get(), f3));
    }
    geo_ = detail::geometry_of(dev_.get(), g);
  }

  virtual void upload_all(const Fields&) = 0;
  virtual void download_all(Fields&) const = 0;

  void push() {
    if (host_dirty_) {
      upload_all(host_);
      host_dirty_ = false;
    }
  }
  void pull() const {
    if (device_newer_) {
      download_all(host_);
      device_newer_ = false;
    }
  }

  GridDims dims_;
  CollisionParams<T> prm_;
  BoundarySpec<T> spec_;
  NodeGeometry geo_;
  WorkerPool* pool_;
  detail::Device dev_;
  mutable Fields host_;
  mutable bool device_newer_ = false;
  bool host_dirty_ = false;
  long steps_ = 0;
};

template <class Lat, typename T>
class SingleFluidSim : public SimCore<Lat, T, FieldSet<T>> {
  using Base = SimCore<Lat, T, FieldSet<T>>;

 public:
  SingleFluidSim(const GridDims& g, const CollisionParams<T>& prm, const BoundarySpec<T>& spec,
                 const std::vector<std::uint8_t>& solid = {}, WorkerPool* pool = nullptr)
      : Base(g, prm, spec, solid, pool, 1, nullptr, nullptr) {
    this->host_ = allocate_fields<T>(g, make_descriptor<T>(Lat::kind));
  }
  ~SingleFluidSim() = default;

  /// Total mass and momentum over fluid nodes (deterministic fp64 device
  /// tree, rounded to T; the reference sums serially in T).
  void totals(T& mass, std::array<T, 3>& momentum) const {
    const_cast<SingleFluidSim*>(this)->push();
    double m = 0, p[3] = {0, 0, 0};
    detail::check(tslb_cuda_totals(this->dev_.get(), &m, p));
    mass = T(m);
    momentum = {T(p[0]), T(p[1]), T(p[2])};
  }

 protected:
  void upload_all(const FieldSet<T>& s) override { detail::upload_single(this->dev_.get(), s); }
  void download_all(FieldSet<T>& s) const override { detail::download_single(this->dev_.get(), s); }
};

template <class Lat, typename T>
class TwoFluidSim : public SimCore<Lat, T, TwoFluidFieldSet<T>> {
  using Base = SimCore<Lat, T, TwoFluidFieldSet<T>>;

 public:
  TwoFluidSim(const GridDims& g, const CollisionParams<T>& prm, const ColorParams<T>& cp,
              const BoundarySpec<T>& spec, const std::vector<std::uint8_t>& solid = {}, WorkerPool* pool = nullptr)
      : Base(g, prm, spec, solid, pool, 2, color_of(cp).c, color_of(cp).ci), cp_(cp) {
    this->host_ = allocate_two_fluid<T>(g, make_descriptor<T>(Lat::kind));
  }

  const ColorParams<T>& colors() const { return cp_; }

  void color_masses(T& red, T& blue) const {
    const_cast<TwoFluidSim*>(this)->push();
    double r = 0, b = 0;
    detail::check(tslb_cuda_color_masses(this->dev_.get(), &r, &b));
    red = T(r);
    blue = T(b);
  }

 protected:
  void upload_all(const TwoFluidFieldSet<T>& s) override { detail::upload_two(this->dev_.get(), s); }
  void download_all(TwoFluidFieldSet<T>& s) const override { detail::download_two(this->dev_.get(), s); }

 private:
  struct Packed {
    double c[5];
    int ci[2];
  };
  static Packed color_of(const ColorParams<T>& cp) {
    Packed p;
    detail::color_arrays(cp, p.c, p.ci);
    return p;
  }
  ColorParams<T> cp_;
};

// ===========================================================================
// measurement (bench.hpp)
// ===========================================================================
struct KernelCost {
  double flops = 0;
  double bytes = 0;
  double intensity = 0;
};

/// count_kernel_cost (bench.hpp:30-66), same counting rules, any lattice.
inline KernelCost count_kernel_cost(LatticeKind kind, std::size_t elem_bytes) {
  const auto d = make_descriptor<double>(kind);
  const int D = d.dim, np = D * (D + 1) / 2;
  double moments = 1 + 3 * D + 2 * (np - D);
  double collide = 12;
  for (int a = 0; a < d.q; ++a) {
    int nz = 0;
    for (int ax = 0; ax < 3; ++ax) nz += d.c(ax, a) != 0;
    const int pairs = (d.c(0, a) && d.c(1, a)) + (d.c(0, a) && d.c(2, a)) + (d.c(1, a) && d.c(2, a));
    moments += 1 + 2 * nz + pairs;
    collide += nz == 0 ? 6 : (nz + 6) + (nz + pairs + 2) + 2;
  }
  KernelCost c;
  c.flops = moments + collide;
  c.bytes = 2.0 * double(d.q + 1 + D + np) * double(elem_bytes);
  c.intensity = c.flops / c.bytes;
  return c;
}

struct MachineModel {
  double peak_flops = 0;
  double peak_bandwidth = 0;
};

inline double roofline_bound(const MachineModel& m, double intensity) {
  const double mem = m.peak_bandwidth * intensity;
  return mem < m.peak_flops ? mem : m.peak_flops;
}

inline std::uint64_t fnv1a(const void* data, std::size_t n, std::uint64_t h = 0xcbf29ce484222325ull) {
  const auto* p = static_cast<const unsigned char*>(data);
  for (std::size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
  return h;
}

template <typename T>
std::uint64_t state_digest(const FieldSet<T>& s) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (const auto& a : s.f) h = fnv1a(a.data(), std::size_t(a.size()) * sizeof(T), h);
  return h;
}

template <typename T>
std::uint64_t state_digest(const TwoFluidFieldSet<T>& s) {
  std::uint64_t h = 0xcbf29ce484222325ull;
  for (const auto& a : s.fr) h = fnv1a(a.data(), std::size_t(a.size()) * sizeof(T), h);
  for (const auto& a : s.fb) h = fnv1a(a.data(), std::size_t(a.size()) * sizeof(T), h);
  return h;
}

struct BenchResult {
  std::string lattice;
  GridDims dims;
  long steps = 0;
  int workers = 1;
  double seconds = 0;
  double glups = 0;
  double mlups = 0;
  KernelCost cost;
  std::uint64_t digest = 0;
};

/// run_benchmark (bench.hpp:129-157): periodic shear box, device-resident,
/// device time of `steps` steps after `warmup`.
template <class Lat, typename T>
BenchResult run_benchmark(const GridDims& g, const CollisionParams<T>& prm, long steps, long warmup,
                          WorkerPool* pool) {
  SingleFluidSim<Lat, T> sim(g, prm, BoundarySpec<T>::all_periodic(), {}, pool);
  initialize_regularized<Lat, T>(sim.fields(), sim.geometry(), [&](int, int j, int) {
    const T ux = T(0.02) * std::sin(2.0 * std::numbers::pi * j / g.ny);
    return prepare_node(T(1), ux, T(0), T(0), T(0), T(0), T(0), T(0), T(0), T(0));
  });
  sim.run(warmup);
  double ms = 0;
  detail::check(tslb_cuda_time_steps(sim.handle(), steps, &ms));
  BenchResult r;
  r.lattice = lattice_name(Lat::kind);
  r.dims = g;
  r.steps = steps;
  r.workers = pool ? pool->size() : 1;
  r.seconds = ms / 1e3;
  const double updates = double(g.n()) * double(steps);
  r.glups = updates / 1e9 / r.seconds;
  r.mlups = updates / 1e6 / r.seconds;
  r.cost = count_kernel_cost(Lat::kind, sizeof(T));
  r.digest = state_digest(static_cast<const SingleFluidSim<Lat, T>&>(sim).fields());
  return r;
}

}  // namespace tslb
