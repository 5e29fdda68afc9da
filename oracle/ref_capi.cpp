// C-ABI wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/tslb/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libtslb_ref.so.
//
// TEST INFRASTRUCTURE ONLY (the "reference" checker and the CPU baseline of
// bench.py --impl reference). Nothing in the product links or loads this.
// Flat buffers are [direction][node] SoA with the reference's x-fastest
// linear_index (fields.hpp:26-29). Scalars: 0 = double, 1 = float storage.
// Lattices: 0 = D2Q9, 1 = D3Q19 (the reference has no D3Q27).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "tslb/bench.hpp"
#include "tslb/boundary.hpp"
#include "tslb/kernels.hpp"
#include "tslb/multicomponent.hpp"
#include "tslb/parallel.hpp"
#include "tslb/solver.hpp"

using namespace tslb;

namespace {

thread_local std::string g_err;

template <typename T>
BoundarySpec<T> make_spec(const int* kinds, const double* uw) {
  BoundarySpec<T> s;
  for (int f = 0; f < 6; ++f) {
    s.faces[f].kind = FaceKind(kinds[f]);
    for (int d = 0; d < 3; ++d) s.faces[f].u_wall[d] = T(uw[3 * f + d]);
  }
  return s;
}

std::vector<std::uint8_t> make_solid(const std::uint8_t* solid, std::size_t n) {
  if (!solid) return {};
  return std::vector<std::uint8_t>(solid, solid + n);
}

template <typename T>
void load_arrays(std::vector<FieldArray<T>>& dst, const T* src, std::size_t n) {
  for (std::size_t a = 0; a < dst.size(); ++a)
    std::memcpy(dst[a].data(), src + a * n, n * sizeof(T));
}

template <typename T>
void store_arrays(const std::vector<FieldArray<T>>& src, T* dst, std::size_t n) {
  for (std::size_t a = 0; a < src.size(); ++a)
    std::memcpy(dst + a * n, src[a].data(), n * sizeof(T));
}

template <typename T>
void store_one(const FieldArray<T>& src, T* dst, std::size_t n) {
  std::memcpy(dst, src.data(), n * sizeof(T));
}

// moments block layout: rho, mom[D], pineq[np]
template <typename T>
void store_moments(const FieldSet<T>& s, T* out) {
  const std::size_t n = s.n();
  std::size_t o = 0;
  store_one(s.rho, out, n);
  o += n;
  for (const auto& a : s.mom) {
    store_one(a, out + o, n);
    o += n;
  }
  for (const auto& a : s.pineq) {
    store_one(a, out + o, n);
    o += n;
  }
}

template <typename T>
void load_moments(FieldSet<T>& s, const T* in) {
  const std::size_t n = s.n();
  std::size_t o = 0;
  std::memcpy(s.rho.data(), in, n * sizeof(T));
  o += n;
  for (auto& a : s.mom) {
    std::memcpy(a.data(), in + o, n * sizeof(T));
    o += n;
  }
  for (auto& a : s.pineq) {
    std::memcpy(a.data(), in + o, n * sizeof(T));
    o += n;
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  } catch (...) {
    g_err = "unknown error";
    return 1;
  }
}

template <class F>
void with_lattice(int lattice, F&& f) {
  if (lattice == 0)
    f(std::type_identity<D2Q9>{});
  else if (lattice == 1)
    f(std::type_identity<D3Q19>{});
  else
    throw std::invalid_argument("reference has no lattice id " +
                                std::to_string(lattice));
}

template <class F>
void with_scalar(int scalar, F&& f) {
  if (scalar == 0)
    f(double(0));
  else
    f(float(0));
}

// mode: 0 = fused_step, 1 = reference_step (two-buffer), 2 = compute_moments
// only, 3 = stream_collide_fused only (moments taken from `moments`),
// 4 = stream_only (pure streaming, f -> f)
template <class Lat, typename T>
void run_single(int nx, int ny, int nz, double omega, const int* kinds,
                const double* uw, const std::uint8_t* solid, T* f, T* moments,
                long steps, int workers, int mode) {
  const GridDims g{nx, ny, nz};
  const auto spec = make_spec<T>(kinds, uw);
  const auto geo = classify_nodes<T, Lat>(g, spec, make_solid(solid, g.n()));
  CollisionParams<T> prm;
  prm.omega = T(omega);
  auto s = allocate_fields<T>(g, make_descriptor<T>(Lat::kind));
  load_arrays(s.f, f, g.n());
  if (moments) load_moments(s, moments);
  std::unique_ptr<WorkerPool> pool;
  if (workers > 1) pool = std::make_unique<WorkerPool>(workers);
  // the second population buffer only for the two-buffer modes (a full-size
  // fused run -- tests/test_gpu_configs.py -- does not need the extra copy)
  std::vector<FieldArray<T>> scratch;
  if (mode == 1 || mode == 4) scratch = s.f;
  for (long k = 0; k < steps; ++k) {
    switch (mode) {
      case 0: fused_step<Lat, T>(s, geo, spec, prm, pool.get()); break;
      case 1: reference_step<Lat, T>(s, scratch, geo, spec, prm, pool.get()); break;
      case 2: compute_moments<Lat, T>(s, geo, pool.get()); break;
      case 3: stream_collide_fused<Lat, T>(s, geo, spec, prm, pool.get()); break;
      case 4:
        for (auto& a : scratch) a.setZero();
        stream_only<Lat, T>(s, scratch, geo, spec, pool.get());
        s.f.swap(scratch);
        break;
      default: throw std::invalid_argument("bad mode");
    }
  }
  store_arrays(s.f, f, g.n());
  if (moments) store_moments(s, moments);
}

}  // namespace

extern "C" {

const char* tslbref_last_error() { return g_err.c_str(); }

int tslbref_classify(int lattice, int nx, int ny, int nz, const int* kinds,
                     const double* uw, const std::uint8_t* solid,
                     std::uint8_t* solid_out, std::uint32_t* slow_out,
                     std::uint64_t* n_fluid) {
  return guarded([&] {
    with_lattice(lattice, [&](auto L) {
      using Lat = typename decltype(L)::type;
      const GridDims g{nx, ny, nz};
      const auto geo = classify_nodes<double, Lat>(
          g, make_spec<double>(kinds, uw), make_solid(solid, g.n()));
      std::memcpy(solid_out, geo.solid.data(), g.n());
      std::memcpy(slow_out, geo.slow_mask.data(), g.n() * 4);
      *n_fluid = geo.n_fluid;
    });
  });
}

int tslbref_single_run(int lattice, int scalar, int nx, int ny, int nz,
                       double omega, const int* kinds, const double* uw,
                       const std::uint8_t* solid, void* f, void* moments,
                       long steps, int workers, int mode) {
  return guarded([&] {
    with_lattice(lattice, [&](auto L) {
      using Lat = typename decltype(L)::type;
      with_scalar(scalar, [&](auto z) {
        using T = decltype(z);
        run_single<Lat, T>(nx, ny, nz, omega, kinds, uw, solid,
                           static_cast<T*>(f), static_cast<T*>(moments), steps,
                           workers, mode);
      });
    });
  });
}

// Two-fluid run. cp = {sigma, beta, nci_strength, eps_bulk, grad_threshold},
// ip = {nci_reach, form(0 squared, 1 linear)}.
// out layout (n scalars each): rho_r, rho_b, rho, mom[D], pineq[np], phi,
// gradphi[D]; flags: n bytes. refresh != 0 calls refresh_moments() at the end.
// mode: 0 = two_fluid_step x steps; 1 = color_moments + gradient_and_nci only
// on the given phi (phi_in != NULL seeds phi, no f needed).
int tslbref_two_run(int lattice, int scalar, int nx, int ny, int nz,
                    double omega, const double* cp, const int* ip,
                    const int* kinds, const double* uw,
                    const std::uint8_t* solid, void* fr, void* fb, void* out,
                    std::uint8_t* flags, long steps, int workers, int refresh,
                    int mode, const void* phi_in) {
  return guarded([&] {
    with_lattice(lattice, [&](auto L) {
      using Lat = typename decltype(L)::type;
      with_scalar(scalar, [&](auto z) {
        using T = decltype(z);
        const GridDims g{nx, ny, nz};
        const std::size_t n = g.n();
        const auto spec = make_spec<T>(kinds, uw);
        CollisionParams<T> prm;
        prm.omega = T(omega);
        ColorParams<T> c;
        c.sigma = T(cp[0]);
        c.beta = T(cp[1]);
        c.nci_strength = T(cp[2]);
        c.eps_bulk = T(cp[3]);
        c.grad_threshold = T(cp[4]);
        c.nci_reach = ip[0];
        c.form = ip[1] ? PerturbationForm::Linear : PerturbationForm::Squared;
        std::unique_ptr<WorkerPool> pool;
        if (workers > 1) pool = std::make_unique<WorkerPool>(workers);
        TwoFluidSim<Lat, T> sim(g, prm, c, spec, make_solid(solid, n),
                                pool.get());
        auto& s = sim.fields();
        if (mode == 1) {
          std::memcpy(s.phi.data(), phi_in, n * sizeof(T));
          gradient_and_nci<Lat, T>(s, sim.geometry(), spec, c, pool.get());
        } else {
          load_arrays(s.fr, static_cast<T*>(fr), n);
          load_arrays(s.fb, static_cast<T*>(fb), n);
          sim.run(steps);
          if (refresh) sim.refresh_moments();
          store_arrays(s.fr, static_cast<T*>(fr), n);
          store_arrays(s.fb, static_cast<T*>(fb), n);
        }
        T* o = static_cast<T*>(out);
        store_one(s.rho_r, o, n); o += n;
        store_one(s.rho_b, o, n); o += n;
        store_one(s.rho, o, n); o += n;
        for (const auto& a : s.mom) { store_one(a, o, n); o += n; }
        for (const auto& a : s.pineq) { store_one(a, o, n); o += n; }
        store_one(s.phi, o, n); o += n;
        for (const auto& a : s.gradphi) { store_one(a, o, n); o += n; }
        std::memcpy(flags, s.nci_flag.data(), n);
      });
    });
  });
}

// run_benchmark (bench.hpp:129-157) on a periodic shear box.
int tslbref_bench(int lattice, int scalar, int nx, int ny, int nz,
                  double omega, long steps, long warmup, int workers,
                  double* seconds, double* glups, std::uint64_t* digest) {
  return guarded([&] {
    with_lattice(lattice, [&](auto L) {
      using Lat = typename decltype(L)::type;
      with_scalar(scalar, [&](auto z) {
        using T = decltype(z);
        CollisionParams<T> prm;
        prm.omega = T(omega);
        std::unique_ptr<WorkerPool> pool;
        if (workers > 1) pool = std::make_unique<WorkerPool>(workers);
        const auto r = run_benchmark<Lat, T>(GridDims{nx, ny, nz}, prm, steps,
                                             warmup, pool.get());
        *seconds = r.seconds;
        *glups = r.glups;
        *digest = r.digest;
      });
    });
  });
}

// Time `steps` fused steps on a caller-provided state (used by
// bench.py --impl reference for the Taylor-Green workload sample).
int tslbref_time_steps(int lattice, int scalar, int nx, int ny, int nz,
                       double omega, const int* kinds, const double* uw,
                       void* f, long steps, long warmup, int workers,
                       double* seconds) {
  return guarded([&] {
    with_lattice(lattice, [&](auto L) {
      using Lat = typename decltype(L)::type;
      with_scalar(scalar, [&](auto z) {
        using T = decltype(z);
        const GridDims g{nx, ny, nz};
        CollisionParams<T> prm;
        prm.omega = T(omega);
        std::unique_ptr<WorkerPool> pool;
        if (workers > 1) pool = std::make_unique<WorkerPool>(workers);
        SingleFluidSim<Lat, T> sim(g, prm, make_spec<T>(kinds, uw), {},
                                   pool.get());
        load_arrays(sim.fields().f, static_cast<T*>(f), g.n());
        sim.run(warmup);
        const auto t0 = std::chrono::steady_clock::now();
        sim.run(steps);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        store_arrays(sim.fields().f, static_cast<T*>(f), g.n());
      });
    });
  });
}

// The same on any face mix and an optional solid mask (bench.py's CPU rows
// of the other workloads: cavity, channel, porous medium).
int tslbref_time_steps_ex(int lattice, int scalar, int nx, int ny, int nz,
                          double omega, const int* kinds, const double* uw,
                          const std::uint8_t* solid, void* f, long steps,
                          long warmup, int workers, double* seconds) {
  return guarded([&] {
    with_lattice(lattice, [&](auto L) {
      using Lat = typename decltype(L)::type;
      with_scalar(scalar, [&](auto z) {
        using T = decltype(z);
        const GridDims g{nx, ny, nz};
        CollisionParams<T> prm;
        prm.omega = T(omega);
        std::unique_ptr<WorkerPool> pool;
        if (workers > 1) pool = std::make_unique<WorkerPool>(workers);
        SingleFluidSim<Lat, T> sim(g, prm, make_spec<T>(kinds, uw),
                                   make_solid(solid, g.n()), pool.get());
        load_arrays(sim.fields().f, static_cast<T*>(f), g.n());
        sim.run(warmup);
        const auto t0 = std::chrono::steady_clock::now();
        sim.run(steps);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
      });
    });
  });
}

// Time `steps` two_fluid_step calls (TwoFluidSim::run) on a caller-provided
// colour state; cp / ip as tslbref_two_run.
int tslbref_time_two(int lattice, int scalar, int nx, int ny, int nz,
                     double omega, const double* cp, const int* ip,
                     const int* kinds, const double* uw, const void* fr,
                     const void* fb, long steps, long warmup, int workers,
                     double* seconds) {
  return guarded([&] {
    with_lattice(lattice, [&](auto L) {
      using Lat = typename decltype(L)::type;
      with_scalar(scalar, [&](auto z) {
        using T = decltype(z);
        const GridDims g{nx, ny, nz};
        const std::size_t n = g.n();
        CollisionParams<T> prm;
        prm.omega = T(omega);
        ColorParams<T> c;
        c.sigma = T(cp[0]);
        c.beta = T(cp[1]);
        c.nci_strength = T(cp[2]);
        c.eps_bulk = T(cp[3]);
        c.grad_threshold = T(cp[4]);
        c.nci_reach = ip[0];
        c.form = ip[1] ? PerturbationForm::Linear : PerturbationForm::Squared;
        std::unique_ptr<WorkerPool> pool;
        if (workers > 1) pool = std::make_unique<WorkerPool>(workers);
        TwoFluidSim<Lat, T> sim(g, prm, c, make_spec<T>(kinds, uw), {},
                                pool.get());
        load_arrays(sim.fields().fr, static_cast<const T*>(fr), n);
        load_arrays(sim.fields().fb, static_cast<const T*>(fb), n);
        sim.run(warmup);
        const auto t0 = std::chrono::steady_clock::now();
        sim.run(steps);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
      });
    });
  });
}

// The headline workload whole: D3Q19 periodic Taylor-Green on nx*ny*nz with
// the reference's own SingleFluidSim and initialize_regularized
// (kernels.hpp:296-311; the state bench.py's device init writes: rho =
// 1 + 3 (U^2/16)(cos 2X + cos 2Y)(cos 2Z + 2), u = U (sin X cos Y cos Z,
// -cos X sin Y cos Z, 0), Pi^neq = 0), `warmup` untimed steps, then `steps`
// timed ones (bench.py --impl reference). *digest: fnv1a of f afterwards.
// classify_full != 0: classify_nodes over the whole grid (the check of the
// expansion, tests/test_cpu_oracle.py).
int tslbref_time_tgv(int scalar, int nx, int ny, int nz, double omega, double amp, long steps, long warmup,
                     int workers, int classify_full, double* init_seconds, double* seconds, std::uint64_t* digest) {
  return guarded([&] {
    with_scalar(scalar, [&](auto z) {
      using T = decltype(z);
      using Lat = D3Q19;
      const GridDims g{nx, ny, nz};
      CollisionParams<T> prm;
      prm.omega = T(omega);
      std::unique_ptr<WorkerPool> pool;
      if (workers > 1) pool = std::make_unique<WorkerPool>(workers);
      const auto t0 = std::chrono::steady_clock::now();
      if (nx < 3 || ny < 3 || nz < 3) throw std::invalid_argument("tslbref_time_tgv: nx, ny, nz >= 3");
      const auto spec = BoundarySpec<T>::all_periodic();
      // classify_nodes (boundary.hpp:61-111) on 3x3x3 and expanded: without
      // solids a node's slow mask only depends on whether it sits on the low
      // face, inside, or on the high face of each axis (the serial loop over
      // 10^9 nodes would take minutes)
      const NodeGeometry g3 = classify_nodes<T, Lat>(GridDims{3, 3, 3}, spec);
      NodeGeometry geo;
      geo.dims = g;
      geo.solid.assign(g.n(), 0);
      geo.slow_mask.resize(g.n());
      geo.n_fluid = g.n();
      auto cls = [](int c, int n) { return c == 0 ? 0 : c == n - 1 ? 2 : 1; };
      auto fill_geo = [&](int k) {
        for (int j = 0; j < ny; ++j)
          for (int i = 0; i < nx; ++i)
            geo.slow_mask[linear_index(g, i, j, k)] =
                g3.slow_mask[linear_index(GridDims{3, 3, 3}, cls(i, nx), cls(j, ny), cls(k, nz))];
      };
      auto par = [&](auto&& fn) {
        const int nt = std::max(1, workers);
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t)
          th.emplace_back([&, t] {
            for (int k = t; k < nz; k += nt) fn(k);
          });
        for (auto& x : th) x.join();
      };
      if (classify_full) geo = classify_nodes<T, Lat>(g, spec);
      else par(fill_geo);
      FieldSet<T> s = allocate_fields<T>(g, make_descriptor<T>(Lat::kind));
      const auto tc = std::chrono::steady_clock::now();
      // initialize_regularized's node loop (kernels.hpp:296-311), split over
      // z planes on the worker threads (a 1024^3 state takes minutes on one
      // thread); trig from per-axis tables
      const double pi2 = 2.0 * 3.14159265358979323846;
      auto tab = [&](int n, double (*fn)(double), double mul) {
        std::vector<double> t(static_cast<std::size_t>(n));
        for (int i = 0; i < n; ++i) t[std::size_t(i)] = fn(mul * pi2 * (i + 0.5) / n);
        return t;
      };
      const auto sx = tab(nx, std::sin, 1), cx = tab(nx, std::cos, 1), c2x = tab(nx, std::cos, 2);
      const auto sy = tab(ny, std::sin, 1), cy = tab(ny, std::cos, 1), c2y = tab(ny, std::cos, 2);
      const auto cz = tab(nz, std::cos, 1), c2z = tab(nz, std::cos, 2);
      auto plane = [&](int k) {
        for (int j = 0; j < ny; ++j)
          for (int i = 0; i < nx; ++i) {
            const double rho = 1.0 + 3.0 * (amp * amp / 16.0) * (c2x[i] + c2y[j]) * (c2z[k] + 2.0);
            const double ux = amp * sx[i] * cy[j] * cz[k];
            const double uy = -amp * cx[i] * sy[j] * cz[k];
            const NodeMoments<T> m = prepare_node<T>(T(rho), T(ux), T(uy), T(0), T(0), T(0), T(0), T(0), T(0), T(0));
            const Eigen::Index idx = Eigen::Index(linear_index(g, i, j, k));
            for_each_dir<Lat>([&](auto A) {
              constexpr int a = A.value;
              s.f[a][idx] = equilibrium_dir<Lat, a, T>(m) + regularized_dir<Lat, a, T>(m);
            });
          }
      };
      par(plane);
      // SingleFluidSim::step (solver.hpp:87-90) is fused_step
      const auto t1 = std::chrono::steady_clock::now();
      for (long k = 0; k < warmup; ++k) fused_step<Lat, T>(s, geo, spec, prm, pool.get());
      const auto t2 = std::chrono::steady_clock::now();
      for (long k = 0; k < steps; ++k) fused_step<Lat, T>(s, geo, spec, prm, pool.get());
      const auto t3 = std::chrono::steady_clock::now();
      *init_seconds = std::chrono::duration<double>(t1 - t0).count();
      if (std::getenv("TSLBREF_VERBOSE"))
        std::fprintf(stderr, "tslbref_time_tgv: construct %.2f s, init %.2f s\n",
                     std::chrono::duration<double>(tc - t0).count(), std::chrono::duration<double>(t1 - tc).count());
      *seconds = std::chrono::duration<double>(t3 - t2).count();
      std::uint64_t h = 0xcbf29ce484222325ull;
      for (const auto& a : s.f) h = fnv1a(a.data(), std::size_t(a.size()) * sizeof(T), h);
      *digest = h;
    });
  });
}

std::uint64_t tslbref_fnv1a(const void* data, std::size_t n, std::uint64_t h) {
  return fnv1a(data, n, h);
}

void tslbref_census(int lattice, int elem_bytes, double* flops, double* bytes) {
  const auto c = count_kernel_cost(lattice == 0 ? LatticeKind::D2Q9
                                                : LatticeKind::D3Q19,
                                   std::size_t(elem_bytes));
  *flops = c.flops;
  *bytes = c.bytes;
}

}  // extern "C"
