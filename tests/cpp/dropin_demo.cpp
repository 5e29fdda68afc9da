// Drop-in demo/test: a reference-style driver compiled against include/tslb
// (the B200 drop-in) -- same types and calls as a tslb user would write.
// Exit status 0 = all checks passed.
#include <cmath>
#include <cstdio>
#include <numbers>

#include "tslb/bench.hpp"
#include "tslb/kernels.hpp"
#include "tslb/multicomponent.hpp"
#include "tslb/solver.hpp"

using namespace tslb;

static int failures = 0;
#define EXPECT(cond)                                                  \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "%s:%d: FAILED %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

template <class Lat, typename T>
void sim_vs_free_functions() {
  const GridDims g{24, 18, Lat::dim == 3 ? 10 : 1};
  auto spec = BoundarySpec<T>::all_periodic();
  spec.faces[YMin].kind = FaceKind::NoSlipWall;
  spec.faces[YMax].kind = FaceKind::MovingWall;
  spec.faces[YMax].u_wall = {T(0.04), T(0), T(0)};
  CollisionParams<T> prm;
  prm.omega = T(1.3);
  SingleFluidSim<Lat, T> sim(g, prm, spec);
  initialize_regularized<Lat, T>(sim.fields(), sim.geometry(), [&](int i, int j, int k) {
    const T ux = T(0.01 * std::sin(2 * std::numbers::pi * (j + k) / g.ny));
    const T uy = T(0.005 * std::cos(2 * std::numbers::pi * i / g.nx));
    return prepare_node(T(1), ux, uy, T(0), T(0), T(0), T(0), T(0), T(0), T(0));
  });
  FieldSet<T> copy = static_cast<const SingleFluidSim<Lat, T>&>(sim).fields();
  sim.run(7);
  for (int s = 0; s < 7; ++s) fused_step<Lat, T>(copy, sim.geometry(), spec, prm);
  const auto& a = static_cast<const SingleFluidSim<Lat, T>&>(sim).fields();
  EXPECT(state_digest(a) == state_digest(copy));
  // conservation of mass with walls
  sim.refresh_moments();
  T m0;
  std::array<T, 3> p0;
  sim.totals(m0, p0);
  sim.run(50);
  sim.refresh_moments();
  T m1;
  std::array<T, 3> p1;
  sim.totals(m1, p1);
  EXPECT(std::abs(double(m1 - m0)) / double(m0) < (sizeof(T) == 8 ? 1e-12 : 1e-5));
  EXPECT(sim.stability().stable());
}

template <typename T>
void two_fluid_roundtrip() {
  const GridDims g{32, 32, 1};
  CollisionParams<T> prm;
  prm.omega = T(1);
  ColorParams<T> cp;
  cp.sigma = T(0.02);
  TwoFluidSim<D2Q9, T> sim(g, prm, cp, BoundarySpec<T>::all_periodic());
  initialize_colors<D2Q9, T>(sim.fields(), sim.geometry(), [&](int i, int j, int) {
    const double r = std::hypot(i - 15.5, j - 15.5);
    const double phi = std::tanh(2.0 * (8.0 - r) / 3.0);
    return ColorInit<T>{T(0.5 * (1 + phi)), T(0.5 * (1 - phi)), T(0), T(0), T(0)};
  });
  sim.refresh_moments();
  T r0, b0;
  sim.color_masses(r0, b0);
  sim.run(40);
  sim.refresh_moments();
  T r1, b1;
  sim.color_masses(r1, b1);
  EXPECT(std::abs(double(r1 - r0)) / double(r0) < (sizeof(T) == 8 ? 1e-12 : 1e-5));
  EXPECT(std::abs(double(b1 - b0)) / double(b0) < (sizeof(T) == 8 ? 1e-12 : 1e-5));
}

int main() {
  sim_vs_free_functions<D2Q9, double>();
  sim_vs_free_functions<D3Q19, float>();
  sim_vs_free_functions<D3Q27, double>();
  two_fluid_roundtrip<double>();
  two_fluid_roundtrip<float>();
  const auto c = count_kernel_cost(LatticeKind::D3Q19, 4);
  EXPECT(c.flops == 377 && c.bytes == 232);
  const auto r = run_benchmark<D3Q19, float>(GridDims{64, 64, 64}, CollisionParams<float>{1.6f, 1.f}, 5, 2, nullptr);
  EXPECT(r.glups > 0);
  std::printf("dropin_demo: %s (%d failures); run_benchmark 64^3 D3Q19 f32: %.3f GLUPS\n",
              failures ? "FAILED" : "ok", failures, r.glups);
  return failures;
}
