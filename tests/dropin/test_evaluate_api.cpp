// The repo's own C++ checks of the batched drop-in API (include/sphbi/evaluate.hpp):
// sphbi::evaluate and sphbi::BasisSweep against per-pair sphbi::integrate_triangle
// calls of the same headers (everything runs on the B200 through libsphbi_cuda.so).
#include <cmath>
#include <random>

#include "gtest/gtest.h"
#include "sphbi/evaluate.hpp"

namespace {

struct Scene {
  std::vector<sphbi::Point2> particles;
  std::vector<sphbi::Triangle> mesh;
  std::vector<std::pair<std::int64_t, std::int64_t>> pairs;
};

// a fan of triangles around (0.5, 0.5) and particles scattered over it
Scene make_scene(unsigned seed) {
  Scene s;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  const int nt = 12;
  for (int k = 0; k < nt; ++k) {
    const double a0 = 2.0 * M_PI * k / nt, a1 = 2.0 * M_PI * (k + 1) / nt;
    s.mesh.push_back(sphbi::Triangle{{0.5, 0.5},
                                     {0.5 + 0.4 * std::cos(a0), 0.5 + 0.4 * std::sin(a0)},
                                     {0.5 + 0.4 * std::cos(a1), 0.5 + 0.4 * std::sin(a1)},
                                     std::nullopt});
  }
  for (int i = 0; i < 200; ++i) s.particles.push_back({u(rng), u(rng)});
  for (std::int64_t i = 0; i < (std::int64_t)s.particles.size(); ++i)
    for (std::int64_t t = 0; t < nt; t += 1) s.pairs.push_back({i, t});
  return s;
}

double tol(double a, double b, double c2, double h) {
  return std::max(1e-11 * std::max(std::abs(a), std::abs(b)), 1e-13 * c2 / (h * h));
}

}  // namespace

TEST(EvaluateApi, ExplicitPairsMatchPerPairCalls) {
  Scene s = make_scene(1);
  const double h = 0.2;
  const auto table = sphbi::table1_terms(sphbi::wendland4());
  std::mt19937_64 rng(5);
  std::normal_distribution<double> nd;
  for (auto& t : s.mesh) t.values = std::array<double, 3>{nd(rng), nd(rng), nd(rng)};
  const auto res = sphbi::evaluate(s.particles, h, s.mesh, table, &s.pairs);
  for (std::size_t i = 0; i < s.particles.size(); ++i) {
    double v = 0, gx = 0, gy = 0;
    for (std::size_t t = 0; t < s.mesh.size(); ++t) {
      const auto r = sphbi::integrate_triangle(s.particles[i], h, s.mesh[t], table);
      v += r.value;
      gx += r.gradient[0];
      gy += r.gradient[1];
    }
    EXPECT_LE(std::abs(res[i].value - v), tol(res[i].value, v, table.normalization, h));
    EXPECT_LE(std::abs(res[i].gradient[0] - gx), tol(res[i].gradient[0], gx, table.normalization, h));
    EXPECT_LE(std::abs(res[i].gradient[1] - gy), tol(res[i].gradient[1], gy, table.normalization, h));
  }
}

TEST(EvaluateApi, BasisSweepVariantsMatchWeightedIntegrals) {
  Scene s = make_scene(2);
  const double h = 0.15;
  const auto table = sphbi::table1_terms(sphbi::wendland4());
  sphbi::BasisSweep sweep(s.particles, h, s.mesh, table);  // device cell list
  EXPECT_GT(sweep.pair_count(), 0);
  std::mt19937_64 rng(9);
  std::normal_distribution<double> nd;
  std::uniform_real_distribution<double> ud(0.5, 2.0);
  std::vector<std::array<double, 3>> A(s.mesh.size()), rho(s.mesh.size());
  std::vector<double> a0(s.particles.size()), rho0(s.particles.size());
  for (std::size_t t = 0; t < s.mesh.size(); ++t) {
    A[t] = {nd(rng), nd(rng), nd(rng)};
    rho[t] = {ud(rng), ud(rng), ud(rng)};
  }
  for (std::size_t i = 0; i < s.particles.size(); ++i) {
    a0[i] = nd(rng);
    rho0[i] = ud(rng);
  }
  for (auto var : {sphbi::GradientVariant::basic, sphbi::GradientVariant::difference,
                   sphbi::GradientVariant::symmetric}) {
    const auto res = sweep.apply(var, A, rho, a0, rho0);
    for (std::size_t i = 0; i < s.particles.size(); ++i) {
      double v = 0, gx = 0, gy = 0;
      for (std::size_t t = 0; t < s.mesh.size(); ++t) {
        // the pair predicate is d(p, closed triangle) < h; farther pairs contribute 0
        const auto w = sphbi::gradient_variant_weights(var, a0[i], rho0[i], A[t], rho[t]);
        const auto r = sphbi::integrate_triangle(s.particles[i], h, s.mesh[t], w, table);
        v += r.value;
        gx += r.gradient[0];
        gy += r.gradient[1];
      }
      EXPECT_LE(std::abs(res[i].value - v), tol(res[i].value, v, table.normalization, h));
      EXPECT_LE(std::abs(res[i].gradient[0] - gx), tol(res[i].gradient[0], gx, table.normalization, h));
      EXPECT_LE(std::abs(res[i].gradient[1] - gy), tol(res[i].gradient[1], gy, table.normalization, h));
    }
  }
  rho[3][1] = -1.0;
  EXPECT_THROW(sweep.apply(sphbi::GradientVariant::difference, A, rho, a0, rho0), std::domain_error);
}

// SPH coupling: contact-point channel and boundary normals
// against per-pair sphbi::integrate_triangle with a constant field.
TEST(EvaluateApi, CouplingPairWeightsAndNormals) {
  const Scene s = make_scene(17);
  const double h = 0.3;
  const auto table = sphbi::table1_terms(sphbi::wendland4());
  sphbi::BasisSweep sweep(s.particles, h, s.mesh, table, &s.pairs);
  const std::int64_t m = sweep.pair_count();
  ASSERT_EQ(m, static_cast<std::int64_t>(s.pairs.size()));  // explicit pairs, kept in (particle, triangle) order
  std::vector<double> w(m);
  for (std::int64_t k = 0; k < m; ++k) w[k] = 0.5 + 0.25 * static_cast<double>(k % 7);
  const auto res = sweep.apply_pairs(w);
  const auto nrm = sweep.boundary_normals();
  const std::array<double, 3> one{1.0, 1.0, 1.0};
  for (std::size_t i = 0; i < s.particles.size(); ++i) {
    double v = 0, gx = 0, gy = 0, nx = 0, ny = 0;
    for (std::size_t t = 0; t < s.mesh.size(); ++t) {
      const std::size_t k = i * s.mesh.size() + t;
      const auto r = sphbi::integrate_triangle(s.particles[i], h, s.mesh[t], one, table);
      v += w[k] * r.value;
      gx += w[k] * r.gradient[0];
      gy += w[k] * r.gradient[1];
      nx += r.gradient[0];
      ny += r.gradient[1];
    }
    const double sc = 2.0;  // max |w|
    EXPECT_LE(std::abs(res[i].value - v), sc * tol(res[i].value, v, table.normalization, h));
    EXPECT_LE(std::abs(res[i].gradient[0] - gx), sc * tol(res[i].gradient[0], gx, table.normalization, h));
    EXPECT_LE(std::abs(res[i].gradient[1] - gy), sc * tol(res[i].gradient[1], gy, table.normalization, h));
    const double mag = std::hypot(nx, ny);
    if (mag > 1e-6) {
      EXPECT_NEAR(nrm[i].x, -nx / mag, 1e-10);
      EXPECT_NEAR(nrm[i].y, -ny / mag, 1e-10);
    } else if (mag <= 1e-12) {
      EXPECT_EQ(nrm[i].x, 0.0);
      EXPECT_EQ(nrm[i].y, 0.0);
    }
  }
}
