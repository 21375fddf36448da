// host_gen.cpp -- seeded host-side generators of the synthetic workload
// (BASELINE.json configs): Arrhenius mechanism, random-phase velocity field,
// initial condition.  Counter-based / splitmix64 streams so any slab of the
// grid reproduces the global field; no std::*_distribution (implementation
// defined).  Compiled with -ffp-contract=off; tests check these are bit-equal
// to the oracle's generators (tests/test_generators.py).
//
// Replaces initial_condition (proj/src/models.cpp:220-250) for the 3D
// reacting-flow workload; the reference has no mechanism generator.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/mri_b200.h"

namespace {

constexpr double kRu = 8.31446261815324e7;     // erg/(mol K)
constexpr double kRc = 1.98720425864083;       // cal/(mol K)
constexpr double kLn1e8 = 18.420680743952367;  // ln(1e8)
constexpr double kLnSpan = 13.815510557964274; // ln(1e14) - ln(1e8)
constexpr double kLn1400 = 7.2442275156033498;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

inline uint64_t mix64(uint64_t z)
{
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

struct SplitMix {
  uint64_t s;
  uint64_t next() { s += kGolden; return mix64(s); }
  double u01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double a, double b) { return a + (b - a) * u01(); }
};

}  // namespace

extern "C" int mr_mechanism_generate(uint64_t seed, int S, int R, double* species,
                                     double* reactions, int* rspecies)
{
  if (S < 4 || R < 1 || !species || !reactions || !rspecies) return MR_CONTRACT;
  SplitMix rng{seed};
  for (int k = 0; k < S; ++k) {
    double* sp = species + 5 * k;
    sp[0] = rng.uniform(2.0, 50.0);         // W  [g/mol]
    sp[1] = rng.uniform(3.4, 3.6);          // a  cp/R constant part
    sp[2] = rng.uniform(0.0, 2.0e-4);       // b  cp/R slope [1/K]
    sp[3] = rng.uniform(-2000.0, 2000.0);   // h0 / R [K]
    // s0 centres g/RT on zero at T_ref = 1400 K
    sp[4] = sp[3] / 1400.0 + sp[1] * (1.0 - kLn1400) + rng.uniform(-1.0, 1.0);
  }
  for (int j = 0; j < R; ++j) {
    reactions[3 * j + 0] = kLn1e8 + kLnSpan * rng.u01();          // ln A, A log-uniform [1e8,1e14]
    reactions[3 * j + 1] = rng.uniform(-1.0, 1.0);                 // beta
    reactions[3 * j + 2] = rng.uniform(0.0, 30000.0) / kRc;       // Ea / Rc [K]
    const int nr = 1 + static_cast<int>(rng.next() % 2u);
    const int np = 1 + static_cast<int>(rng.next() % 2u);
    int picked[4] = {-1, -1, -1, -1};
    int n = 0;
    while (n < nr + np) {
      const int k = static_cast<int>(rng.next() % static_cast<uint64_t>(S));
      bool dup = false;
      for (int q = 0; q < n; ++q) dup |= picked[q] == k;
      if (!dup) picked[n++] = k;
    }
    rspecies[4 * j + 0] = picked[0];
    rspecies[4 * j + 1] = nr == 2 ? picked[1] : -1;
    rspecies[4 * j + 2] = picked[nr];
    rspecies[4 * j + 3] = np == 2 ? picked[nr + 1] : -1;
  }
  return MR_OK;
}

extern "C" int mr_velocity_profiles(uint64_t seed, int n0, int n1, int n2, double length,
                                    double* prof)
{
  (void)length;
  if (n0 < 1 || n1 < 1 || n2 < 1 || !prof) return MR_CONTRACT;
  const int n[3] = {n0, n1, n2};
  const int nmax = std::max(n0, std::max(n1, n2));
  std::memset(prof, 0, sizeof(double) * 6 * static_cast<size_t>(nmax));
  SplitMix rng{seed};
  const double two_pi = 6.283185307179586;
  for (int d = 0; d < 3; ++d) {
    const int axes[2] = {d == 0 ? 1 : 0, d == 2 ? 1 : 2};
    for (int mode = 0; mode < 3; ++mode) {
      const int slot = static_cast<int>(rng.next() % 2u);
      const int kappa = 1 + static_cast<int>(rng.next() % 3u);
      const double phi = two_pi * rng.u01();
      const int ax = axes[slot];
      double* P = prof + (static_cast<size_t>(d) * 2 + slot) * nmax;
      for (int i = 0; i < n[ax]; ++i)
        P[i] += (1.0 / 3.0) * std::sin(two_pi * kappa * ((i + 0.5) / n[ax]) + phi);
    }
  }
  return MR_OK;
}

extern "C" int mr_initial_condition(uint64_t seed, int S, double rho, const double* species,
                                    int n0, int n1, int n2, double length, int i0, int n0_local,
                                    double* Y, int threads)
{
  (void)rho;
  if (S < 1 || !species || !Y || n0_local < 1 || i0 < 0 || i0 + n0_local > n0) return MR_CONTRACT;
  std::vector<double> c0(S), c1(S), c2(S);
  for (int k = 0; k < S; ++k) {
    const double W = species[5 * k], a = species[5 * k + 1], b = species[5 * k + 2];
    const double rW = kRu / W;
    c0[k] = rW * species[5 * k + 3];
    c1[k] = rW * (a - 1.0);
    c2[k] = rW * (0.5 * b);
  }
  const size_t ncell = static_cast<size_t>(n0_local) * n1 * n2;
  const int ng[3] = {n0, n1, n2};
  const double sig = 0.1 * length;
  auto work = [&](int plo, int phi) {
    std::vector<double> E(S);
    for (int i = plo; i < phi; ++i)
      for (int j = 0; j < n1; ++j)
        for (int k = 0; k < n2; ++k) {
          const size_t cell = (static_cast<size_t>(i) * n1 + j) * n2 + k;
          const uint64_t gcell = (static_cast<uint64_t>(i0 + i) * n1 + j) * n2 + k;
          double sum = 0.0;
          for (int s = 0; s < S; ++s) {
            const uint64_t key = gcell * static_cast<uint64_t>(S) + static_cast<uint64_t>(s);
            const uint64_t h = mix64(seed + (key + 1) * kGolden);
            const double u = static_cast<double>((h >> 11) + 1) * 0x1.0p-53;
            E[s] = -std::log(u);
            sum += E[s];
          }
          for (int s = 0; s < S; ++s) Y[static_cast<size_t>(s) * ncell + cell] = E[s] / sum;
          const int co[3] = {i0 + i, j, k};
          double r2 = 0.0;
          for (int d = 0; d < 3; ++d) {
            const double x = (co[d] + 0.5) * (length / ng[d]) - 0.5 * length;
            r2 += x * x;
          }
          const double T = 800.0 + 1200.0 * std::exp(-r2 / (2.0 * sig * sig));
          double E0 = 0.0, E1 = 0.0, E2 = 0.0;
          for (int s = 0; s < S; ++s) {
            const double y = Y[static_cast<size_t>(s) * ncell + cell];
            E0 += y * c0[s];
            E1 += y * c1[s];
            E2 += y * c2[s];
          }
          Y[static_cast<size_t>(S) * ncell + cell] = (E2 * T + E1) * T + E0;
        }
  };
  int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  if (nt < 1) nt = 1;
  if (nt > n0_local) nt = n0_local;
  if (nt == 1) {
    work(0, n0_local);
  } else {
    std::vector<std::thread> pool;
    const int chunk = (n0_local + nt - 1) / nt;
    for (int t = 0; t < nt; ++t) {
      const int lo = t * chunk, hi = std::min(n0_local, lo + chunk);
      if (lo >= hi) break;
      pool.emplace_back(work, lo, hi);
    }
    for (auto& th : pool) th.join();
  }
  return MR_OK;
}
