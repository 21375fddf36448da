/*
 * oracle/mri_oracle.c -- CPU ORACLE (test infrastructure only; see header).
 *
 * Plain-C restatement of the reference's explicit MRI slow step plus the
 * builder-defined physics.  Build with -ffp-contract=off (oracle/Makefile) so
 * the stepper arithmetic is bit-identical to the reference's C++ (no FMA
 * contraction on either side).  Never linked into the product.
 */
#include "mri_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* RNG: splitmix64 (portable; no std::*_distribution)                  */
/* ------------------------------------------------------------------ */
uint64_t orc_mix64(uint64_t z)
{
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t orc_splitmix64_next(uint64_t* state)
{
  *state += 0x9E3779B97F4A7C15ULL;
  return orc_mix64(*state);
}

static double u01(uint64_t* st) { return (double)(orc_splitmix64_next(st) >> 11) * 0x1.0p-53; }
static double uniform(uint64_t* st, double a, double b) { return a + (b - a) * u01(st); }

/* ------------------------------------------------------------------ */
/* tiny pthread parallel-for (used only to time the oracle on all cores) */
/* ------------------------------------------------------------------ */
typedef void (*range_fn)(void* ctx, size_t lo, size_t hi);
typedef struct { range_fn fn; void* ctx; size_t lo, hi; } range_job;
static void* range_thread(void* p)
{
  range_job* j = (range_job*)p;
  j->fn(j->ctx, j->lo, j->hi);
  return NULL;
}
static void parallel_for(size_t n, int threads, range_fn fn, void* ctx)
{
  if (threads <= 1 || n < 1024) { fn(ctx, 0, n); return; }
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  range_job jobs[256];
  size_t chunk = (n + (size_t)threads - 1) / (size_t)threads;
  int used = 0;
  for (int t = 0; t < threads; ++t) {
    size_t lo = (size_t)t * chunk, hi = lo + chunk;
    if (lo >= n) break;
    if (hi > n) hi = n;
    jobs[t].fn = fn; jobs[t].ctx = ctx; jobs[t].lo = lo; jobs[t].hi = hi;
    pthread_create(&tid[t], NULL, range_thread, &jobs[t]);
    ++used;
  }
  for (int t = 0; t < used; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------ */
/* Vector contract: proj/include/multirate/state_vector.hpp            */
/* ------------------------------------------------------------------ */
/* wrms_norm, state_vector.hpp:119-129 */
double orc_wrms_norm(const double* x, const double* w, size_t n)
{
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double xw = x[i] * w[i];
    sum += xw * xw;
  }
  return sqrt(sum / (double)n);
}
/* two_norm, state_vector.hpp:131-136 */
double orc_two_norm(const double* x, size_t n)
{
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) sum += x[i] * x[i];
  return sqrt(sum);
}
/* dot, state_vector.hpp:138-144 */
double orc_dot(const double* x, const double* y, size_t n)
{
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) sum += x[i] * y[i];
  return sum;
}
/* max_norm, state_vector.hpp:146-152 (std::max(m, |v|) keeps m on NaN) */
double orc_max_norm(const double* x, size_t n)
{
  double m = 0.0;
  for (size_t i = 0; i < n; ++i) { double a = fabs(x[i]); m = (m < a) ? a : m; }
  return m;
}
/* max_norm_component, state_vector.hpp:157-168 */
double orc_max_norm_component(const double* x, size_t offset, size_t count)
{
  return orc_max_norm(x + offset, count);
}
/* all_finite, state_vector.hpp:170-176 */
int orc_all_finite(const double* x, size_t n)
{
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return 0;
  return 1;
}
/* axpy_into, state_vector.hpp:104-108 */
static void axpy_into(double* y, double a, const double* x, size_t n)
{
  for (size_t i = 0; i < n; ++i) y[i] += a * x[i];
}

/* ------------------------------------------------------------------ */
/* Butcher tables: proj/src/butcher.cpp:229-362 (textbook data)       */
/* ------------------------------------------------------------------ */
static void table_zero(orc_table* t, int s, int order)
{
  memset(t, 0, sizeof(*t));
  t->s = s; t->order = order; t->is_explicit = 1;
}

int orc_table_lookup(const char* name, orc_table* t)
{
  if (!strcmp(name, "heun2")) { /* butcher.cpp:229-240 */
    table_zero(t, 2, 2);
    t->A[1][0] = 1; t->b[0] = 0.5; t->b[1] = 0.5; t->c[1] = 1;
  } else if (!strcmp(name, "kutta3")) { /* butcher.cpp:242-253 */
    table_zero(t, 3, 3);
    t->A[1][0] = 0.5; t->A[2][0] = -1; t->A[2][1] = 2;
    t->b[0] = 1.0 / 6.0; t->b[1] = 2.0 / 3.0; t->b[2] = 1.0 / 6.0;
    t->c[1] = 0.5; t->c[2] = 1;
  } else if (!strcmp(name, "bogacki-shampine3")) { /* butcher.cpp:258-269 */
    table_zero(t, 3, 3);
    t->A[1][0] = 0.5; t->A[2][1] = 0.75;
    t->b[0] = 2.0 / 9.0; t->b[1] = 1.0 / 3.0; t->b[2] = 4.0 / 9.0;
    t->c[1] = 0.5; t->c[2] = 0.75;
  } else if (!strcmp(name, "zonneveld4")) { /* butcher.cpp:274-289 */
    table_zero(t, 5, 4);
    t->A[1][0] = 0.5; t->A[2][1] = 0.5; t->A[3][2] = 1;
    t->A[4][0] = 5.0 / 32.0; t->A[4][1] = 7.0 / 32.0; t->A[4][2] = 13.0 / 32.0;
    t->A[4][3] = -1.0 / 32.0;
    t->b[0] = 1.0 / 6.0; t->b[1] = 1.0 / 3.0; t->b[2] = 1.0 / 3.0; t->b[3] = 1.0 / 6.0;
    t->c[1] = 0.5; t->c[2] = 0.5; t->c[3] = 1; t->c[4] = 0.75;
  } else if (!strcmp(name, "classic-rk4")) { /* butcher.cpp:291-302 */
    table_zero(t, 4, 4);
    t->A[1][0] = 0.5; t->A[2][1] = 0.5; t->A[3][2] = 1;
    t->b[0] = 1.0 / 6.0; t->b[1] = 1.0 / 3.0; t->b[2] = 1.0 / 3.0; t->b[3] = 1.0 / 6.0;
    t->c[1] = 0.5; t->c[2] = 0.5; t->c[3] = 1;
  } else if (!strcmp(name, "cash-karp5")) { /* butcher.cpp:305-321 */
    table_zero(t, 6, 5);
    t->A[1][0] = 1.0 / 5.0;
    t->A[2][0] = 3.0 / 40.0; t->A[2][1] = 9.0 / 40.0;
    t->A[3][0] = 3.0 / 10.0; t->A[3][1] = -9.0 / 10.0; t->A[3][2] = 6.0 / 5.0;
    t->A[4][0] = -11.0 / 54.0; t->A[4][1] = 5.0 / 2.0; t->A[4][2] = -70.0 / 27.0;
    t->A[4][3] = 35.0 / 27.0;
    t->A[5][0] = 1631.0 / 55296.0; t->A[5][1] = 175.0 / 512.0; t->A[5][2] = 575.0 / 13824.0;
    t->A[5][3] = 44275.0 / 110592.0; t->A[5][4] = 253.0 / 4096.0;
    t->b[0] = 37.0 / 378.0; t->b[2] = 250.0 / 621.0; t->b[3] = 125.0 / 594.0;
    t->b[5] = 512.0 / 1771.0;
    t->c[1] = 1.0 / 5.0; t->c[2] = 3.0 / 10.0; t->c[3] = 3.0 / 5.0; t->c[4] = 1; t->c[5] = 7.0 / 8.0;
  } else if (!strcmp(name, "knoth-wolke3")) { /* butcher.cpp:347-362 */
    table_zero(t, 3, 3);
    t->A[1][0] = 1.0 / 3.0; t->A[2][0] = -3.0 / 16.0; t->A[2][1] = 15.0 / 16.0;
    t->b[0] = 1.0 / 6.0; t->b[1] = 3.0 / 10.0; t->b[2] = 8.0 / 15.0;
    t->c[1] = 1.0 / 3.0; t->c[2] = 3.0 / 4.0;
  } else {
    return ORC_CONTRACT;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* MriCoupling::finalize, proj/src/mri.cpp:59-167                     */
/* ------------------------------------------------------------------ */
#define CONSISTENCY_TOL 1.0e-12 /* mri.cpp:14 */

static int any_nonzero(const double m[ORC_MAX_DEG][ORC_MAX_STAGES][ORC_MAX_STAGES], int nd, int s)
{
  for (int k = 0; k < nd; ++k)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j)
        if (m[k][i][j] != 0.0) return 1;
  return 0;
}

static int fail(char* err, size_t n, const char* msg, const char* name, int stage)
{
  if (err && n) {
    if (stage >= 0) snprintf(err, n, "MriCoupling %s: %s %d", name, msg, stage);
    else snprintf(err, n, "MriCoupling %s: %s", name, msg);
  }
  return ORC_CONTRACT;
}

int orc_coupling_finalize(orc_coupling* cp, char* err, size_t errlen)
{
  const int s = cp->s;
  if (s < 2 || s > ORC_MAX_STAGES) return fail(err, errlen, "inconsistent sizes", cp->name, -1);
  if (fabs(cp->c[0]) > 0.0 || fabs(cp->c[s - 1] - 1.0) > CONSISTENCY_TOL)
    return fail(err, errlen, "need c[0]=0 and c[s-1]=1", cp->name, -1);
  for (int i = 1; i < s; ++i)
    if (cp->c[i] < cp->c[i - 1] - CONSISTENCY_TOL)
      return fail(err, errlen, "abscissae decrease", cp->name, -1);
  /* check_shape, mri.cpp:77-99 */
  for (int pass = 0; pass < 2; ++pass) {
    const int nd = pass == 0 ? cp->ndeg_gamma : cp->ndeg_omega;
    for (int k = 0; k < nd; ++k)
      for (int i = 0; i < s; ++i)
        for (int j = i; j < s; ++j) {
          const double v = pass == 0 ? cp->gamma[k][i][j] : cp->omega[k][i][j];
          const int diag_ok = pass == 0 && j == i && cp->kind[i] == ORC_IMPLICIT_SOLVE;
          if (v != 0.0 && !diag_ok)
            return fail(err, errlen, pass == 0 ? "gamma not lower triangular at stage"
                                               : "omega not lower triangular at stage",
                        cp->name, i);
        }
  }
  /* average_matrices, mri.cpp:34-44 */
  memset(cp->gbar, 0, sizeof(cp->gbar));
  memset(cp->wbar, 0, sizeof(cp->wbar));
  for (int k = 0; k < cp->ndeg_gamma; ++k) {
    const double w = 1.0 / (double)(k + 1);
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) cp->gbar[i][j] += w * cp->gamma[k][i][j];
  }
  for (int k = 0; k < cp->ndeg_omega; ++k) {
    const double w = 1.0 / (double)(k + 1);
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < s; ++j) cp->wbar[i][j] += w * cp->omega[k][i][j];
  }
  const int has_gamma = any_nonzero(cp->gamma, cp->ndeg_gamma, s);
  const int has_omega = any_nonzero(cp->omega, cp->ndeg_omega, s);

  for (int i = 1; i < s; ++i) {
    const double dc = cp->c[i] - cp->c[i - 1];
    if (cp->kind[i] == ORC_FAST_IVP) {
      if (dc <= 0.0) return fail(err, errlen, "fast-ivp stage has dc <= 0 at", cp->name, i);
    } else {
      if (dc > CONSISTENCY_TOL) return fail(err, errlen, "solves/updates with dc > 0 at", cp->name, i);
      if (cp->kind[i] == ORC_IMPLICIT_SOLVE && cp->gbar[i][i] == 0.0)
        return fail(err, errlen, "implicit stage has zero diagonal at", cp->name, i);
    }
    /* check_rows, mri.cpp:131-150 */
    for (int pass = 0; pass < 2; ++pass) {
      const int used = pass == 0 ? has_gamma : has_omega;
      if (!used) continue;
      const int nd = pass == 0 ? cp->ndeg_gamma : cp->ndeg_omega;
      double bar_sum = 0.0;
      for (int k = 0; k < nd; ++k) {
        double rk = 0.0;
        for (int j = 0; j < s; ++j) rk += pass == 0 ? cp->gamma[k][i][j] : cp->omega[k][i][j];
        bar_sum += rk / (double)(k + 1);
        if (k >= 1 && fabs(rk) > CONSISTENCY_TOL)
          return fail(err, errlen, "higher-degree row sum nonzero at stage", cp->name, i);
      }
      if (fabs(bar_sum - dc) > CONSISTENCY_TOL)
        return fail(err, errlen, "row integral != dc at stage", cp->name, i);
    }
  }
  int fE_ref[ORC_MAX_STAGES] = {0};
  for (int i = 0; i < s; ++i) cp->fI_referenced[i] = 0;
  for (int k = 0; k < cp->ndeg_gamma; ++k)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < i; ++j)
        if (cp->gamma[k][i][j] != 0.0) cp->fI_referenced[j] = 1;
  for (int k = 0; k < cp->ndeg_omega; ++k)
    for (int i = 0; i < s; ++i)
      for (int j = 0; j < i; ++j)
        if (cp->omega[k][i][j] != 0.0) fE_ref[j] = 1;
  for (int i = 0; i < s; ++i) cp->eval_explicit_at[i] = fE_ref[i];
  if (!has_gamma && has_omega) cp->eval_explicit_at[s - 1] = 1; /* mri.cpp:162-166 */
  return ORC_OK;
}

/* coupling_from_mis, proj/src/mri.cpp:203-264 */
int orc_coupling_from_mis(const char* name, const orc_table* base, int order,
                          int split_widest, orc_coupling* out)
{
  const int sb = base->s;
  orc_coupling cp;
  memset(&cp, 0, sizeof(cp));
  snprintf(cp.name, sizeof(cp.name), "%s", name);
  cp.order = order;
  cp.s = sb + 1;
  for (int i = 0; i < sb; ++i) cp.c[i] = base->c[i];
  cp.c[sb] = 1.0;
  for (int i = 0; i < cp.s; ++i) cp.kind[i] = ORC_FAST_IVP;
  cp.kind[0] = ORC_EXPLICIT_UPDATE;
  cp.ndeg_omega = 1;
  cp.ndeg_gamma = 0;
  for (int i = 1; i < sb; ++i)
    for (int j = 0; j < sb; ++j) cp.omega[0][i][j] = base->A[i][j] - base->A[i - 1][j];
  for (int j = 0; j < sb; ++j) cp.omega[0][sb][j] = base->b[j] - base->A[sb - 1][j];

  if (split_widest) {
    int widest = 1;
    double width = 0.0;
    for (int i = 1; i < cp.s; ++i) {
      const double dc = cp.c[i] - cp.c[i - 1];
      if (dc > width) { width = dc; widest = i; }
    }
    const double mid = 0.5 * (cp.c[widest - 1] + cp.c[widest]);
    orc_coupling sp;
    memset(&sp, 0, sizeof(sp));
    snprintf(sp.name, sizeof(sp.name), "%s", name);
    sp.order = order;
    sp.s = cp.s + 1;
    for (int i = 0; i < sp.s; ++i) sp.kind[i] = ORC_FAST_IVP;
    sp.kind[0] = ORC_EXPLICIT_UPDATE;
    sp.ndeg_omega = 1;
    for (int i = 0; i < cp.s; ++i) {
      const int ti = (i < widest) ? i : i + 1;
      sp.c[ti] = cp.c[i];
      const double scale = (i == widest) ? 0.5 : 1.0;
      for (int j = 0; j < cp.s; ++j) {
        const int tj = (j < widest) ? j : j + 1;
        sp.omega[0][ti][tj] = scale * cp.omega[0][i][j];
        if (i == widest) sp.omega[0][ti - 1][tj] = scale * cp.omega[0][i][j];
      }
    }
    sp.c[widest] = mid;
    int rc = orc_coupling_finalize(&sp, NULL, 0);
    *out = sp;
    return rc;
  }
  int rc = orc_coupling_finalize(&cp, NULL, 0);
  *out = cp;
  return rc;
}

/* register_coupling("mis-kw3"), proj/src/mri_tables.cpp:222-229.  The two
 * IMEX couplings are fitted parameter sets; they are loaded from the
 * reference's own export_coupling audit files (tests/golden/couplings/,
 * regenerated by oracle/gen_golden.py) through orc_coupling_import. */
int orc_coupling_register(const char* name, orc_coupling* out)
{
  if (!strcmp(name, "mis-kw3")) {
    orc_table kw;
    orc_table_lookup("knoth-wolke3", &kw);
    return orc_coupling_from_mis("mis-kw3", &kw, 3, 1, out);
  }
  return ORC_CONTRACT;
}

/* import_coupling, proj/src/mri.cpp:590-626 (text v1 audit format) */
int orc_coupling_import(const char* text, orc_coupling* out, char* err, size_t errlen)
{
  orc_coupling cp;
  memset(&cp, 0, sizeof(cp));
  char magic[64], version[16], name[64], sfield[32], dfield[32];
  int consumed = 0;
  if (sscanf(text, "%63s %15s %63s %31s %31s%n", magic, version, name, sfield, dfield, &consumed) != 5 ||
      strcmp(magic, "mri-coupling") || strcmp(version, "v1") || strncmp(sfield, "s=", 2) ||
      strncmp(dfield, "degrees=", 8)) {
    if (err) snprintf(err, errlen, "import_coupling: bad header");
    return ORC_CONTRACT;
  }
  snprintf(cp.name, sizeof(cp.name), "%s", name);
  cp.s = atoi(sfield + 2);
  const int d = atoi(dfield + 8);
  if (cp.s < 2 || d < 1 || cp.s > ORC_MAX_STAGES || d > ORC_MAX_DEG) {
    if (err) snprintf(err, errlen, "import_coupling: bad dimensions");
    return ORC_CONTRACT;
  }
  const char* p = text + consumed;
  char* end;
  for (int i = 0; i < cp.s; ++i) {
    cp.c[i] = strtod(p, &end);
    if (end == p) goto truncated;
    p = end;
  }
  for (int i = 0; i < cp.s; ++i) {
    char tok[32];
    int n = 0;
    if (sscanf(p, "%31s%n", tok, &n) != 1) goto truncated;
    p += n;
    if (!strcmp(tok, "fast-ivp")) cp.kind[i] = ORC_FAST_IVP;
    else if (!strcmp(tok, "implicit-solve")) cp.kind[i] = ORC_IMPLICIT_SOLVE;
    else if (!strcmp(tok, "explicit-update")) cp.kind[i] = ORC_EXPLICIT_UPDATE;
    else {
      if (err) snprintf(err, errlen, "import_coupling: unknown stage kind '%s'", tok);
      return ORC_CONTRACT;
    }
  }
  cp.ndeg_gamma = cp.ndeg_omega = d;
  for (int pass = 0; pass < 2; ++pass)
    for (int k = 0; k < d; ++k)
      for (int i = 0; i < cp.s; ++i)
        for (int j = 0; j < cp.s; ++j) {
          double v = strtod(p, &end);
          if (end == p) goto truncated;
          p = end;
          if (pass == 0) cp.gamma[k][i][j] = v; else cp.omega[k][i][j] = v;
        }
  cp.order = 0;
  {
    int rc = orc_coupling_finalize(&cp, err, errlen);
    *out = cp;
    return rc;
  }
truncated:
  if (err) snprintf(err, errlen, "import_coupling: truncated input");
  return ORC_CONTRACT;
}

/* export_coupling, proj/src/mri.cpp:560-588 (precision 17 == %.17g) */
int orc_coupling_export(const orc_coupling* cp, char* buf, size_t buflen)
{
  static const char* tok[3] = {"fast-ivp", "implicit-solve", "explicit-update"};
  const int d = cp->ndeg_gamma > cp->ndeg_omega ? cp->ndeg_gamma : cp->ndeg_omega;
  size_t off = 0;
#define EMIT(...) do { int w_ = snprintf(buf + off, off < buflen ? buflen - off : 0, __VA_ARGS__); off += (size_t)w_; } while (0)
  EMIT("mri-coupling v1 %s s=%d degrees=%d\n", cp->name, cp->s, d);
  for (int i = 0; i < cp->s; ++i) EMIT("%s%.17g", i ? " " : "", cp->c[i]);
  EMIT("\n");
  for (int i = 0; i < cp->s; ++i) EMIT("%s%s", i ? " " : "", tok[cp->kind[i]]);
  EMIT("\n");
  for (int pass = 0; pass < 2; ++pass)
    for (int k = 0; k < d; ++k)
      for (int i = 0; i < cp->s; ++i) {
        for (int j = 0; j < cp->s; ++j) {
          double v = 0.0;
          if (pass == 0 && k < cp->ndeg_gamma) v = cp->gamma[k][i][j];
          if (pass == 1 && k < cp->ndeg_omega) v = cp->omega[k][i][j];
          EMIT("%s%.17g", j ? " " : "", v);
        }
        EMIT("\n");
      }
#undef EMIT
  return (int)off;
}

/* ------------------------------------------------------------------ */
/* Physics: synthetic Arrhenius mechanism (builder-defined)  */
/* ------------------------------------------------------------------ */
#define R_U 8.31446261815324e7     /* erg/(mol K) */
#define R_C 1.98720425864083       /* cal/(mol K) */
#define P_ATM 1.01325e6            /* dyn/cm^2 */
#define LN_1E8 18.420680743952367  /* ln(1e8)  */
#define LN_SPAN 13.815510557964274 /* ln(1e14) - ln(1e8) */

int orc_mech_generate(uint64_t seed, int S, int R, double* species, double* reactions,
                      int* rspecies)
{
  if (S < 4 || R < 1) return ORC_CONTRACT;
  uint64_t st = seed;
  for (int k = 0; k < S; ++k) {
    species[5 * k + 0] = uniform(&st, 2.0, 50.0);      /* W   [g/mol]      */
    species[5 * k + 1] = uniform(&st, 3.4, 3.6);       /* a   cp/R const   */
    species[5 * k + 2] = uniform(&st, 0.0, 2.0e-4);    /* b   cp/R slope   */
    species[5 * k + 3] = uniform(&st, -2000.0, 2000.0);/* h0  [K]          */
    /* s0 centres g/RT on zero at T_ref = 1400 K (synthetic thermo without the
     * standard-state offset, so Kc stays O(e^{+-few}) times (RT/P)^dnu) */
    species[5 * k + 4] = species[5 * k + 3] / 1400.0 +
                         species[5 * k + 1] * (1.0 - 7.2442275156033498) +
                         uniform(&st, -1.0, 1.0);     /* s0; 7.2442... = ln(1400) */
  }
  for (int j = 0; j < R; ++j) {
    reactions[3 * j + 0] = LN_1E8 + LN_SPAN * u01(&st);         /* ln A, A log-uniform */
    reactions[3 * j + 1] = uniform(&st, -1.0, 1.0);             /* beta */
    reactions[3 * j + 2] = uniform(&st, 0.0, 30000.0) / R_C;    /* Ea/Rc [K] */
    const int nr = 1 + (int)(orc_splitmix64_next(&st) % 2u);
    const int np = 1 + (int)(orc_splitmix64_next(&st) % 2u);
    int picked[4] = {-1, -1, -1, -1};
    int n = 0;
    while (n < nr + np) {
      const int k = (int)(orc_splitmix64_next(&st) % (uint64_t)S);
      int dup = 0;
      for (int q = 0; q < n; ++q) dup |= picked[q] == k;
      if (!dup) picked[n++] = k;
    }
    rspecies[4 * j + 0] = picked[0];
    rspecies[4 * j + 1] = nr == 2 ? picked[1] : -1;
    rspecies[4 * j + 2] = picked[nr];
    rspecies[4 * j + 3] = np == 2 ? picked[nr + 1] : -1;
  }
  return ORC_OK;
}

int orc_mech_init(orc_mech* m, int S, int R, double rho, const double* species,
                  const double* reactions, const int* rspecies)
{
  memset(m, 0, sizeof(*m));
  m->S = S; m->R = R; m->rho = rho;
  m->species = (double*)malloc(sizeof(double) * 5 * S);
  m->reactions = (double*)malloc(sizeof(double) * 3 * R);
  m->rspecies = (int*)malloc(sizeof(int) * 4 * R);
  memcpy(m->species, species, sizeof(double) * 5 * S);
  memcpy(m->reactions, reactions, sizeof(double) * 3 * R);
  memcpy(m->rspecies, rspecies, sizeof(int) * 4 * R);
  m->rhoW = (double*)malloc(sizeof(double) * S);
  m->Wrho = (double*)malloc(sizeof(double) * S);
  m->c0 = (double*)malloc(sizeof(double) * S);
  m->c1 = (double*)malloc(sizeof(double) * S);
  m->c2 = (double*)malloc(sizeof(double) * S);
  m->hb = (double*)malloc(sizeof(double) * S);
  m->dnu = (int*)malloc(sizeof(int) * R);
  for (int k = 0; k < S; ++k) {
    const double W = species[5 * k], a = species[5 * k + 1], b = species[5 * k + 2];
    const double h0 = species[5 * k + 3];
    const double rW = R_U / W;
    m->rhoW[k] = rho / W;
    m->Wrho[k] = W / rho;
    m->c0[k] = rW * h0;
    m->c1[k] = rW * (a - 1.0);
    m->c2[k] = rW * (0.5 * b);
    m->hb[k] = 0.5 * b;
  }
  for (int j = 0; j < R; ++j) {
    for (int q = 0; q < 4; ++q)
      if (rspecies[4 * j + q] >= S) return ORC_CONTRACT;
    const int nr = 1 + (rspecies[4 * j + 1] >= 0);
    const int np = 1 + (rspecies[4 * j + 3] >= 0);
    m->dnu[j] = np - nr;
  }
  /* species <- reaction incidence, reaction index ascending */
  m->csr_off = (int*)calloc((size_t)S + 1, sizeof(int));
  for (int j = 0; j < R; ++j)
    for (int q = 0; q < 4; ++q)
      if (rspecies[4 * j + q] >= 0) m->csr_off[rspecies[4 * j + q] + 1]++;
  for (int k = 0; k < S; ++k) m->csr_off[k + 1] += m->csr_off[k];
  const int nnz = m->csr_off[S];
  m->csr_rxn = (int*)malloc(sizeof(int) * (nnz ? nnz : 1));
  m->csr_sgn = (int*)malloc(sizeof(int) * (nnz ? nnz : 1));
  int* fill = (int*)calloc((size_t)S, sizeof(int));
  for (int j = 0; j < R; ++j)
    for (int q = 0; q < 4; ++q) {
      const int k = rspecies[4 * j + q];
      if (k < 0) continue;
      const int pos = m->csr_off[k] + fill[k]++;
      m->csr_rxn[pos] = j;
      m->csr_sgn[pos] = q < 2 ? -1 : +1;
    }
  free(fill);
  return ORC_OK;
}

void orc_mech_free(orc_mech* m)
{
  free(m->species); free(m->reactions); free(m->rspecies);
  free(m->rhoW); free(m->Wrho); free(m->c0); free(m->c1); free(m->c2); free(m->hb);
  free(m->dnu); free(m->csr_off); free(m->csr_rxn); free(m->csr_sgn);
  memset(m, 0, sizeof(*m));
}

/* Temperature from energy: e(T) = E0 + E1 T + E2 T^2 solved in closed form
 * (E2 >= 0, E1 > 0 root), v = per-cell state with the given stride. */
double orc_temperature(const orc_mech* m, const double* v, size_t stride)
{
  const int S = m->S;
  double E0 = 0.0, E1 = 0.0, E2 = 0.0;
  for (int k = 0; k < S; ++k) {
    const double y = v[(size_t)k * stride];
    E0 += y * m->c0[k];
    E1 += y * m->c1[k];
    E2 += y * m->c2[k];
  }
  const double de = v[(size_t)S * stride] - E0;
  return (2.0 * de) / (E1 + sqrt(E1 * E1 + 4.0 * E2 * de));
}

/* One cell of the chemistry RHS.  v/out strided by `stride` (species-major).
 *   C_k  = rho Y_k / W_k,   E_k = exp(g_k/RT)
 *   Dp_k = (E_k C_k) (RT/P),   Ei_k = (1/E_k) (P/RT)   (absent slot: 1, 1, 1)
 *   kf_j = exp(lnA + beta lnT - Ea/(Rc T))
 *   q_j  = kf_j (C_r1 C_r2 - (Dp_p1 Dp_p2)(Ei_r1 Ei_r2))
 * i.e. kr = kf / Kc, Kc = exp(-dG/RT) (P/RT)^dnu: each present product
 * contributes RT/P and each present reactant P/RT, so (RT/P)^dnu needs no
 * per-reaction logic. */
static void chem_cell(const orc_mech* m, const double* v, double* out, size_t stride,
                      double* D, double* Ei, double* C, double* q)
{
  const int S = m->S, R = m->R;
  const double T = orc_temperature(m, v, stride);
  const double lnT = log(T);
  const double invT = 1.0 / T;
  const double RTP = (R_U / P_ATM) * T;
  const double iRTP = 1.0 / RTP;
  for (int k = 0; k < S; ++k) {
    const double* sp = m->species + 5 * k;
    const double g = sp[3] * invT + sp[1] * (1.0 - lnT) - m->hb[k] * T - sp[4];
    const double E = exp(g);
    C[k] = m->rhoW[k] * v[(size_t)k * stride];
    Ei[k] = (1.0 / E) * iRTP;
    D[k] = (E * C[k]) * RTP;
  }
  D[S] = 1.0; Ei[S] = 1.0; C[S] = 1.0; /* absent-slot dummy */
  for (int j = 0; j < R; ++j) {
    const double* rp = m->reactions + 3 * j;
    const int* rs = m->rspecies + 4 * j;
    const int r1 = rs[0], r2 = rs[1] < 0 ? S : rs[1];
    const int p1 = rs[2], p2 = rs[3] < 0 ? S : rs[3];
    const double kf = exp(rp[0] + rp[1] * lnT - rp[2] * invT);
    const double fwd = C[r1] * C[r2];
    const double rev = (D[p1] * D[p2]) * (Ei[r1] * Ei[r2]);
    q[j] = kf * (fwd - rev);
  }
  /* production: w_k = sum over reactions producing k (ascending) minus the
   * sum over reactions consuming k (ascending), accumulated in that order */
  for (int k = 0; k < S; ++k) {
    double w = 0.0;
    for (int p = m->csr_off[k]; p < m->csr_off[k + 1]; ++p)
      if (m->csr_sgn[p] > 0) w = w + q[m->csr_rxn[p]];
    for (int p = m->csr_off[k]; p < m->csr_off[k + 1]; ++p)
      if (m->csr_sgn[p] < 0) w = w - q[m->csr_rxn[p]];
    out[(size_t)k * stride] = m->Wrho[k] * w;
  }
  out[(size_t)S * stride] = 0.0; /* constant-volume adiabatic: de/dt = 0 */
}

typedef struct { const orc_mech* m; size_t ncell; const double* Y; double* out; } chem_job;
static void chem_range(void* p, size_t lo, size_t hi)
{
  chem_job* j = (chem_job*)p;
  const int S = j->m->S, R = j->m->R;
  double* buf = (double*)malloc(sizeof(double) * (size_t)(3 * (S + 1) + R));
  double *E = buf, *Ei = buf + (S + 1), *C = buf + 2 * (S + 1), *q = buf + 3 * (S + 1);
  for (size_t c = lo; c < hi; ++c) chem_cell(j->m, j->Y + c, j->out + c, j->ncell, E, Ei, C, q);
  free(buf);
}

static void chem_rhs_threads(const orc_mech* m, size_t ncell, const double* Y, double* out, int threads)
{
  chem_job j = {m, ncell, Y, out};
  parallel_for(ncell, threads, chem_range, &j);
}

void orc_chem_rhs(const orc_mech* m, size_t ncell, const double* Y, double* out)
{
  chem_rhs_threads(m, ncell, Y, out, 1);
}

/* ------------------------------------------------------------------ */
/* Physics: 3D periodic centred advection-diffusion stencil             */
/* Extends rhs_advection/rhs_diffusion (proj/src/models.cpp:129-211) to */
/* 3D and orders 2/4/8; species-major layout as models.cpp:155-157.     */
/* ------------------------------------------------------------------ */
static int stencil_coeffs(int order, double* a /*[5]*/, double* b /*[5]*/)
{
  for (int i = 0; i < 5; ++i) { a[i] = 0.0; b[i] = 0.0; }
  if (order == 2) {
    a[1] = 1.0 / 2.0;
    b[0] = -2.0; b[1] = 1.0;
    return 1;
  }
  if (order == 4) {
    a[1] = 2.0 / 3.0; a[2] = -1.0 / 12.0;
    b[0] = -5.0 / 2.0; b[1] = 4.0 / 3.0; b[2] = -1.0 / 12.0;
    return 2;
  }
  if (order == 8) {
    a[1] = 4.0 / 5.0; a[2] = -1.0 / 5.0; a[3] = 4.0 / 105.0; a[4] = -1.0 / 280.0;
    b[0] = -205.0 / 72.0; b[1] = 8.0 / 5.0; b[2] = -1.0 / 5.0; b[3] = 8.0 / 315.0;
    b[4] = -1.0 / 560.0;
    return 4;
  }
  return 0;
}

typedef struct { const orc_grid* g; const double* Y; double* out; } sten_job;
static void sten_range(void* p, size_t lo, size_t hi)
{
  sten_job* jb = (sten_job*)p;
  const orc_grid* g = jb->g;
  double a[5], b[5];
  const int M = stencil_coeffs(g->order, a, b);
  const int n[3] = {g->n0, g->n1, g->n2};
  const size_t ncell = (size_t)g->n0 * g->n1 * g->n2;
  double inv_dx[3], inv_dx2[3];
  for (int d = 0; d < 3; ++d) {
    const double dx = g->length / n[d];
    inv_dx[d] = 1.0 / dx;
    inv_dx2[d] = 1.0 / (dx * dx);
  }
  const size_t strides[3] = {(size_t)g->n1 * g->n2, (size_t)g->n2, 1};
  /* lo..hi index (comp, cell) pairs */
  for (size_t idx = lo; idx < hi; ++idx) {
    const size_t comp = idx / ncell, cell = idx % ncell;
    const int co[3] = {(int)(cell / strides[0]), (int)((cell / strides[1]) % g->n1),
                       (int)(cell % g->n2)};
    const double* y = jb->Y + comp * ncell;
    double acc = 0.0;
    for (int d = 0; d < 3; ++d) {
      double u;
      if (g->vel_kind == 0) {
        u = g->u_const[d];
      } else {
        const int a0 = d == 0 ? 1 : 0, a1 = d == 2 ? 1 : 2;
        u = g->prof[d][0][co[a0]] + g->prof[d][1][co[a1]];
      }
      const size_t base = cell - (size_t)co[d] * strides[d];
      double adv = 0.0;
      double dif = b[0] * y[cell];
      for (int m = 1; m <= M; ++m) {
        const double yp = y[base + (size_t)((co[d] + m) % n[d]) * strides[d]];
        const double ym = y[base + (size_t)((co[d] - m + n[d]) % n[d]) * strides[d]];
        adv += a[m] * (yp - ym);
        dif += b[m] * (yp + ym);
      }
      acc += g->diffusion * inv_dx2[d] * dif - u * inv_dx[d] * adv;
    }
    jb->out[comp * ncell + cell] = acc;
  }
}

static void stencil_threads(const orc_grid* g, const double* Y, double* out, int threads)
{
  sten_job j = {g, Y, out};
  parallel_for((size_t)g->ncomp * g->n0 * g->n1 * g->n2, threads, sten_range, &j);
}

void orc_stencil_rhs(const orc_grid* g, const double* Y, double* out) { stencil_threads(g, Y, out, 1); }

/* Random-phase velocity field, 3 Fourier modes per component, amplitude 1.
 * u_d depends only on the two axes != d (divergence-free); tabulated as two
 * 1-D profiles per component. prof layout [d][slot][nmax]. */
int orc_velocity_profiles(uint64_t seed, int n0, int n1, int n2, double length, double* prof)
{
  (void)length;
  const int n[3] = {n0, n1, n2};
  int nmax = n0 > n1 ? n0 : n1;
  nmax = nmax > n2 ? nmax : n2;
  memset(prof, 0, sizeof(double) * 6 * (size_t)nmax);
  uint64_t st = seed;
  const double two_pi = 6.283185307179586;
  for (int d = 0; d < 3; ++d) {
    const int axes[2] = {d == 0 ? 1 : 0, d == 2 ? 1 : 2};
    for (int mode = 0; mode < 3; ++mode) {
      const int slot = (int)(orc_splitmix64_next(&st) % 2u);
      const int kappa = 1 + (int)(orc_splitmix64_next(&st) % 3u);
      const double phi = two_pi * u01(&st);
      const int ax = axes[slot];
      double* P = prof + ((size_t)d * 2 + slot) * nmax;
      for (int i = 0; i < n[ax]; ++i)
        P[i] += (1.0 / 3.0) * sin(two_pi * kappa * ((i + 0.5) / n[ax]) + phi);
    }
  }
  return ORC_OK;
}

/* Seeded initial condition: Dirichlet(1..1) mass fractions (normalised Exp(1)
 * draws, counter-based so slabs reproduce the global field), T = 800 K +
 * 1200 K Gaussian hotspot (sigma = 0.1 L) at the domain centre, energy e(T,Y). */
void orc_initial_condition(uint64_t seed, const orc_mech* m, int n0, int n1, int n2,
                           double length, int i0_global, int n0_global, double* Y)
{
  const int S = m->S;
  const size_t ncell = (size_t)n0 * n1 * n2;
  const int ng[3] = {n0_global, n1, n2};
  const double sig = 0.1 * length;
  double* E = (double*)malloc(sizeof(double) * S);
  for (int i = 0; i < n0; ++i)
    for (int j = 0; j < n1; ++j)
      for (int k = 0; k < n2; ++k) {
        const size_t cell = ((size_t)i * n1 + j) * n2 + k;
        const uint64_t gcell = ((uint64_t)(i0_global + i) * n1 + j) * n2 + k;
        double sum = 0.0;
        for (int s = 0; s < S; ++s) {
          const uint64_t key = gcell * (uint64_t)S + (uint64_t)s;
          const uint64_t h = orc_mix64(seed + (key + 1) * 0x9E3779B97F4A7C15ULL);
          const double u = (double)((h >> 11) + 1) * 0x1.0p-53;
          E[s] = -log(u);
          sum += E[s];
        }
        for (int s = 0; s < S; ++s) Y[(size_t)s * ncell + cell] = E[s] / sum;
        const int co[3] = {i0_global + i, j, k};
        double r2 = 0.0;
        for (int d = 0; d < 3; ++d) {
          const double x = (co[d] + 0.5) * (length / ng[d]) - 0.5 * length;
          r2 += x * x;
        }
        const double T = 800.0 + 1200.0 * exp(-r2 / (2.0 * sig * sig));
        double E0 = 0.0, E1 = 0.0, E2 = 0.0;
        for (int s = 0; s < S; ++s) {
          const double y = Y[(size_t)s * ncell + cell];
          E0 += y * m->c0[s];
          E1 += y * m->c1[s];
          E2 += y * m->c2[s];
        }
        Y[(size_t)S * ncell + cell] = (E2 * T + E1) * T + E0;
      }
  free(E);
}

/* ------------------------------------------------------------------ */
/* Problem callbacks (PartitionedSystem analogue)                     */
/* ------------------------------------------------------------------ */
typedef struct { const double* A; int n; size_t ncell; const double* y; double* out; } lin_job;
static void lin_range(void* p, size_t lo, size_t hi)
{
  lin_job* j = (lin_job*)p;
  const int n = j->n;
  for (size_t c = lo; c < hi; ++c)
    for (int a = 0; a < n; ++a) {
      /* mat_apply order, proj/src/models.cpp:30-34 */
      double acc = j->A[a * n] * j->y[c];
      for (int b = 1; b < n; ++b) acc = acc + j->A[a * n + b] * j->y[(size_t)b * j->ncell + c];
      j->out[(size_t)a * j->ncell + c] = acc;
    }
}

static void linear_rhs(const double* A, int n, size_t ncell, const double* y, double* out, int threads)
{
  lin_job j = {A, n, ncell, y, out};
  parallel_for(ncell, threads, lin_range, &j);
}

void orc_fast_rhs(const orc_problem* p, double t, const double* y, double* out)
{
  (void)t;
  const size_t dof = p->ncell * (size_t)p->ncomp;
  if (p->fast_kind == ORC_FAST_CHEM) chem_rhs_threads(p->mech, p->ncell, y, out, p->threads);
  else if (p->fast_kind == ORC_FAST_LINEAR) linear_rhs(p->fast_A, p->ncomp, p->ncell, y, out, p->threads);
  else memset(out, 0, sizeof(double) * dof);
}

void orc_slow_rhs(const orc_problem* p, double t, const double* y, double* out)
{
  (void)t;
  const size_t dof = p->ncell * (size_t)p->ncomp;
  if (p->slow_kind == ORC_SLOW_STENCIL) stencil_threads(p->grid, y, out, p->threads);
  else if (p->slow_kind == ORC_SLOW_LINEAR) linear_rhs(p->slow_A, p->ncomp, p->ncell, y, out, p->threads);
  else memset(out, 0, sizeof(double) * dof);
}

/* f_implicit of the IMEX split: d_impl * L7 y, L7 = 7-point Laplacian
 * (periodic; per axis (y+ + y-) - 2y over dx^2, axes summed in order) */
typedef struct { const orc_grid* g; const double* Y; double* out; double scale; } lap_job;
static void lap_range(void* pj, size_t lo, size_t hi)
{
  lap_job* jb = (lap_job*)pj;
  const orc_grid* g = jb->g;
  const int n[3] = {g->n0, g->n1, g->n2};
  const size_t ncell = (size_t)g->n0 * g->n1 * g->n2;
  const size_t strides[3] = {(size_t)g->n1 * g->n2, (size_t)g->n2, 1};
  double inv_dx2[3];
  for (int d = 0; d < 3; ++d) {
    const double dx = g->length / n[d];
    inv_dx2[d] = 1.0 / (dx * dx);
  }
  for (size_t idx = lo; idx < hi; ++idx) {
    const size_t comp = idx / ncell, cell = idx % ncell;
    const int co[3] = {(int)(cell / strides[0]), (int)((cell / strides[1]) % g->n1),
                       (int)(cell % g->n2)};
    const double* y = jb->Y + comp * ncell;
    double lap = 0.0;
    for (int d = 0; d < 3; ++d) {
      const size_t base = cell - (size_t)co[d] * strides[d];
      const double yp = y[base + (size_t)((co[d] + 1) % n[d]) * strides[d]];
      const double ym = y[base + (size_t)((co[d] - 1 + n[d]) % n[d]) * strides[d]];
      lap += ((yp + ym) - 2.0 * y[cell]) * inv_dx2[d];
    }
    jb->out[comp * ncell + cell] = jb->scale * lap;
  }
}

void orc_implicit_rhs(const orc_problem* p, double t, const double* y, double* out)
{
  (void)t;
  lap_job j = {p->grid, y, out, p->grid->d_impl};
  parallel_for(p->ncell * (size_t)p->ncomp, p->threads, lap_range, &j);
}

/* ------------------------------------------------------------------ */
/* Stepper                                                           */
/* ------------------------------------------------------------------ */
typedef struct {
  const orc_problem* p;
  int ndeg;              /* r.coeffs.size() = max(degrees(), 1) */
  double* coeffs;        /* ndeg x dof */
  double t_start, span;
  double* tmp;           /* forcing evaluation buffer */
} forced_rhs;

/* fast_rhs lambda, proj/src/mri.cpp:364-371, with ForcingPolynomial::evaluate
 * (proj/include/multirate/mri.hpp:98-107) */
static void eval_forced(const forced_rhs* fr, double theta, const double* v, double* out)
{
  const size_t dof = fr->p->ncell * (size_t)fr->p->ncomp;
  const double tau = (theta - fr->t_start) / fr->span;
  if (fr->p->fast_kind != ORC_FAST_NONE) orc_fast_rhs(fr->p, theta, v, out);
  else memset(out, 0, sizeof(double) * dof);
  double* f = fr->tmp;
  memcpy(f, fr->coeffs + (size_t)(fr->ndeg - 1) * dof, sizeof(double) * dof);
  for (int k = fr->ndeg - 2; k >= 0; --k) {
    const double* ck = fr->coeffs + (size_t)k * dof;
    for (size_t i = 0; i < dof; ++i) f[i] = f[i] * tau + ck[i];
  }
  axpy_into(out, 1.0, f, dof);
}

typedef struct { double* k[ORC_MAX_TABLE]; double* stage; double* out; } erk_ws;

/* erk_step, proj/src/erk.cpp:9-38; y is overwritten with the result on success */
static int erk_step_ws(const orc_table* tb, const forced_rhs* fr, double t, double* y,
                       double h, uint64_t* counter, int* fail_stage, erk_ws* ws)
{
  const size_t dof = fr->p->ncell * (size_t)fr->p->ncomp;
  if (h <= 0.0) return ORC_CONTRACT;
  const int s = tb->s;
  for (int i = 0; i < s; ++i) {
    memcpy(ws->stage, y, sizeof(double) * dof);
    for (int j = 0; j < i; ++j)
      if (tb->A[i][j] != 0.0) axpy_into(ws->stage, h * tb->A[i][j], ws->k[j], dof);
    if (!orc_all_finite(ws->stage, dof)) { *fail_stage = i; return ORC_INTEGRATION; }
    eval_forced(fr, t + tb->c[i] * h, ws->stage, ws->k[i]);
    if (counter) ++(*counter);
  }
  memcpy(ws->out, y, sizeof(double) * dof);
  for (int i = 0; i < s; ++i)
    if (tb->b[i] != 0.0) axpy_into(ws->out, h * tb->b[i], ws->k[i], dof);
  if (!orc_all_finite(ws->out, dof)) { *fail_stage = s; return ORC_INTEGRATION; }
  memcpy(y, ws->out, sizeof(double) * dof);
  return ORC_OK;
}

static int uses_implicit(const orc_coupling* cp) { return any_nonzero(cp->gamma, cp->ndeg_gamma, cp->s); }

static double dotv(const double* a, const double* b, size_t n)
{
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

/* ImplicitSolve of the IMEX split: newton_solve (proj/src/solvers.cpp:150-208)
 * on G(Y) = Y - gamma f_I(Y) - known from Y = known (WRMS weights newton_w), the
 * linear solve (I - gamma d_impl L7) dY = -G done by cg_iters iterations of
 * Jacobi-preconditioned CG from dY = 0, accumulated straight into Y.  Replaces
 * gmres_solve (solvers.cpp:34-117) for this linear SPD stage operator
 * (SURVEY.md 8(f)); the device runs the identical iteration.  Counters follow
 * newton_solve: one implicit eval per residual, one nonlinear iteration per
 * update; CG adds cg_iters linear iterations and cg_iters + 1 Jacobi
 * applications per update.  Returns 1 when converged. */
static int newton_pcg_stage(const orc_problem* p, double gamma, const double* known, double* Y,
                            double* r, double* z, double* q, double* pv, orc_counters* cnt)
{
  const orc_grid* g = p->grid;
  const size_t dof = p->ncell * (size_t)p->ncomp;
  const int n[3] = {g->n0, g->n1, g->n2};
  double sdx = 0.0;
  for (int d = 0; d < 3; ++d) {
    const double dx = g->length / n[d];
    sdx += 2.0 / (dx * dx);
  }
  const double dg = 1.0 + gamma * (g->d_impl * sdx);
  const double target = g->newton_safety * g->newton_tol;
  memcpy(Y, known, sizeof(double) * dof);
  for (int iter = 0; iter <= g->newton_max_iters; ++iter) {
    orc_implicit_rhs(p, 0.0, Y, q);              /* residual (solvers.cpp:168-177) */
    ++cnt->n_implicit_evals;
    double ss = 0.0;
    for (size_t i = 0; i < dof; ++i) {
      double G = Y[i] + (-gamma) * q[i];
      G = G + (-1.0) * known[i];
      r[i] = -G;
      const double Gw = g->newton_w ? G * g->newton_w[i] : G; /* wrms_norm, state_vector.hpp:119-129 */
      ss += Gw * Gw;
    }
    const double wrms = sqrt(ss / (double)dof);
    if (!isfinite(wrms)) return 0;
    if (wrms <= target) return 1;
    if (iter == g->newton_max_iters) break;
    for (size_t i = 0; i < dof; ++i) z[i] = r[i] / dg;
    memcpy(pv, z, sizeof(double) * dof);
    double rz = dotv(r, z, dof);
    for (int it = 0; it < g->cg_iters; ++it) {
      orc_implicit_rhs(p, 0.0, pv, q);           /* q = A p = p - gamma f_I(p) */
      for (size_t i = 0; i < dof; ++i) q[i] = pv[i] - gamma * q[i];
      const double pAp = dotv(pv, q, dof);
      const double alpha = pAp != 0.0 ? rz / pAp : 0.0;
      for (size_t i = 0; i < dof; ++i) {
        Y[i] = Y[i] + alpha * pv[i];
        r[i] = r[i] - alpha * q[i];
        z[i] = r[i] / dg;
      }
      const double rz_new = dotv(r, z, dof);
      const double beta = rz != 0.0 ? rz_new / rz : 0.0;
      for (size_t i = 0; i < dof; ++i) pv[i] = z[i] + beta * pv[i];
      rz = rz_new;
    }
    cnt->n_linear_iters += (uint64_t)g->cg_iters;
    cnt->n_precond_solves += (uint64_t)g->cg_iters + 1;
    ++cnt->n_nonlinear_iters;
  }
  return 0;
}

/* mri_step, proj/src/mri.cpp:323-435.  ImplicitSolve stages use
 * newton_pcg_stage.  y is overwritten on success, untouched on error. */
int orc_mri_step(const orc_coupling* cp, const orc_table* fast, int m, const orc_problem* p,
                 double t, double* y, double H, orc_counters* cnt, int* fail_stage, char* err,
                 size_t errlen)
{
  *fail_stage = -1;
  if (H <= 0.0) { if (err) snprintf(err, errlen, "mri_step: H must be positive"); return ORC_CONTRACT; }
  const int s = cp->s;
  const size_t dof = p->ncell * (size_t)p->ncomp;
  const int needs_implicit = uses_implicit(cp);
  const int has_imp = p->slow_kind == ORC_SLOW_STENCIL && p->grid && p->grid->imex;
  if (needs_implicit && !has_imp) {
    if (err) snprintf(err, errlen, "mri_step: coupling needs f_implicit");
    return ORC_CONTRACT;
  }
  if (!needs_implicit && has_imp) {
    if (err) snprintf(err, errlen, "mri_step: explicit coupling on a split slow partition");
    return ORC_CONTRACT;
  }
  const int has_slow = p->slow_kind != ORC_SLOW_NONE; /* resolve_slow_explicit, mri.cpp:310-319 */
  const int d = cp->ndeg_gamma > cp->ndeg_omega ? cp->ndeg_gamma : cp->ndeg_omega;
  const int ndeg = d > 1 ? d : 1;

  double* fE[ORC_MAX_STAGES] = {0};
  double* fI[ORC_MAX_STAGES] = {0};
  double* Y = (double*)malloc(sizeof(double) * dof);
  double* coeffs = (double*)malloc(sizeof(double) * dof * (size_t)ndeg);
  double* tmp = (double*)malloc(sizeof(double) * dof);
  double* cgw = needs_implicit ? (double*)malloc(sizeof(double) * dof * 5) : NULL;
  erk_ws ws;
  for (int i = 0; i < fast->s; ++i) ws.k[i] = (double*)malloc(sizeof(double) * dof);
  ws.stage = (double*)malloc(sizeof(double) * dof);
  ws.out = (double*)malloc(sizeof(double) * dof);
  int rc = ORC_OK;
  memcpy(Y, y, sizeof(double) * dof);

#define EVAL_SLOW_AT(j)                                                  \
  do {                                                                   \
    if (has_slow && cp->eval_explicit_at[(j)]) {                         \
      if (!fE[(j)]) fE[(j)] = (double*)malloc(sizeof(double) * dof);    \
      orc_slow_rhs(p, t + cp->c[(j)] * H, Y, fE[(j)]);                   \
      ++cnt->n_explicit_evals;                                           \
    }                                                                    \
    if (needs_implicit && cp->fI_referenced[(j)] &&                     \
        cp->kind[(j)] != ORC_IMPLICIT_SOLVE) {                           \
      if (!fI[(j)]) fI[(j)] = (double*)malloc(sizeof(double) * dof);    \
      orc_implicit_rhs(p, t + cp->c[(j)] * H, Y, fI[(j)]);               \
      ++cnt->n_implicit_evals;                                           \
    }                                                                    \
  } while (0)

  EVAL_SLOW_AT(0);
  for (int i = 1; i < s && rc == ORC_OK; ++i) {
    const double dc = cp->c[i] - cp->c[i - 1];
    if (cp->kind[i] == ORC_FAST_IVP) {
      /* build_forcing, mri.cpp:266-303: gamma over fI, then omega over fE */
      memset(coeffs, 0, sizeof(double) * dof * (size_t)ndeg);
      for (int pass = 0; pass < 2 && rc == ORC_OK; ++pass) {
        const int nd = pass == 0 ? cp->ndeg_gamma : cp->ndeg_omega;
        for (int k = 0; k < nd && rc == ORC_OK; ++k)
          for (int j = 0; j < i; ++j) {
            const double coef = pass == 0 ? cp->gamma[k][i][j] : cp->omega[k][i][j];
            if (coef == 0.0) continue;
            double* h = pass == 0 ? fI[j] : fE[j];
            if (!h) {
              if (err) snprintf(err, errlen, "build_forcing: missing %s value at stage %d",
                                pass == 0 ? "implicit" : "explicit", j);
              *fail_stage = i;
              rc = ORC_INTEGRATION;
              break;
            }
            axpy_into(coeffs + (size_t)k * dof, coef / dc, h, dof);
          }
      }
      if (rc != ORC_OK) break;
      forced_rhs fr = {p, ndeg, coeffs, t + cp->c[i - 1] * H, dc * H, tmp};
      long ns = lround((double)m * dc);
      const int n_sub = (int)(ns > 1 ? ns : 1);
      const double h_sub = fr.span / n_sub;
      uint64_t* counter = p->fast_kind != ORC_FAST_NONE ? &cnt->n_fast_evals : NULL;
      for (int sub = 0; sub < n_sub; ++sub) {
        rc = erk_step_ws(fast, &fr, fr.t_start + sub * h_sub, Y, h_sub, counter, fail_stage, &ws);
        if (rc != ORC_OK) {
          if (err) snprintf(err, errlen, "erk_step: non-finite stage value");
          break;
        }
      }
      if (rc != ORC_OK) break;
      ++cnt->n_fast_ivps;
    } else {
      /* mri.cpp:380-384: known = Y + sum_j H (gbar_ij fI_j + wbar_ij fE_j) */
      for (int j = 0; j < i && rc == ORC_OK; ++j) {
        if (cp->gbar[i][j] != 0.0) {
          if (!fI[j]) { rc = ORC_CONTRACT; break; }
          axpy_into(Y, H * cp->gbar[i][j], fI[j], dof);
        }
        if (cp->wbar[i][j] != 0.0) {
          if (!fE[j]) { rc = ORC_CONTRACT; break; }
          axpy_into(Y, H * cp->wbar[i][j], fE[j], dof);
        }
      }
      if (rc != ORC_OK) {
        if (err) snprintf(err, errlen, "axpy_into: length mismatch");
        break;
      }
      if (cp->kind[i] == ORC_IMPLICIT_SOLVE) {
        if (!orc_all_finite(Y, dof)) { /* mri.cpp:386-390 */
          if (err) snprintf(err, errlen, "mri_step: non-finite stage data at stage %d", i);
          *fail_stage = i;
          rc = ORC_INTEGRATION;
          break;
        }
        const double gamma = H * cp->gbar[i][i];
        double* known = cgw;
        memcpy(known, Y, sizeof(double) * dof);
        const int ok = newton_pcg_stage(p, gamma, known, Y, cgw + dof, cgw + 2 * dof,
                                        cgw + 3 * dof, cgw + 4 * dof, cnt);
        ++cnt->n_implicit_solves;
        if (!ok) { /* mri.cpp:404-410 */
          if (err) snprintf(err, errlen, "mri_step: nonlinear solve failed at stage %d", i);
          *fail_stage = i;
          rc = ORC_INTEGRATION;
          break;
        }
        /* mri.cpp:418-421: fI_i = (Y - known) / gamma */
        if (!fI[i]) fI[i] = (double*)malloc(sizeof(double) * dof);
        memcpy(fI[i], Y, sizeof(double) * dof);
        axpy_into(fI[i], -1.0, known, dof);
        for (size_t q = 0; q < dof; ++q) fI[i][q] /= gamma;
      }
    }
    if (!orc_all_finite(Y, dof)) { /* mri.cpp:427-431 */
      if (err) snprintf(err, errlen, "mri_step: non-finite state at stage %d", i);
      *fail_stage = i;
      rc = ORC_INTEGRATION;
      break;
    }
    EVAL_SLOW_AT(i);
  }
#undef EVAL_SLOW_AT
  if (rc == ORC_OK) memcpy(y, Y, sizeof(double) * dof);
  for (int i = 0; i < s; ++i) { free(fE[i]); free(fI[i]); }
  for (int i = 0; i < fast->s; ++i) free(ws.k[i]);
  free(ws.stage); free(ws.out); free(Y); free(coeffs); free(tmp); free(cgw);
  return rc;
}

/* mri_integrate, proj/src/mri.cpp:524-540 */
int orc_mri_integrate(const orc_coupling* cp, const orc_table* fast, int m, const orc_problem* p,
                      double t0, double tf, double H, double* y, orc_counters* cnt,
                      int* fail_stage, char* err, size_t errlen)
{
  *fail_stage = -1;
  if (tf <= t0) { if (err) snprintf(err, errlen, "mri_integrate: tf must exceed t0"); return ORC_CONTRACT; }
  const long n_steps = (long)ceil((tf - t0) / H - 1e-12);
  const size_t dof = p->ncell * (size_t)p->ncomp;
  double* work = (double*)malloc(sizeof(double) * dof);
  memcpy(work, y, sizeof(double) * dof);
  double t = t0;
  int rc = ORC_OK;
  for (long i = 0; i < n_steps; ++i) {
    const double step = (i == n_steps - 1) ? (tf - t) : H;
    rc = orc_mri_step(cp, fast, m, p, t, work, step, cnt, fail_stage, err, errlen);
    if (rc != ORC_OK) break;
    t = (i == n_steps - 1) ? tf : t0 + (double)(i + 1) * H;
  }
  if (rc == ORC_OK) memcpy(y, work, sizeof(double) * dof);
  free(work);
  return rc;
}

/* ARK4(3)6L[2]SA pair, proj/src/butcher.cpp:362-427 (make_ark436) */
typedef struct { double AE[6][6], AI[6][6], b[6], c[6]; } ark436;
static void ark436_tables(ark436* t)
{
  memset(t, 0, sizeof(*t));
  t->c[0] = 0; t->c[1] = 0.5; t->c[2] = 83.0 / 250.0; t->c[3] = 31.0 / 50.0;
  t->c[4] = 17.0 / 20.0; t->c[5] = 1.0;
  t->AE[1][0] = 0.5;
  t->AE[2][0] = 13861.0 / 62500.0;
  t->AE[2][1] = 6889.0 / 62500.0;
  t->AE[3][0] = -116923316275.0 / 2393684061468.0;
  t->AE[3][1] = -2731218467317.0 / 15368042101831.0;
  t->AE[3][2] = 9408046702089.0 / 11113171139209.0;
  t->AE[4][0] = -451086348788.0 / 2902428689909.0;
  t->AE[4][1] = -2682348792572.0 / 7519795681897.0;
  t->AE[4][2] = 12662868775082.0 / 11960479115383.0;
  t->AE[4][3] = 3355817975965.0 / 11060851509271.0;
  t->AE[5][0] = 647845179188.0 / 3216320057751.0;
  t->AE[5][1] = 73281519250.0 / 8382639484533.0;
  t->AE[5][2] = 552539513391.0 / 3454668386233.0;
  t->AE[5][3] = 3354512671639.0 / 8306763924573.0;
  t->AE[5][4] = 4040.0 / 17871.0;
  t->b[0] = 82889.0 / 524892.0; t->b[1] = 0.0; t->b[2] = 15625.0 / 83664.0;
  t->b[3] = 69875.0 / 102672.0; t->b[4] = -2260.0 / 8211.0; t->b[5] = 0.25;
  t->AI[1][0] = 0.25; t->AI[1][1] = 0.25;
  t->AI[2][0] = 8611.0 / 62500.0; t->AI[2][1] = -1743.0 / 31250.0; t->AI[2][2] = 0.25;
  t->AI[3][0] = 5012029.0 / 34652500.0; t->AI[3][1] = -654441.0 / 2922500.0;
  t->AI[3][2] = 174375.0 / 388108.0; t->AI[3][3] = 0.25;
  t->AI[4][0] = 15267082809.0 / 155376265600.0; t->AI[4][1] = -71443401.0 / 120774400.0;
  t->AI[4][2] = 730878875.0 / 902184768.0; t->AI[4][3] = 2285395.0 / 8070912.0;
  t->AI[4][4] = 0.25;
  t->AI[5][0] = 82889.0 / 524892.0; t->AI[5][1] = 0.0; t->AI[5][2] = 15625.0 / 83664.0;
  t->AI[5][3] = 69875.0 / 102672.0; t->AI[5][4] = -2260.0 / 8211.0; t->AI[5][5] = 0.25;
}

/* combined_explicit of ark_imex_step, proj/src/mri.cpp:450-456:
 * out = f_fast (or 0); out += 1.0 f_explicit */
static void combined_explicit(const orc_problem* p, double t, const double* y, double* out,
                              double* tmp)
{
  const size_t dof = p->ncell * (size_t)p->ncomp;
  if (p->fast_kind != ORC_FAST_NONE) orc_fast_rhs(p, t, y, out);
  else memset(out, 0, sizeof(double) * dof);
  if (p->slow_kind != ORC_SLOW_NONE) {
    orc_slow_rhs(p, t, y, tmp);
    axpy_into(out, 1.0, tmp, dof);
  }
}

/* ark_imex_step, proj/src/mri.cpp:437-522, with newton_pcg_stage as the
 * ImplicitStageSolver (same Newton iteration; fixed-iteration PCG instead of
 * GMRES).  y is overwritten on success, untouched on error. */
int orc_ark_imex_step(const orc_problem* p, double t, double* y, double H, orc_counters* cnt,
                      int* fail_stage, char* err, size_t errlen)
{
  *fail_stage = -1;
  if (H <= 0.0) { if (err) snprintf(err, errlen, "ark_imex_step: H must be positive"); return ORC_CONTRACT; }
  if (!(p->slow_kind == ORC_SLOW_STENCIL && p->grid && p->grid->imex)) {
    if (err) snprintf(err, errlen, "ark_imex_step: f_implicit required");
    return ORC_CONTRACT;
  }
  ark436 tb;
  ark436_tables(&tb);
  const int s = 6;
  const size_t dof = p->ncell * (size_t)p->ncomp;
  double* fE[6];
  double* fI[6];
  for (int i = 0; i < s; ++i) {
    fE[i] = (double*)malloc(sizeof(double) * dof);
    fI[i] = (double*)malloc(sizeof(double) * dof);
  }
  double* Y = (double*)malloc(sizeof(double) * dof);
  double* cgw = (double*)malloc(sizeof(double) * dof * 5);
  int rc = ORC_OK;
  combined_explicit(p, t, y, fE[0], cgw);
  ++cnt->n_explicit_evals;
  orc_implicit_rhs(p, t, y, fI[0]);
  ++cnt->n_implicit_evals;
  for (int i = 1; i < s && rc == ORC_OK; ++i) {
    double* known = cgw;
    memcpy(known, y, sizeof(double) * dof);
    for (int j = 0; j < i; ++j) {
      if (tb.AE[i][j] != 0.0) axpy_into(known, H * tb.AE[i][j], fE[j], dof);
      if (tb.AI[i][j] != 0.0) axpy_into(known, H * tb.AI[i][j], fI[j], dof);
    }
    const double t_stage = t + tb.c[i] * H;
    if (!orc_all_finite(known, dof)) {
      if (err) snprintf(err, errlen, "ark_imex_step: non-finite stage data at stage %d", i);
      *fail_stage = i;
      rc = ORC_INTEGRATION;
      break;
    }
    const double gamma = H * tb.AI[i][i];
    const int ok = newton_pcg_stage(p, gamma, known, Y, cgw + dof, cgw + 2 * dof, cgw + 3 * dof,
                                    cgw + 4 * dof, cnt);
    ++cnt->n_implicit_solves;
    if (!ok) {
      if (err) snprintf(err, errlen, "ark_imex_step: nonlinear solve failed at stage %d", i);
      *fail_stage = i;
      rc = ORC_INTEGRATION;
      break;
    }
    memcpy(fI[i], Y, sizeof(double) * dof);
    axpy_into(fI[i], -1.0, known, dof);
    for (size_t q = 0; q < dof; ++q) fI[i][q] /= gamma;
    combined_explicit(p, t_stage, Y, fE[i], cgw + dof);
    ++cnt->n_explicit_evals;
  }
  if (rc == ORC_OK) {
    memcpy(Y, y, sizeof(double) * dof);
    for (int j = 0; j < s; ++j) {
      const double b = tb.b[j];
      if (b != 0.0) {
        axpy_into(Y, H * b, fE[j], dof);
        axpy_into(Y, H * b, fI[j], dof);
      }
    }
    if (!orc_all_finite(Y, dof)) {
      if (err) snprintf(err, errlen, "ark_imex_step: non-finite result");
      *fail_stage = s;
      rc = ORC_INTEGRATION;
    } else {
      memcpy(y, Y, sizeof(double) * dof);
    }
  }
  for (int i = 0; i < s; ++i) { free(fE[i]); free(fI[i]); }
  free(Y); free(cgw);
  return rc;
}

/* ark_imex_integrate, proj/src/mri.cpp:542-557 */
int orc_ark_imex_integrate(const orc_problem* p, double t0, double tf, double H, double* y,
                           orc_counters* cnt, int* fail_stage, char* err, size_t errlen)
{
  *fail_stage = -1;
  if (tf <= t0) { if (err) snprintf(err, errlen, "ark_imex_integrate: tf must exceed t0"); return ORC_CONTRACT; }
  const long n_steps = (long)ceil((tf - t0) / H - 1e-12);
  const size_t dof = p->ncell * (size_t)p->ncomp;
  double* work = (double*)malloc(sizeof(double) * dof);
  memcpy(work, y, sizeof(double) * dof);
  double t = t0;
  int rc = ORC_OK;
  for (long i = 0; i < n_steps; ++i) {
    const double step = (i == n_steps - 1) ? (tf - t) : H;
    rc = orc_ark_imex_step(p, t, work, step, cnt, fail_stage, err, errlen);
    if (rc != ORC_OK) break;
    t = (i == n_steps - 1) ? tf : t0 + (double)(i + 1) * H;
  }
  if (rc == ORC_OK) memcpy(y, work, sizeof(double) * dof);
  free(work);
  return rc;
}

/* PartitionedSystem::sum_rhs, proj/include/multirate/partitioned_system.hpp:41-48:
 * out = 0; out += 1.0 f_fast; out += 1.0 f_implicit; out += 1.0 f_explicit */
static void sum_rhs(const orc_problem* p, double t, const double* y, double* out, double* tmp)
{
  const size_t dof = p->ncell * (size_t)p->ncomp;
  memset(out, 0, sizeof(double) * dof);
  if (p->fast_kind != ORC_FAST_NONE) {
    orc_fast_rhs(p, t, y, tmp);
    axpy_into(out, 1.0, tmp, dof);
  }
  if (p->slow_kind == ORC_SLOW_STENCIL && p->grid && p->grid->imex) {
    orc_implicit_rhs(p, t, y, tmp);
    axpy_into(out, 1.0, tmp, dof);
  }
  if (p->slow_kind != ORC_SLOW_NONE) {
    orc_slow_rhs(p, t, y, tmp);
    axpy_into(out, 1.0, tmp, dof);
  }
}

/* reference_solution, proj/src/erk.cpp:59-75: erk_integrate (:40-57) of the
 * registered cash-karp5 table (butcher.cpp:305-321) on sum_rhs; erk_step
 * (:9-38) semantics, no counters.  y is overwritten on success. */
/* erk_integrate (proj/src/erk.cpp:40-57) with erk_step (:9-38) on sum_rhs;
   *evals (may be NULL) += 1 per stage evaluation (:28) */
int orc_erk_integrate(const orc_problem* p, const char* table, double t0, double tf, double h,
                      double* y, uint64_t* evals, int* fail_stage, char* err, size_t errlen)
{
  *fail_stage = -1;
  if (tf <= t0) { if (err) snprintf(err, errlen, "erk_integrate: tf must exceed t0"); return ORC_CONTRACT; }
  if (h <= 0.0) { if (err) snprintf(err, errlen, "erk_integrate: h must be positive"); return ORC_CONTRACT; }
  orc_table tb;
  if (orc_table_lookup(table, &tb) != ORC_OK) {
    if (err) snprintf(err, errlen, "unknown Butcher table '%s'", table);
    return ORC_CONTRACT;
  }
  for (int i = 0; i < tb.s; ++i)
    for (int j = i; j < tb.s; ++j)
      if (tb.A[i][j] != 0.0) {
        if (err) snprintf(err, errlen, "erk_step: table must be explicit");
        return ORC_CONTRACT;
      }
  const size_t dof = p->ncell * (size_t)p->ncomp;
  const int s = tb.s;
  double* k[ORC_MAX_TABLE];
  for (int i = 0; i < s; ++i) k[i] = (double*)malloc(sizeof(double) * dof);
  double* stage = (double*)malloc(sizeof(double) * dof);
  double* tmp = (double*)malloc(sizeof(double) * dof);
  double* work = (double*)malloc(sizeof(double) * dof);
  memcpy(work, y, sizeof(double) * dof);
  const long n_steps = (long)ceil((tf - t0) / h - 1e-12);
  double t = t0;
  int rc = ORC_OK;
  for (long n = 0; n < n_steps && rc == ORC_OK; ++n) {
    const double step = (n == n_steps - 1) ? (tf - t) : h;
    for (int i = 0; i < s && rc == ORC_OK; ++i) {
      memcpy(stage, work, sizeof(double) * dof);
      for (int j = 0; j < i; ++j)
        if (tb.A[i][j] != 0.0) axpy_into(stage, step * tb.A[i][j], k[j], dof);
      if (!orc_all_finite(stage, dof)) {
        if (err) snprintf(err, errlen, "erk_step: non-finite stage value");
        *fail_stage = i;
        rc = ORC_INTEGRATION;
        break;
      }
      sum_rhs(p, t + tb.c[i] * step, stage, k[i], tmp);
      if (evals) ++*evals;
    }
    if (rc != ORC_OK) break;
    memcpy(stage, work, sizeof(double) * dof);
    for (int i = 0; i < s; ++i)
      if (tb.b[i] != 0.0) axpy_into(stage, step * tb.b[i], k[i], dof);
    if (!orc_all_finite(stage, dof)) {
      if (err) snprintf(err, errlen, "erk_step: non-finite result");
      *fail_stage = s;
      rc = ORC_INTEGRATION;
      break;
    }
    memcpy(work, stage, sizeof(double) * dof);
    t = (n == n_steps - 1) ? tf : t0 + (double)(n + 1) * h;
  }
  if (rc == ORC_OK) memcpy(y, work, sizeof(double) * dof);
  for (int i = 0; i < s; ++i) free(k[i]);
  free(stage); free(tmp); free(work);
  return rc;
}

/* reference_solution (proj/src/erk.cpp:59-75): cash-karp5 on sum_rhs */
int orc_reference_solution(const orc_problem* p, double t0, double tf, double h, double* y,
                           int* fail_stage, char* err, size_t errlen)
{
  return orc_erk_integrate(p, "cash-karp5", t0, tf, h, y, NULL, fail_stage, err, errlen);
}

/* ------------------------------------------------------------------ */
/* Flat session API for ctypes callers (tests, bench cpu_baseline)     */
/* ------------------------------------------------------------------ */
struct orc_sys {
  orc_sys_cfg cfg;
  orc_mech mech;
  orc_grid grid;
  orc_problem prob;
  int has_mech;
};

orc_sys* orc_sys_create(const orc_sys_cfg* cfg)
{
  orc_sys* s = (orc_sys*)calloc(1, sizeof(orc_sys));
  s->cfg = *cfg;
  if (cfg->fast_kind == ORC_FAST_CHEM || cfg->species) {
    if (orc_mech_init(&s->mech, cfg->S, cfg->R, cfg->rho, cfg->species, cfg->reactions,
                      cfg->rspecies) != ORC_OK) {
      free(s);
      return NULL;
    }
    s->has_mech = 1;
  }
  s->grid.n0 = cfg->n0; s->grid.n1 = cfg->n1; s->grid.n2 = cfg->n2;
  s->grid.length = cfg->length;
  s->grid.ncomp = cfg->ncomp;
  s->grid.order = cfg->order;
  s->grid.diffusion = cfg->diffusion;
  s->grid.vel_kind = cfg->vel_kind;
  s->grid.imex = cfg->imex;
  s->grid.d_impl = cfg->d_impl;
  s->grid.cg_iters = cfg->cg_iters;
  s->grid.newton_tol = cfg->newton_tol;
  s->grid.newton_safety = cfg->newton_safety;
  s->grid.newton_max_iters = cfg->newton_max_iters;
  s->grid.newton_w = cfg->newton_w;
  for (int d = 0; d < 3; ++d) s->grid.u_const[d] = cfg->u_const[d];
  if (cfg->vel_kind == 1)
    for (int d = 0; d < 3; ++d)
      for (int q = 0; q < 2; ++q) s->grid.prof[d][q] = cfg->prof + ((size_t)d * 2 + q) * cfg->prof_nmax;
  s->prob.ncell = (size_t)cfg->n0 * cfg->n1 * cfg->n2;
  s->prob.ncomp = cfg->ncomp;
  s->prob.fast_kind = cfg->fast_kind;
  s->prob.slow_kind = cfg->slow_kind;
  s->prob.mech = s->has_mech ? &s->mech : NULL;
  s->prob.grid = &s->grid;
  s->prob.fast_A = cfg->fast_A;
  s->prob.slow_A = cfg->slow_A;
  s->prob.threads = cfg->threads;
  return s;
}

void orc_sys_destroy(orc_sys* s)
{
  if (!s) return;
  if (s->has_mech) orc_mech_free(&s->mech);
  free(s);
}

const orc_problem* orc_sys_problem(const orc_sys* s) { return &s->prob; }
void orc_sys_set_threads(orc_sys* s, int threads) { s->prob.threads = threads; }

int orc_sys_fast_rhs(orc_sys* s, double t, const double* y, double* out)
{
  orc_fast_rhs(&s->prob, t, y, out);
  return ORC_OK;
}

int orc_sys_slow_rhs(orc_sys* s, double t, const double* y, double* out)
{
  orc_slow_rhs(&s->prob, t, y, out);
  return ORC_OK;
}

int orc_sys_implicit_rhs(orc_sys* s, double t, const double* y, double* out)
{
  if (!s->cfg.imex) return ORC_CONTRACT;
  orc_implicit_rhs(&s->prob, t, y, out);
  return ORC_OK;
}

int orc_sys_initial_condition(orc_sys* s, uint64_t seed, double* Y)
{
  if (!s->has_mech) return ORC_CONTRACT;
  orc_initial_condition(seed, &s->mech, s->cfg.n0, s->cfg.n1, s->cfg.n2, s->cfg.length,
                        s->cfg.i0_global, s->cfg.n0_global, Y);
  return ORC_OK;
}

int orc_coupling_load(const char* spec, orc_coupling* out, char* err, size_t errlen)
{
  if (!strncmp(spec, "mri-coupling", 12)) return orc_coupling_import(spec, out, err, errlen);
  int rc = orc_coupling_register(spec, out);
  if (rc != ORC_OK && err) snprintf(err, errlen, "register_coupling: unknown name '%s'", spec);
  return rc;
}

static void counters_in(const uint64_t* c, orc_counters* o) { memcpy(o, c, sizeof(*o)); }
static void counters_out(const orc_counters* o, uint64_t* c) { memcpy(c, o, sizeof(*o)); }

int orc_sys_mri_step(orc_sys* s, const char* coupling, const char* fast_table, int m, double t,
                     double H, double* y, uint64_t* counters, int* fail_stage, char* err,
                     size_t errlen)
{
  orc_coupling cp;
  orc_table tb;
  int rc = orc_coupling_load(coupling, &cp, err, errlen);
  if (rc != ORC_OK) return rc;
  if (orc_table_lookup(fast_table, &tb) != ORC_OK) {
    if (err) snprintf(err, errlen, "lookup_table: unknown method '%s'", fast_table);
    return ORC_CONTRACT;
  }
  orc_counters c;
  counters_in(counters, &c);
  rc = orc_mri_step(&cp, &tb, m, &s->prob, t, y, H, &c, fail_stage, err, errlen);
  counters_out(&c, counters);
  return rc;
}

int orc_sys_mri_integrate(orc_sys* s, const char* coupling, const char* fast_table, int m,
                          double t0, double tf, double H, double* y, uint64_t* counters,
                          int* fail_stage, char* err, size_t errlen)
{
  orc_coupling cp;
  orc_table tb;
  int rc = orc_coupling_load(coupling, &cp, err, errlen);
  if (rc != ORC_OK) return rc;
  if (orc_table_lookup(fast_table, &tb) != ORC_OK) {
    if (err) snprintf(err, errlen, "lookup_table: unknown method '%s'", fast_table);
    return ORC_CONTRACT;
  }
  orc_counters c;
  counters_in(counters, &c);
  rc = orc_mri_integrate(&cp, &tb, m, &s->prob, t0, tf, H, y, &c, fail_stage, err, errlen);
  counters_out(&c, counters);
  return rc;
}

int orc_sys_reference_solution(orc_sys* s, double t0, double tf, double h, double* y,
                               int* fail_stage, char* err, size_t errlen)
{
  return orc_reference_solution(&s->prob, t0, tf, h, y, fail_stage, err, errlen);
}

int orc_sys_erk_integrate(orc_sys* s, const char* table, double t0, double tf, double h, double* y,
                          uint64_t* evals, int* fail_stage, char* err, size_t errlen)
{
  return orc_erk_integrate(&s->prob, table, t0, tf, h, y, evals, fail_stage, err, errlen);
}

int orc_sys_ark_imex_integrate(orc_sys* s, double t0, double tf, double H, double* y,
                               uint64_t* counters, int* fail_stage, char* err, size_t errlen)
{
  orc_counters c;
  counters_in(counters, &c);
  const int rc = orc_ark_imex_integrate(&s->prob, t0, tf, H, y, &c, fail_stage, err, errlen);
  counters_out(&c, counters);
  return rc;
}
