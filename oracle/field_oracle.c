/*
 * field_oracle.c -- TEST INFRASTRUCTURE ONLY.  CPU restatement of the field
 * arithmetic of the synthetic BRAMS-like timestep, over the UNDECOMPOSED grid.
 * Used by tests/ (parity checker), __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg.  Never linked into the product.
 *
 * PARITY STATUS: field values are "parity unpinned" by the reference.  The
 * reference simulator computes no field values ("No actual numerical stencil
 * values are computed -- only work/byte counts"; f is "abstracted
 * to a fixed per-iteration work unit").  This file therefore fixes
 * the arithmetic the paper leaves open and is itself pinned by
 *   - the reference's trip counts: sum over a chunk of T(x,y) equals
 *     physics_work(sub, C, nz).total()   (workload.hpp:199-204), and
 *   - committed golden vectors (tests/golden/fields_*.json, made by
 *     oracle/gen_golden.py from this file) plus the invariant that results are
 *     bitwise independent of chunking, mapping, GPU count and balancing.
 *
 * Semantics:
 *  State U[f][k][y][x] (F fields, x fastest) and physics array A[k][y][x].
 *  One timestep (Fig. 2, :107-134): Jacobi U^t -> U^{t+1}
 *  and physics A <- Phys(A, B = U^t field 0, C); the two read only U^t.
 *  Jacobi ("3D Jacobi ... laminar diffusion"): 7-point,
 *    s = ((xm + xp) + (ym + yp)) + (zm + zp);  u' = fma(1/8, s, 1/4 * u),
 *    zero-flux boundaries (an out-of-domain neighbour is the cell itself).
 *  Physics (Fig. 4, :227-243; Fig. 1, :89-97): per column
 *    T = floor(nz * C(x,y)) - 1 trips (the Fortran `do k=2,mzp*C`), level
 *    index cycling k -> k mod nz (the legal form of Fig. 4's wrap), and
 *    A(l) = f(B(l), A(l-1 mod nz)) starting from A(0).
 *    f(b,a): y = fma(1/2, a, b/2); eb = fma(b, 2^-9, 2^-9);
 *            n_inner times { u = fma(-y, y, y); y = fma(255/64, u, eb) }.
 *  Initial values: splitmix64 hash of the global index (engine.hpp:112-118
 *    mixer), (h >> 11) * 2^-53; A is "field F".
 * Every value operation is a correctly rounded IEEE add/mul/fma, compiled
 * with -ffp-contract=off, so the CUDA kernels can match it bit for bit.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define W0 0.25
#define W1 0.125
#define RMAP 3.984375
#define EPS 0.001953125
#define OBLK 64

static uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

static double unit_hash(uint64_t seed, uint64_t idx) {
  return (double)(mix64(seed ^ mix64(idx)) >> 11) * 0x1.0p-53;
}

/* U: F*nz*ny*nx, A: nz*ny*nx */
void oracle_init(int nx, int ny, int nz, int F, uint64_t seed, double* U, double* A) {
  const int64_t plane = (int64_t)nx * ny;
#pragma omp parallel for schedule(static)
  for (int64_t fk = 0; fk < (int64_t)(F + 1) * nz; ++fk) {
    double* dst = fk < (int64_t)F * nz ? U + fk * plane : A + (fk - (int64_t)F * nz) * plane;
    for (int64_t r = 0; r < plane; ++r)
      dst[r] = unit_hash(seed, (uint64_t)(fk * plane + r));
  }
}

void oracle_jacobi(int nx, int ny, int nz, int F, const double* in, double* out) {
  const int64_t plane = (int64_t)nx * ny;
#pragma omp parallel for schedule(static)
  for (int64_t fk = 0; fk < (int64_t)F * nz; ++fk) {
    const int k = (int)(fk % nz);
    const double* c = in + fk * plane;
    const double* dn = k > 0 ? c - plane : c;
    const double* up = k + 1 < nz ? c + plane : c;
    double* o = out + fk * plane;
    for (int y = 0; y < ny; ++y) {
      const double* row = c + (int64_t)y * nx;
      const double* rn = y > 0 ? row - nx : row;
      const double* rs = y + 1 < ny ? row + nx : row;
      const double* zd = dn + (int64_t)y * nx;
      const double* zu = up + (int64_t)y * nx;
      double* orow = o + (int64_t)y * nx;
      /* x = 0 and x = nx-1 carry the zero-flux boundary; the interior loop is
       * branch free so it vectorises */
      for (int x = 0; x < nx; x += (nx > 1 ? nx - 1 : 1)) {
        const double u = row[x];
        const double xm = x > 0 ? row[x - 1] : u;
        const double xp = x + 1 < nx ? row[x + 1] : u;
        const double s = ((xm + xp) + (rn[x] + rs[x])) + (zd[x] + zu[x]);
        orow[x] = fma(W1, s, W0 * row[x]);
      }
      for (int x = 1; x < nx - 1; ++x) {
        const double s = ((row[x - 1] + row[x + 1]) + (rn[x] + rs[x])) + (zd[x] + zu[x]);
        orow[x] = fma(W1, s, W0 * row[x]);
      }
    }
  }
}

/* Column recurrence for one grid row, columns processed side by side so the
 * compiler can vectorise the micro-steps across columns. */
static void physics_row(int nx, int ny, int nz, int n_inner, int y, const double* crow,
                        const double* B, double* A, int* T, double* a, double* yy,
                        double* eb, int* act) {
  const int64_t plane = (int64_t)nx * ny;
  int tmax = 0;
  for (int x = 0; x < nx; ++x) {
    int t = (int)floor((double)nz * crow[x]) - 1;
    if (t < 0) t = 0;
    T[x] = t;
    if (t > tmax) tmax = t;
    a[x] = A[(int64_t)y * nx + x];
  }
  for (int t = 1; t <= tmax; ++t) {
    const int l = t % nz;
    const double* b = B + l * plane + (int64_t)y * nx;
    int n = 0;
    for (int x = 0; x < nx; ++x)
      if (T[x] >= t) act[n++] = x;
    for (int j = 0; j < n; ++j) {
      const double bv = b[act[j]];
      eb[j] = fma(bv, EPS, EPS);
      yy[j] = fma(0.5, a[act[j]], 0.5 * bv);
    }
    /* micro-steps on register blocks of OBLK columns (independent chains) */
    int j0 = 0;
    for (; j0 + OBLK <= n; j0 += OBLK) {
      double yv[OBLK], ev[OBLK];
      for (int j = 0; j < OBLK; ++j) {
        yv[j] = yy[j0 + j];
        ev[j] = eb[j0 + j];
      }
      for (int i = 0; i < n_inner; ++i) {
#pragma omp simd
        for (int j = 0; j < OBLK; ++j) {
          const double u = fma(-yv[j], yv[j], yv[j]);
          yv[j] = fma(RMAP, u, ev[j]);
        }
      }
      for (int j = 0; j < OBLK; ++j) yy[j0 + j] = yv[j];
    }
    for (int i = 0; i < n_inner; ++i)
      for (int j = j0; j < n; ++j) {
        const double u = fma(-yy[j], yy[j], yy[j]);
        yy[j] = fma(RMAP, u, eb[j]);
      }
    double* arow = A + l * plane + (int64_t)y * nx;
    for (int j = 0; j < n; ++j) {
      a[act[j]] = yy[j];
      arow[act[j]] = yy[j];
    }
  }
}

/* cbase: base load multiplier (ny*nx, y-major); the field used is cbase shifted
 * down by `shift` rows with wrap (workload.hpp:185-195).  B = field 0 of Uin. */
void oracle_physics(int nx, int ny, int nz, int n_inner, const double* cbase, int shift,
                    const double* Uin, double* A) {
  shift %= ny;
#pragma omp parallel
  {
    int* T = (int*)malloc(sizeof(int) * nx * 2);
    int* act = T + nx;
    double* buf = (double*)malloc(sizeof(double) * nx * 3);
#pragma omp for schedule(dynamic, 1)
    for (int y = 0; y < ny; ++y) {
      const int src = (y - shift + ny) % ny;
      physics_row(nx, ny, nz, n_inner, y, cbase + (int64_t)src * nx, Uin, A, T, buf, buf + nx,
                  buf + 2 * nx, act);
    }
    free(buf);
    free(T);
  }
}

/* One timestep; returns the buffer holding U^{t+1} (0 -> U0, 1 -> U1). */
void oracle_step(int nx, int ny, int nz, int F, int n_inner, const double* cbase, int shift,
                 const double* Uin, double* Uout, double* A) {
  oracle_physics(nx, ny, nz, n_inner, cbase, shift, Uin, A);
  oracle_jacobi(nx, ny, nz, F, Uin, Uout);
}

/* Runs `steps` timesteps with per-step shifts; U0 holds the initial state on
 * entry and the final state on exit (U1 is scratch). */
void oracle_run(int nx, int ny, int nz, int F, int n_inner, const double* cbase,
                const int* shifts, int steps, double* U0, double* U1, double* A) {
  double* cur = U0;
  double* nxt = U1;
  for (int s = 0; s < steps; ++s) {
    oracle_step(nx, ny, nz, F, n_inner, cbase, shifts[s], cur, nxt, A);
    double* t = cur;
    cur = nxt;
    nxt = t;
  }
  if (cur != U0) memcpy(U0, cur, sizeof(double) * (size_t)F * nz * ny * nx);
}

/* Sum of physics trips over a rectangle of the shifted field (checks
 * physics_work totals).  */
int64_t oracle_trips(int nx, int ny, int nz, const double* cbase, int shift, int x0, int x1,
                     int y0, int y1) {
  int64_t s = 0;
  shift %= ny;
  for (int y = y0; y < y1; ++y)
    for (int x = x0; x < x1; ++x) {
      const int src = (y - shift + ny) % ny;
      int t = (int)floor((double)nz * cbase[(int64_t)src * nx + x]) - 1;
      s += t > 0 ? t : 0;
    }
  return s;
}

/* thread count of the OpenMP loops (torchrun exports OMP_NUM_THREADS=1) */
#ifdef _OPENMP
#include <omp.h>
#endif
int oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}
