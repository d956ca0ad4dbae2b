/*
 * qtnh_oracle.c -- CPU restatement of the reference hot path. TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg as the checker; never part of the product path.
 *
 * Pinned against the reference itself (oracle/_ref/libqtnh_ref.so, built from
 * the unmodified headers) and against the reference's own known-answer tests,
 * see tests/test_oracle.py. Every function cites the reference it restates.
 *
 * Tensors are global row-major vectors of interleaved (re, im) doubles.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- RNG: common.hpp:83-146 ------------------------------------------------- */
static uint64_t mix64(uint64_t x) { /* splitmix64 finaliser, common.hpp:84-89 */
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t qo_hash_counter(uint64_t seed, uint64_t k0, uint64_t k1, uint64_t k2) { /* :93-100 */
  uint64_t h = mix64(seed ^ 0x243f6a8885a308d3ULL);
  h = mix64(h ^ k0);
  h = mix64(h ^ k1);
  return mix64(h ^ k2);
}

double qo_u64_to_unit(uint64_t u) { return (double)(u >> 11) * 0x1.0p-53; } /* :103-105 */

/* Sequential Rng(seed).next_complex_normal() x count (common.hpp:109-140):
 * Box-Muller pairs, cos branch first, the sin branch is the spare. */
void qo_rng_complex_normals(uint64_t seed, int64_t count, double* out) {
  uint64_t state = mix64(seed);
  int have_spare = 0;
  double spare = 0.0;
  for (int64_t i = 0; i < 2 * count; ++i) {
    double v;
    if (have_spare) {
      have_spare = 0;
      v = spare;
    } else {
      double u1 = 0.0, u2;
      while (u1 <= 1e-300) {
        state = mix64(state);
        u1 = qo_u64_to_unit(state);
      }
      state = mix64(state);
      u2 = qo_u64_to_unit(state);
      double r = sqrt(-2.0 * log(u1));
      double a = 6.283185307179586476925286766559 * u2;
      spare = r * sin(a);
      have_spare = 1;
      v = r * cos(a);
    }
    out[i] = v;
  }
}

/* Counter-based complex normal for element j (SURVEY.md section 8(d), C0/C2
 * inputs): u1 from hash_counter(seed, j, 0, k2) with k2 = 0, 1, ... redrawn while
 * u1 <= 1e-300 (the guard of common.hpp:127), u2 from hash_counter(seed, j, 1, 0);
 * value = r (cos a, sin a). Independent per element, so shards generate alone. */
void qo_counter_normals(uint64_t seed, int64_t start, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) {
    uint64_t j = (uint64_t)(start + i);
    double u1 = 0.0;
    for (uint64_t k2 = 0; u1 <= 1e-300; ++k2) u1 = qo_u64_to_unit(qo_hash_counter(seed, j, 0, k2));
    double u2 = qo_u64_to_unit(qo_hash_counter(seed, j, 1, 0));
    double r = sqrt(-2.0 * log(u1));
    double a = 6.283185307179586476925286766559 * u2;
    out[2 * i] = r * cos(a);
    out[2 * i + 1] = r * sin(a);
  }
}

/* The same generator at arbitrary global element indices (a strided slice of a
 * sharded input, e.g. bench.py's reference sample of the C1 operand A). */
void qo_counter_normals_at(uint64_t seed, const int64_t* idx, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) qo_counter_normals(seed, idx[i], 1, out + 2 * i);
}

/* ---- permutation: ops.hpp:27-49 via remap.hpp:56-161 ------------------------
 * result index p is source index perm[p]. Zero elements (both parts == 0.0,
 * either sign) are skipped by the reference's remap and the destination starts
 * zeroed (remap.hpp:69-70, :125-127), so they come out as (+0, +0). */
int qo_permute(int n, const int64_t* dims, const double* in, const int* perm, double* out) {
  int64_t st_in[64], nd[64], cnt[64];
  if (n > 64) return 1;
  int64_t total = 1;
  for (int i = 0; i < n; ++i) total *= dims[i];
  {
    int64_t s = 1;
    for (int i = n - 1; i >= 0; --i) {
      st_in[i] = s;
      s *= dims[i];
    }
  }
  for (int p = 0; p < n; ++p) {
    nd[p] = dims[perm[p]];
    cnt[p] = 0;
  }
  int64_t src = 0;
  for (int64_t f = 0; f < total; ++f) {
    double re = in[2 * src], im = in[2 * src + 1];
    if (re == 0.0 && im == 0.0) re = im = 0.0;
    out[2 * f] = re;
    out[2 * f + 1] = im;
    for (int p = n - 1; p >= 0; --p) { /* odometer over the output, row-major */
      src += st_in[perm[p]];
      if (++cnt[p] < nd[p]) break;
      src -= st_in[perm[p]] * nd[p];
      cnt[p] = 0;
    }
  }
  return 0;
}

/* ---- contraction: SPEC.md:361-369 (brute-force loop oracle) ------
 * C[open(a) then open(b)] = sum over the paired indices a[a_pos[i]] == b[b_pos[i]]
 * (SPEC.md:408). */
int qo_contract(int na, const int64_t* da, const double* a, int nb, const int64_t* db,
                const double* b, int np, const int* apos, const int* bpos, double* c) {
  int ca[64] = {0}, cb[64] = {0};
  int ao[64], bo[64], nao = 0, nbo = 0;
  int64_t sa[64], sb[64];
  if (na > 64 || nb > 64) return 1;
  for (int i = 0; i < np; ++i) {
    ca[apos[i]] = 1;
    cb[bpos[i]] = 1;
  }
  for (int i = 0; i < na; ++i)
    if (!ca[i]) ao[nao++] = i;
  for (int i = 0; i < nb; ++i)
    if (!cb[i]) bo[nbo++] = i;
  int64_t s = 1;
  for (int i = na - 1; i >= 0; --i) { sa[i] = s; s *= da[i]; }
  s = 1;
  for (int i = nb - 1; i >= 0; --i) { sb[i] = s; s *= db[i]; }
  int64_t M = 1, N = 1, K = 1;
  for (int i = 0; i < nao; ++i) M *= da[ao[i]];
  for (int i = 0; i < nbo; ++i) N *= db[bo[i]];
  for (int i = 0; i < np; ++i) K *= da[apos[i]];
  int64_t* aoff = malloc(sizeof(int64_t) * M);
  int64_t* boff = malloc(sizeof(int64_t) * N);
  int64_t* akoff = malloc(sizeof(int64_t) * K);
  int64_t* bkoff = malloc(sizeof(int64_t) * K);
  for (int64_t m = 0; m < M; ++m) {
    int64_t r = m, off = 0;
    for (int i = nao - 1; i >= 0; --i) { off += (r % da[ao[i]]) * sa[ao[i]]; r /= da[ao[i]]; }
    aoff[m] = off;
  }
  for (int64_t nn = 0; nn < N; ++nn) {
    int64_t r = nn, off = 0;
    for (int i = nbo - 1; i >= 0; --i) { off += (r % db[bo[i]]) * sb[bo[i]]; r /= db[bo[i]]; }
    boff[nn] = off;
  }
  for (int64_t k = 0; k < K; ++k) {
    int64_t r = k, oa = 0, ob = 0;
    for (int i = np - 1; i >= 0; --i) {
      int64_t ci = r % da[apos[i]];
      r /= da[apos[i]];
      oa += ci * sa[apos[i]];
      ob += ci * sb[bpos[i]];
    }
    akoff[k] = oa;
    bkoff[k] = ob;
  }
  for (int64_t m = 0; m < M; ++m)
    for (int64_t nn = 0; nn < N; ++nn) {
      double re = 0.0, im = 0.0;
      for (int64_t k = 0; k < K; ++k) {
        const double* x = a + 2 * (aoff[m] + akoff[k]);
        const double* y = b + 2 * (boff[nn] + bkoff[k]);
        re += x[0] * y[0] - x[1] * y[1];
        im += x[0] * y[1] + x[1] * y[0];
      }
      c[2 * (m * N + nn)] = re;
      c[2 * (m * N + nn) + 1] = im;
    }
  free(aoff);
  free(boff);
  free(akoff);
  free(bkoff);
  return 0;
}

/* ---- gate application --------------------------------------------------------
 * Values of contract(state, gate) + permute back (the reference path of a gate
 * tensor, PAPER.md III-E-1): y_f = G x_f on every fiber. gate is D x D row-major,
 * row = output, targets[0] most significant; diagonal: only D entries. */
int qo_gate(int n, const int64_t* dims, double* psi, int k, const int* targets, const double* gate,
            int diagonal) {
  int64_t st[64], total = 1, D = 1;
  int is_t[64] = {0};
  if (n > 64 || k > 16) return 1;
  for (int i = n - 1; i >= 0; --i) { st[i] = total; total *= dims[i]; }
  for (int j = 0; j < k; ++j) { is_t[targets[j]] = 1; D *= dims[targets[j]]; }
  int64_t* toff = malloc(sizeof(int64_t) * D);
  for (int64_t d = 0; d < D; ++d) {
    int64_t r = d, off = 0;
    for (int j = k - 1; j >= 0; --j) { off += (r % dims[targets[j]]) * st[targets[j]]; r /= dims[targets[j]]; }
    toff[d] = off;
  }
  double* x = malloc(sizeof(double) * 2 * D);
  for (int64_t e = 0; e < total; ++e) {
    /* fiber bases: elements whose target coordinates are all zero */
    int64_t r = e;
    int zero = 1;
    for (int i = n - 1; i >= 0 && zero; --i) {
      if (is_t[i] && (r % dims[i]) != 0) zero = 0;
      r /= dims[i];
    }
    if (!zero) continue;
    for (int64_t d = 0; d < D; ++d) {
      x[2 * d] = psi[2 * (e + toff[d])];
      x[2 * d + 1] = psi[2 * (e + toff[d]) + 1];
    }
    for (int64_t i = 0; i < D; ++i) {
      double re = 0.0, im = 0.0;
      if (diagonal) {
        re = gate[2 * i] * x[2 * i] - gate[2 * i + 1] * x[2 * i + 1];
        im = gate[2 * i] * x[2 * i + 1] + gate[2 * i + 1] * x[2 * i];
      } else {
        for (int64_t d = 0; d < D; ++d) {
          const double* g = gate + 2 * (i * D + d);
          re += g[0] * x[2 * d] - g[1] * x[2 * d + 1];
          im += g[0] * x[2 * d + 1] + g[1] * x[2 * d];
        }
      }
      psi[2 * (e + toff[i])] = re;
      psi[2 * (e + toff[i]) + 1] = im;
    }
  }
  free(x);
  free(toff);
  return 0;
}

/* ---- QFT circuit -------------------------
 * For j = 0..n-1: H on qubit j, then CP(2 pi / 2^m) on (j+m-1, j) for
 * m = 2..n-j; then SWAP(j, n-1-j) for j < n/2 when `swaps`. Qubit 0 is the most
 * significant (leftmost) index. In place on psi (2^n amplitudes). */
int qo_qft(int n, double* psi, int swaps) {
  int64_t dims[64];
  if (n > 64) return 1;
  for (int i = 0; i < n; ++i) dims[i] = 2;
  const double r = 1.0 / sqrt(2.0);
  const double h[8] = {r, 0, r, 0, r, 0, -r, 0};
  for (int j = 0; j < n; ++j) {
    int t1[1] = {j};
    qo_gate(n, dims, psi, 1, t1, h, 0);
    for (int m = 2; m <= n - j; ++m) {
      double th = 2.0 * 3.14159265358979323846 / ldexp(1.0, m);
      double d[8] = {1, 0, 1, 0, 1, 0, cos(th), sin(th)};
      int t2[2] = {j + m - 1, j};
      qo_gate(n, dims, psi, 2, t2, d, 1);
    }
  }
  if (swaps) {
    int64_t total = (int64_t)1 << n;
    double* tmp = malloc(sizeof(double) * 2 * total);
    int perm[64];
    for (int j = 0; j < n / 2; ++j) {
      for (int p = 0; p < n; ++p) perm[p] = p;
      perm[j] = n - 1 - j;
      perm[n - 1 - j] = j;
      qo_permute(n, dims, psi, perm, tmp);
      memcpy(psi, tmp, sizeof(double) * 2 * total);
    }
    free(tmp);
  }
  return 0;
}
