/* rhosolve-b200 ORACLE -- test infrastructure only.
 *
 * A plain-C restatement of the reference rhosolve hot-path kernels, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * CHECKER for the CUDA library.  Nothing under paper_1504_06768_b200/ links,
 * loads or calls this file.
 *
 * Restated (reference file:line):
 *   orc_csr_matvec   kernels/_ckernels.pyx:34-50
 *   orc_lower_solve  kernels/_ckernels.pyx:53-67
 *   orc_upper_solve  kernels/_ckernels.pyx:70-85
 *   orc_factorize    kernels/_ckernels.pyx:144-385 (binary-heap left-looking LU)
 *   orc_rcm          ordering.py:62-118 (queue BFS, (deg, idx) neighbour order)
 *   orc_liouvillian  liouville.py:54-77 via sparse.kron/add/matmul
 *                    (sparse.py:77-97, 202-265) as a chain of sorted merges
 * Complex products: the Cython kernels use the plain two-rounding formula
 * (CYTHON_CCOMPLEX=0, -ffp-contract=off: setup.py:13-27); numpy's array loop
 * (kron, add scaling) uses fma(ar,br,-(ai*bi)) / fma(ar,bi,ai*br) on x86-64
 * FMA hosts, and numpy scalars (matmul) use the plain form.  Compile with
 * -ffp-contract=off.
 *
 * Parity pin: tests/golden/*.npz generated from the reference itself
 * (tests/golden/make_golden.py) -- see tests/test_oracle_golden.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cx;

static inline cx cx_mul_plain(cx a, cx b) {
  cx r;
  r.re = a.re * b.re - a.im * b.im;
  r.im = a.re * b.im + a.im * b.re;
  return r;
}
static inline cx cx_mul_np(cx a, cx b) {
  cx r;
  r.re = fma(a.re, b.re, -(a.im * b.im));
  r.im = fma(a.re, b.im, a.im * b.re);
  return r;
}
static inline cx cx_add(cx a, cx b) {
  cx r = {a.re + b.re, a.im + b.im};
  return r;
}
static inline cx cx_sub(cx a, cx b) {
  cx r = {a.re - b.re, a.im - b.im};
  return r;
}
static inline double cx_abs1(cx z) { return fabs(z.re) + fabs(z.im); }
static inline cx cx_recip(cx z) {
  const double d = 1.0 / (z.re * z.re + z.im * z.im);
  cx r = {z.re * d, -z.im * d};
  return r;
}
static inline int cx_zero(cx z) { return z.re == 0.0 && z.im == 0.0; }

/* ------------------------------------------------------------- SpMV ---- */
void orc_csr_matvec(int64_t n, const int64_t* rp, const int64_t* ci, const cx* v,
                    const cx* x, cx* y) {
  for (int64_t r = 0; r < n; ++r) {
    cx s = {0.0, 0.0};
    if (rp[r] < rp[r + 1]) {
      s = cx_mul_plain(v[rp[r]], x[ci[rp[r]]]);
      for (int64_t p = rp[r] + 1; p < rp[r + 1]; ++p)
        s = cx_add(s, cx_mul_plain(v[p], x[ci[p]]));
    }
    y[r] = s;
  }
}

/* ------------------------------------------------ triangular solves ---- */
void orc_lower_solve(int64_t n, const int64_t* Lp, const int64_t* Li, const cx* Lx, cx* y) {
  for (int64_t c = 0; c < n; ++c) {
    const cx yc = y[c];
    for (int64_t p = Lp[c] + 1; p < Lp[c + 1]; ++p)
      y[Li[p]] = cx_sub(y[Li[p]], cx_mul_plain(Lx[p], yc));
  }
}

void orc_upper_solve(int64_t n, const int64_t* Up, const int64_t* Ui, const cx* Ux, cx* y) {
  for (int64_t c = n - 1; c >= 0; --c) {
    const int64_t last = Up[c + 1] - 1;
    const cx xc = cx_mul_plain(y[c], cx_recip(Ux[last]));
    y[c] = xc;
    for (int64_t p = Up[c]; p < last; ++p) y[Ui[p]] = cx_sub(y[Ui[p]], cx_mul_plain(Ux[p], xc));
  }
}

/* ---------------------------------------------------- factorization ---- */
typedef struct {
  double mag;
  int64_t dom, idx, tag;
} cand_t;

static int cand_cmp(const void* pa, const void* pb) {
  const cand_t* a = (const cand_t*)pa;
  const cand_t* b = (const cand_t*)pb;
  if (a->mag != b->mag) return a->mag > b->mag ? -1 : 1; /* larger magnitude first */
  if (a->dom != b->dom) return a->dom < b->dom ? -1 : 1; /* U before L */
  if (a->idx != b->idx) return a->idx < b->idx ? -1 : 1;
  return 0;
}

/* min-heap of pivotal column indices */
static void heap_push(int64_t* h, int64_t* hn, int64_t v) {
  int64_t i = (*hn)++;
  h[i] = v;
  while (i > 0) {
    const int64_t up = (i - 1) / 2;
    if (h[up] <= h[i]) break;
    const int64_t t = h[up];
    h[up] = h[i];
    h[i] = t;
    i = up;
  }
}
static int64_t heap_pop(int64_t* h, int64_t* hn) {
  const int64_t top = h[0];
  const int64_t last = --(*hn);
  h[0] = h[last];
  int64_t i = 0;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= last) break;
    if (c + 1 < last && h[c + 1] < h[c]) ++c;
    if (h[i] <= h[c]) break;
    const int64_t t = h[i];
    h[i] = h[c];
    h[c] = t;
    i = c;
  }
  return top;
}

typedef struct {
  int64_t *Lp, *Li, *Up, *Ui, *pinv;
  cx *Lx, *Ux;
  int64_t lnnz, unnz, fail_col;
} orc_factors;

static int grow(int64_t** I, cx** X, int64_t* cap, int64_t need) {
  if (need <= *cap) return 0;
  int64_t nc = *cap * 2 > need ? *cap * 2 : need;
  int64_t* ni = (int64_t*)realloc(*I, sizeof(int64_t) * nc);
  if (!ni) return -1;
  *I = ni;
  cx* nx = (cx*)realloc(*X, sizeof(cx) * nc);
  if (!nx) return -1;
  *X = nx;
  *cap = nc;
  return 0;
}

int orc_factorize_opts(int64_t n, const int64_t* Ap, const int64_t* Ai, const cx* Ax,
                       const int64_t* q, double drop_tol, int64_t fill_cap, const double* rn,
                       double pivot_floor, int early_drop, int64_t* nfloor, orc_factors* out);

/* Returns 0 and fills *out (caller frees with orc_free_factors); -1 on OOM. */
int orc_factorize(int64_t n, const int64_t* Ap, const int64_t* Ai, const cx* Ax,
                  const int64_t* q, double drop_tol, int64_t fill_cap, const double* rn,
                  orc_factors* out) {
  return orc_factorize_opts(n, Ap, Ai, Ax, q, drop_tol, fill_cap, rn, 0.0, 0, 0, out);
}

/* The reference factorization (_ckernels.pyx:144-385) plus TWO opt-in
 * extensions the reference does not have (the checker of rs_factorize_opts;
 * both off = the reference algorithm unchanged):
 *   pivot_floor > 0: a column without a usable pivot takes the real value
 *     pivot_floor on the lowest non-pivotal row of its pattern (what the
 *     reference's tie rule selects among all-zero candidates) or, when the
 *     pattern has no such row, on the lowest row not yet pivotal;
 *   early_drop: a U entry that the drop rule is going to discard anyway
 *     (|x| < drop_tol * rownorm when its column is reached) is discarded at
 *     once, WITHOUT eliminating with it -- Saad's ILUT rule; the reference
 *     eliminates first and drops at the end of the column. */
int orc_factorize_opts(int64_t n, const int64_t* Ap, const int64_t* Ai, const cx* Ax,
                       const int64_t* q, double drop_tol, int64_t fill_cap, const double* rn,
                       double pivot_floor, int early_drop, int64_t* nfloor, orc_factors* out) {
  int64_t nnzA = Ap[n];
  int64_t capL = 4 * nnzA > 2 * n ? 4 * nnzA : 2 * n;
  if (capL < 16) capL = 16;
  int64_t capU = capL;
  memset(out, 0, sizeof(*out));
  out->Lp = (int64_t*)calloc(n + 1, sizeof(int64_t));
  out->Up = (int64_t*)calloc(n + 1, sizeof(int64_t));
  out->Li = (int64_t*)malloc(sizeof(int64_t) * capL);
  out->Lx = (cx*)malloc(sizeof(cx) * capL);
  out->Ui = (int64_t*)malloc(sizeof(int64_t) * capU);
  out->Ux = (cx*)malloc(sizeof(cx) * capU);
  out->pinv = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  int64_t* prow = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  cx* x = (cx*)calloc(n ? n : 1, sizeof(cx));
  int64_t* mark = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  int64_t* pat = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  int64_t* heap = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  int64_t* ur = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  cx* uv = (cx*)malloc(sizeof(cx) * (n ? n : 1));
  int64_t* lr = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  unsigned char* uk = (unsigned char*)malloc(n ? n : 1);
  unsigned char* lk = (unsigned char*)malloc(n ? n : 1);
  cand_t* cands = (cand_t*)malloc(sizeof(cand_t) * (n ? n : 1));
  if (!out->Lp || !out->Up || !out->Li || !out->Lx || !out->Ui || !out->Ux || !out->pinv ||
      !prow || !x || !mark || !pat || !heap || !ur || !uv || !lr || !uk || !lk || !cands)
    return -1;
  for (int64_t i = 0; i < n; ++i) {
    out->pinv[i] = -1;
    prow[i] = -1;
    mark[i] = -1;
  }
  int64_t lnnz = 0, unnz = 0;
  out->fail_col = -1;
  for (int64_t k = 0; k < n; ++k) {
    const int64_t j = q ? q[k] : k;
    int64_t np_ = 0, hn = 0;
    for (int64_t p = Ap[j]; p < Ap[j + 1]; ++p) {
      const int64_t i = Ai[p];
      x[i] = Ax[p];
      mark[i] = k;
      pat[np_++] = i;
      if (out->pinv[i] >= 0) heap_push(heap, &hn, out->pinv[i]);
    }
    int64_t nu = 0;
    while (hn > 0) {
      const int64_t c = heap_pop(heap, &hn);
      const cx xc = x[prow[c]];
      if (early_drop && drop_tol > 0.0 && cx_abs1(xc) < drop_tol * rn[prow[c]]) continue;
      ur[nu] = c;
      uv[nu] = xc;
      ++nu;
      for (int64_t p = out->Lp[c] + 1; p < out->Lp[c + 1]; ++p) {
        const int64_t i = out->Li[p];
        if (mark[i] != k) {
          mark[i] = k;
          x[i].re = 0.0;
          x[i].im = 0.0;
          pat[np_++] = i;
          if (out->pinv[i] >= 0) heap_push(heap, &hn, out->pinv[i]);
        }
        x[i] = cx_sub(x[i], cx_mul_plain(out->Lx[p], xc));
      }
    }
    double best = -1.0;
    int64_t ipiv = -1, nl = 0;
    for (int64_t t = 0; t < np_; ++t) {
      const int64_t i = pat[t];
      if (out->pinv[i] >= 0) continue;
      lr[nl++] = i;
      const double m = cx_abs1(x[i]);
      if (m > best || (m == best && i < ipiv)) {
        best = m;
        ipiv = i;
      }
    }
    if (ipiv < 0 || best == 0.0) {
      if (!(pivot_floor > 0.0)) {
        out->fail_col = k;
        break;
      }
      if (ipiv < 0) {
        for (int64_t i = 0; i < n; ++i)
          if (out->pinv[i] < 0) {
            ipiv = i;
            break;
          }
        mark[ipiv] = k;
        lr[nl++] = ipiv;
      }
      x[ipiv].re = pivot_floor;
      x[ipiv].im = 0.0;
      if (nfloor) ++*nfloor;
    }
    const cx piv = x[ipiv];
    int64_t ku = 0, kl = 0;
    for (int64_t t = 0; t < nu; ++t) {
      uk[t] = !(drop_tol > 0.0 && cx_abs1(uv[t]) < drop_tol * rn[prow[ur[t]]]);
      ku += uk[t];
    }
    for (int64_t t = 0; t < nl; ++t) {
      const int64_t i = lr[t];
      lk[t] = (i != ipiv) && !(drop_tol > 0.0 && cx_abs1(x[i]) < drop_tol * rn[i]);
      kl += lk[t];
    }
    if (fill_cap >= 0 && ku + kl + 2 > fill_cap && ku + kl > 0) {
      int64_t allowed = fill_cap - 2 < 0 ? 0 : fill_cap - 2;
      int64_t nc = 0;
      for (int64_t t = 0; t < nu; ++t)
        if (uk[t]) {
          cand_t c = {cx_abs1(uv[t]), 0, ur[t], t};
          cands[nc++] = c;
          uk[t] = 0;
        }
      for (int64_t t = 0; t < nl; ++t)
        if (lk[t]) {
          cand_t c = {cx_abs1(x[lr[t]]), 1, lr[t], t};
          cands[nc++] = c;
          lk[t] = 0;
        }
      qsort(cands, (size_t)nc, sizeof(cand_t), cand_cmp);
      if (allowed > nc) allowed = nc;
      ku = kl = 0;
      for (int64_t t = 0; t < allowed; ++t) {
        if (cands[t].dom == 0) {
          uk[cands[t].tag] = 1;
          ++ku;
        } else {
          lk[cands[t].tag] = 1;
          ++kl;
        }
      }
    }
    if (grow(&out->Ui, &out->Ux, &capU, unnz + ku + 1)) return -1;
    for (int64_t t = 0; t < nu; ++t)
      if (uk[t]) {
        out->Ui[unnz] = ur[t];
        out->Ux[unnz] = uv[t];
        ++unnz;
      }
    out->Ui[unnz] = k;
    out->Ux[unnz] = piv;
    ++unnz;
    out->Up[k + 1] = unnz;
    const cx rp = cx_recip(piv);
    if (grow(&out->Li, &out->Lx, &capL, lnnz + kl + 1)) return -1;
    out->Li[lnnz] = ipiv;
    out->Lx[lnnz].re = 1.0;
    out->Lx[lnnz].im = 0.0;
    ++lnnz;
    for (int64_t t = 0; t < nl; ++t)
      if (lk[t]) {
        out->Li[lnnz] = lr[t];
        out->Lx[lnnz] = cx_mul_plain(x[lr[t]], rp);
        ++lnnz;
      }
    out->Lp[k + 1] = lnnz;
    out->pinv[ipiv] = k;
    prow[k] = ipiv;
  }
  if (out->fail_col < 0)
    for (int64_t t = 0; t < lnnz; ++t) out->Li[t] = out->pinv[out->Li[t]];
  out->lnnz = lnnz;
  out->unnz = unnz;
  free(prow);
  free(x);
  free(mark);
  free(pat);
  free(heap);
  free(ur);
  free(uv);
  free(lr);
  free(uk);
  free(lk);
  free(cands);
  return 0;
}

void orc_free_factors(orc_factors* f) {
  free(f->Lp);
  free(f->Li);
  free(f->Lx);
  free(f->Up);
  free(f->Ui);
  free(f->Ux);
  free(f->pinv);
  memset(f, 0, sizeof(*f));
}

/* ------------------------------------------------------------- RCM ------ */
/* order_out[k] = original index at CM position k (NOT yet reversed). */
int orc_rcm(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* order_out) {
  /* symmetric adjacency without self loops, deduplicated */
  int64_t* deg = (int64_t*)calloc(n + 1, sizeof(int64_t));
  int64_t nnz = rp[n];
  int64_t* tr = (int64_t*)calloc(n + 1, sizeof(int64_t)); /* transpose pointers */
  int64_t* tc = (int64_t*)malloc(sizeof(int64_t) * (nnz ? nnz : 1));
  if (!deg || !tr || !tc) return -1;
  for (int64_t p = 0; p < nnz; ++p) tr[ci[p] + 1]++;
  for (int64_t i = 0; i < n; ++i) tr[i + 1] += tr[i];
  {
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
    memcpy(fill, tr, sizeof(int64_t) * n);
    for (int64_t r = 0; r < n; ++r)
      for (int64_t p = rp[r]; p < rp[r + 1]; ++p) tc[fill[ci[p]]++] = r; /* ascending r */
    free(fill);
  }
  int64_t* ap = (int64_t*)calloc(n + 1, sizeof(int64_t));
  int64_t* aj = (int64_t*)malloc(sizeof(int64_t) * (2 * nnz + 1));
  if (!ap || !aj) return -1;
  for (int64_t i = 0; i < n; ++i) {
    int64_t a = rp[i], ae = rp[i + 1], b = tr[i], be = tr[i + 1], last = -1;
    ap[i + 1] = ap[i];
    while (a < ae || b < be) {
      int64_t c;
      if (b >= be || (a < ae && ci[a] <= tc[b])) c = ci[a++];
      else c = tc[b++];
      if (c == i || c == last) continue;
      last = c;
      aj[ap[i + 1]++] = c;
    }
  }
  for (int64_t i = 0; i < n; ++i) deg[i] = ap[i + 1] - ap[i];
  /* sort each neighbour list by (deg, idx): insertion sort */
  for (int64_t i = 0; i < n; ++i)
    for (int64_t s = ap[i] + 1; s < ap[i + 1]; ++s) {
      const int64_t u = aj[s];
      int64_t y = s;
      while (y > ap[i]) {
        const int64_t w = aj[y - 1];
        if (deg[w] < deg[u] || (deg[w] == deg[u] && w < u)) break;
        aj[y] = w;
        --y;
      }
      aj[y] = u;
    }
  /* start candidates sorted by (deg, idx): counting sort on degree (stable) */
  int64_t maxd = 0;
  for (int64_t i = 0; i < n; ++i) maxd = deg[i] > maxd ? deg[i] : maxd;
  int64_t* bucket = (int64_t*)calloc(maxd + 2, sizeof(int64_t));
  int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (n ? n : 1));
  unsigned char* seen = (unsigned char*)calloc(n ? n : 1, 1);
  if (!bucket || !cand || !seen) return -1;
  for (int64_t i = 0; i < n; ++i) bucket[deg[i] + 1]++;
  for (int64_t d = 0; d <= maxd; ++d) bucket[d + 1] += bucket[d];
  for (int64_t i = 0; i < n; ++i) cand[bucket[deg[i]]++] = i;
  int64_t head = 0, tail = 0, ci_pos = 0;
  while (tail < n) {
    while (seen[cand[ci_pos]]) ++ci_pos;
    const int64_t s = cand[ci_pos];
    seen[s] = 1;
    order_out[tail++] = s;
    while (head < tail) {
      const int64_t v = order_out[head++];
      for (int64_t e = ap[v]; e < ap[v + 1]; ++e) {
        const int64_t u = aj[e];
        if (!seen[u]) {
          seen[u] = 1;
          order_out[tail++] = u;
        }
      }
    }
  }
  free(deg);
  free(tr);
  free(tc);
  free(ap);
  free(aj);
  free(bucket);
  free(cand);
  free(seen);
  return 0;
}
