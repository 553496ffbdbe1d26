/*
 * sta_oracle.c -- the CPU oracle (TEST INFRASTRUCTURE ONLY; see sta_oracle.h).
 *
 * Plain single-thread C, fp64 arithmetic, written step by step after
 * SURVEY.md §8(c) O1-O9 with the conventions of SPEC.md:371-532.  No blocking,
 * no fusion, no reordering: each step is a loop a reader can check against the
 * cited passage.  Pinned by tests/test_oracle_*.py (hand examples, closed
 * forms, brute force); see DESIGN.md §4 for the pin list.
 */
#include "sta_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define INF HUGE_VAL
/* quantity index q = el*2 + rf with el: 0 early, 1 late; rf: 0 rise, 1 fall */
#define Q(el, rf) ((el) * 2 + (rf))

/* ---------------------------------------------------------------- O6: LUT */
/* bilinear inside the grid, linear extrapolation from the
 * boundary cell outside (tx, ty not clamped); 1-D tables interpolate on their
 * single axis; a 1x1 table is a constant.  Segment: i = clamp(ub(x,s)-1, 0,
 * n-2) (SURVEY.md §8(c) reading #4). */
static uint32_t seg(const float* x, uint32_t n, double s) {
  uint32_t ub = 0;                       /* upper_bound: first x[k] > s */
  while (ub < n && (double)x[ub] <= s) ub++;
  long i = (long)ub - 1;
  if (i < 0) i = 0;
  if (i > (long)n - 2) i = (long)n - 2;
  return (uint32_t)i;
}

double orc_lut(uint32_t n1, uint32_t n2, const float* tab, double s, double c) {
  const float* x = tab;
  const float* y = tab + n1;
  const float* v = tab + n1 + n2;       /* v[i*n2 + j] */
  if (n1 == 1 && n2 == 1) return v[0];
  if (n1 == 1) {
    uint32_t j = seg(y, n2, c);
    double ty = (c - y[j]) / ((double)y[j + 1] - y[j]);
    return (1 - ty) * v[j] + ty * v[j + 1];
  }
  if (n2 == 1) {
    uint32_t i = seg(x, n1, s);
    double tx = (s - x[i]) / ((double)x[i + 1] - x[i]);
    return (1 - tx) * v[i] + tx * v[i + 1];
  }
  uint32_t i = seg(x, n1, s), j = seg(y, n2, c);
  double tx = (s - x[i]) / ((double)x[i + 1] - x[i]);
  double ty = (c - y[j]) / ((double)y[j + 1] - y[j]);
  double v00 = v[i * n2 + j], v10 = v[(i + 1) * n2 + j];
  double v01 = v[i * n2 + j + 1], v11 = v[(i + 1) * n2 + j + 1];
  return (1 - tx) * (1 - ty) * v00 + tx * (1 - ty) * v10 + (1 - tx) * ty * v01 + tx * ty * v11;
}

static double lut_id(const orc_design* d, uint32_t t, double s, double c) {
  return orc_lut(d->tab_n1[t], d->tab_n2[t], d->tab_data + d->tab_off[t], s, c);
}

/* ---------------------------------------------------------------- O1: arcs */
/* Net arcs: driver -> each sink, nets in order, sinks in order; then cell
 * arcs in input order.  Check arcs are not edges
 * (SPEC.md:223). */
typedef struct {
  uint32_t E, En;        /* total arcs, net arcs */
  uint32_t* from;
  uint32_t* to;
  uint32_t* cell;        /* cell arc index for id >= En */
  uint32_t *fi_ptr, *fi; /* fan-in CSR of arc ids (canonical order) */
  uint32_t *fo_ptr, *fo; /* fan-out CSR */
} arcs_t;

static void free_arcs(arcs_t* g) {
  free(g->from); free(g->to); free(g->cell);
  free(g->fi_ptr); free(g->fi); free(g->fo_ptr); free(g->fo);
}

/* off (optional, per canonical arc id): O16's disabled arcs, left out */
static int build_arcs_off(const orc_design* d, arcs_t* g, const uint8_t* off) {
  uint32_t P = d->num_pins;
  uint32_t En = d->net_ptr[d->num_nets] - d->num_nets;
  uint32_t E = En + d->num_arcs;
  g->E = E; g->En = En;
  g->from = malloc(sizeof(uint32_t) * (E + 1));
  g->to = malloc(sizeof(uint32_t) * (E + 1));
  g->cell = malloc(sizeof(uint32_t) * (E + 1));
  g->fi_ptr = calloc(P + 1, sizeof(uint32_t));
  g->fo_ptr = calloc(P + 1, sizeof(uint32_t));
  g->fi = malloc(sizeof(uint32_t) * (E + 1));
  g->fo = malloc(sizeof(uint32_t) * (E + 1));
  if (!g->from || !g->to || !g->cell || !g->fi_ptr || !g->fo_ptr || !g->fi || !g->fo) return 2;
  uint32_t k = 0, id = 0;
  for (uint32_t n = 0; n < d->num_nets; n++) {
    uint32_t drv = d->net_pins[d->net_ptr[n]];
    for (uint32_t j = d->net_ptr[n] + 1; j < d->net_ptr[n + 1]; j++, id++) {
      if (off && off[id]) continue;
      g->from[k] = drv; g->to[k] = d->net_pins[j]; g->cell[k] = 0; k++;
    }
  }
  g->En = En = k;
  for (uint32_t a = 0; a < d->num_arcs; a++, id++) {
    if (off && off[id]) continue;
    g->from[k] = d->arc_from[a]; g->to[k] = d->arc_to[a]; g->cell[k] = a; k++;
  }
  g->E = E = k;
  for (uint32_t e = 0; e < E; e++) { g->fi_ptr[g->to[e] + 1]++; g->fo_ptr[g->from[e] + 1]++; }
  for (uint32_t p = 0; p < P; p++) { g->fi_ptr[p + 1] += g->fi_ptr[p]; g->fo_ptr[p + 1] += g->fo_ptr[p]; }
  uint32_t* fi_fill = malloc(sizeof(uint32_t) * (P + 1));
  uint32_t* fo_fill = malloc(sizeof(uint32_t) * (P + 1));
  if (!fi_fill || !fo_fill) { free(fi_fill); free(fo_fill); return 2; }
  memcpy(fi_fill, g->fi_ptr, sizeof(uint32_t) * (P + 1));
  memcpy(fo_fill, g->fo_ptr, sizeof(uint32_t) * (P + 1));
  for (uint32_t e = 0; e < E; e++) {
    g->fi[fi_fill[g->to[e]]++] = e;
    g->fo[fo_fill[g->from[e]]++] = e;
  }
  free(fi_fill); free(fo_fill);
  return 0;
}

static int build_arcs(const orc_design* d, arcs_t* g) { return build_arcs_off(d, g, NULL); }

/* ---------------------------------------------------------- O2: levelize */
/* Kahn with a FIFO seeded by in-degree-0 pins in increasing id;
 * level(v) = 0 without fan-in, else 1 + max level over fan-in.  `order`
 * receives the pop order, itself a topological order. */
static int kahn(const orc_design* d, const arcs_t* g, uint32_t* level, uint32_t* order) {
  uint32_t P = d->num_pins;
  uint32_t* indeg = malloc(sizeof(uint32_t) * (P + 1));
  if (!indeg) return 2;
  uint32_t head = 0, tail = 0;
  for (uint32_t p = 0; p < P; p++) {
    indeg[p] = g->fi_ptr[p + 1] - g->fi_ptr[p];
    level[p] = 0;
    if (indeg[p] == 0) order[tail++] = p;
  }
  while (head < tail) {
    uint32_t u = order[head++];
    for (uint32_t k = g->fo_ptr[u]; k < g->fo_ptr[u + 1]; k++) {
      uint32_t v = g->to[g->fo[k]];
      if (level[u] + 1 > level[v]) level[v] = level[u] + 1;
      if (--indeg[v] == 0) order[tail++] = v;
    }
  }
  free(indeg);
  return tail == P ? 0 : 1;
}

int orc_levelize(const orc_design* d, uint32_t* level, uint32_t* perm, uint32_t* num_levels) {
  arcs_t g; memset(&g, 0, sizeof g);
  int st = build_arcs(d, &g);
  uint32_t P = d->num_pins;
  uint32_t* order = malloc(sizeof(uint32_t) * (P + 1));
  if (st || !order) { free_arcs(&g); free(order); return 2; }
  st = kahn(d, &g, level, order);
  free(order);
  free_arcs(&g);
  if (st) return st;
  uint32_t L = 0;
  for (uint32_t p = 0; p < P; p++) if (level[p] + 1 > L) L = level[p] + 1;
  *num_levels = L;
  if (perm) { /* stable counting sort by level: pins of one level in id order */
    uint32_t* start = calloc(L + 1, sizeof(uint32_t));
    if (!start) return 2;
    for (uint32_t p = 0; p < P; p++) start[level[p] + 1]++;
    for (uint32_t l = 0; l < L; l++) start[l + 1] += start[l];
    for (uint32_t p = 0; p < P; p++) perm[start[level[p]]++] = p;
    free(start);
  }
  return 0;
}

/* --------------------------------------------------------------- O3: RC */
/* Per net with RC nodes: node cap C_i = Cw_i + pin cap of
 * the pin at node i (+ its PO load, reading R10); Cdown bottom-up
 * (parent[i] < i); load = Cdown_0; elm_i = elm_parent + R_i * Cdown_i.
 * Nets without RC nodes are lumped: load = sum of the net's pin caps (+ PO
 * loads), every net-arc delay 0. */
void orc_rc(const orc_design* d, double* load, double* elm) {
  uint32_t P = d->num_pins;
  double* po_ld = calloc(P + 1, sizeof(double));
  for (uint32_t k = 0; k < d->n_po; k++) po_ld[d->po_pin[k]] += d->po_load[k];
  for (uint32_t p = 0; p < P; p++) elm[p] = 0.0;
  uint32_t maxn = 1;
  for (uint32_t n = 0; n < d->num_nets; n++) {
    uint32_t m = d->rc_ptr[n + 1] - d->rc_ptr[n];
    if (m > maxn) maxn = m;
  }
  double* cd = malloc(sizeof(double) * maxn);
  double* el = malloc(sizeof(double) * maxn);
  for (uint32_t n = 0; n < d->num_nets; n++) {
    uint32_t b = d->rc_ptr[n], m = d->rc_ptr[n + 1] - b;
    if (m == 0) {
      double c = 0;
      for (uint32_t j = d->net_ptr[n]; j < d->net_ptr[n + 1]; j++) {
        uint32_t p = d->net_pins[j];
        c += d->pin_cap[p] + po_ld[p];
      }
      load[n] = c;
      continue;
    }
    for (uint32_t i = 0; i < m; i++) {
      uint32_t p = d->rc_node_pin[b + i];
      cd[i] = d->rc_cap[b + i] + (p != ORC_NO_PIN ? d->pin_cap[p] + po_ld[p] : 0.0);
    }
    for (uint32_t i = m - 1; i >= 1; i--) cd[d->rc_parent[b + i]] += cd[i];
    load[n] = cd[0];
    el[0] = 0.0;
    for (uint32_t i = 1; i < m; i++) el[i] = el[d->rc_parent[b + i]] + (double)d->rc_res[b + i] * cd[i];
    for (uint32_t i = 1; i < m; i++) {
      uint32_t p = d->rc_node_pin[b + i];
      if (p != ORC_NO_PIN) elm[p] = el[i];
    }
  }
  free(cd); free(el); free(po_ld);
}


/* --------------------------------------------------- O12: Arnoldi net model */
/* "Per-net Lanczos on trees (q = 4) with O(n) tree
 * solves; delay and slew from the ramp response" ("an
 * Arnoldi-based reduced-order model").  The driver node 0 is
 * driven by the ideal source; the unknowns are nodes 1..m-1 with
 * C v' + G v = b u, G the conductance Laplacian.  A = G^-1 C is self-adjoint
 * in <x, y> = sum_i C_i x_i y_i and G^-1 b = 1, so V(s)/U(s) = (I + s A)^-1 1.
 * A x is one tree solve (the RC-tree moment recursion): subtree sums of
 * C_j x_j, then root-path sums of R_a times them. */
static void tree_apply(uint32_t m, const int32_t* parent, const float* res, const double* cap, const double* x,
                       double* y, double* t) {
  t[0] = 0.0;
  for (uint32_t i = 1; i < m; i++) t[i] = cap[i] * x[i];
  for (uint32_t i = m - 1; i >= 1; i--) t[parent[i]] += t[i];
  y[0] = 0.0;
  for (uint32_t i = 1; i < m; i++) y[i] = y[parent[i]] + (double)res[i] * t[i];
}

static double cdot(uint32_t m, const double* cap, const double* x, const double* y) {
  double s = 0.0;
  for (uint32_t i = 1; i < m; i++) s += cap[i] * x[i] * y[i];
  return s;
}

/* cyclic Jacobi eigen-decomposition of the symmetric n x n matrix a (row
 * major, destroyed): eigenvalues in w, eigenvectors in the columns of v */
static void jacobi_eig(uint32_t n, double* a, double* w, double* v) {
  for (uint32_t i = 0; i < n; i++)
    for (uint32_t j = 0; j < n; j++) v[i * n + j] = i == j;
  for (int sweep = 0; sweep < 100; sweep++) {
    double off = 0.0, nrm = 0.0;
    for (uint32_t i = 0; i < n; i++)
      for (uint32_t j = 0; j < n; j++) {
        nrm += a[i * n + j] * a[i * n + j];
        if (i != j) off += a[i * n + j] * a[i * n + j];
      }
    if (off <= 1e-30 * nrm || off == 0.0) break;
    for (uint32_t p = 0; p < n; p++)
      for (uint32_t q = p + 1; q < n; q++) {
        double apq = a[p * n + q];
        if (apq == 0.0) continue;
        double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
        double tt = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double c = 1.0 / sqrt(tt * tt + 1.0), sn = tt * c;
        for (uint32_t k = 0; k < n; k++) {          /* rotate rows / columns p, q */
          double akp = a[k * n + p], akq = a[k * n + q];
          a[k * n + p] = c * akp - sn * akq;
          a[k * n + q] = sn * akp + c * akq;
        }
        for (uint32_t k = 0; k < n; k++) {
          double apk = a[p * n + k], aqk = a[q * n + k];
          a[p * n + k] = c * apk - sn * aqk;
          a[q * n + k] = sn * apk + c * aqk;
        }
        for (uint32_t k = 0; k < n; k++) {
          double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = c * vkp - sn * vkq;
          v[k * n + q] = sn * vkp + c * vkq;
        }
      }
  }
  for (uint32_t i = 0; i < n; i++) w[i] = a[i * n + i];
}

int orc_arnoldi_reduce(uint32_t m, const int32_t* parent, const float* res, const double* cap, uint32_t q,
                       double* lam, double* resid) {
  double ctot = 0.0;
  for (uint32_t i = 1; i < m; i++) ctot += cap[i];
  if (q < 1) q = 1;
  if (m <= 1 || ctot <= 0.0) {               /* no dynamics: the output follows the input */
    lam[0] = 0.0;
    for (uint32_t i = 0; i < m; i++) { resid[(size_t)i * q] = 1.0; for (uint32_t k = 1; k < q; k++) resid[(size_t)i * q + k] = 0.0; }
    return 1;
  }
  double* V = calloc((size_t)(q + 1) * m, sizeof(double));   /* Lanczos vectors, V[j*m + i] */
  double* w = malloc(sizeof(double) * m);
  double* t = malloc(sizeof(double) * m);
  double alpha[16], beta[16];
  /* step 1: v_1 = 1 / ||1||_C */
  for (uint32_t i = 1; i < m; i++) V[i] = 1.0 / sqrt(ctot);
  uint32_t qq = 0;
  for (uint32_t j = 0; j < q; j++) {
    /* step 2: w = A v_j - beta_{j-1} v_{j-1}; alpha_j = <w, v_j>; w -= alpha_j v_j */
    tree_apply(m, parent, res, cap, V + (size_t)j * m, w, t);
    if (j > 0) for (uint32_t i = 1; i < m; i++) w[i] -= beta[j - 1] * V[(size_t)(j - 1) * m + i];
    alpha[j] = cdot(m, cap, w, V + (size_t)j * m);
    for (uint32_t i = 1; i < m; i++) w[i] -= alpha[j] * V[(size_t)j * m + i];
    /* full reorthogonalisation against v_1 .. v_j (twice) */
    for (int pass = 0; pass < 2; pass++)
      for (uint32_t k = 0; k <= j; k++) {
        double c = cdot(m, cap, w, V + (size_t)k * m);
        for (uint32_t i = 1; i < m; i++) w[i] -= c * V[(size_t)k * m + i];
      }
    qq = j + 1;
    beta[j] = sqrt(cdot(m, cap, w, w));
    /* step 3: breakdown (the Krylov space is exhausted) truncates the order */
    if (j + 1 == q || !(beta[j] > 1e-10 * fabs(alpha[j]))) break;
    for (uint32_t i = 1; i < m; i++) V[(size_t)(j + 1) * m + i] = w[i] / beta[j];
  }
  /* step 4: T = tridiag(beta, alpha, beta) = Q diag(lam) Q^T */
  double T[256], Qm[256], ev[16];
  for (uint32_t a = 0; a < qq; a++)
    for (uint32_t b = 0; b < qq; b++)
      T[a * qq + b] = a == b ? alpha[a] : (a + 1 == b ? beta[a] : (b + 1 == a ? beta[b] : 0.0));
  jacobi_eig(qq, T, ev, Qm);
  int stable = 1;
  double lmax = 0.0;
  for (uint32_t k = 0; k < qq; k++) if (ev[k] > lmax) lmax = ev[k];
  for (uint32_t k = 0; k < qq; k++) {
    if (ev[k] < -1e-9 * lmax) stable = 0;     /* a positive pole */
    lam[k] = ev[k] < 0.0 ? 0.0 : ev[k];
  }
  /* step 5: residues H_i(s) = sqrt(Ctot) e_i^T V Q (I + s Lam)^-1 Q^T e_1 */
  for (uint32_t i = 0; i < m; i++)
    for (uint32_t k = 0; k < q; k++) {
      double r = 0.0;
      if (k < qq) {
        if (i == 0) r = k == 0 ? 1.0 : 0.0;    /* the driven root follows the input */
        else {
          for (uint32_t j = 0; j < qq; j++) r += V[(size_t)j * m + i] * Qm[j * qq + k];
          r *= sqrt(ctot) * Qm[0 * qq + k];
        }
      }
      resid[(size_t)i * q + k] = r;
    }
  free(V); free(w); free(t);
  return stable ? (int)qq : -1;
}

/* response of one reduced term 1 / (1 + s lam) to the saturated ramp of
 * duration D (0: a step) at time t */
static double ramp_term(double lam, double D, double t) {
  if (t <= 0.0) return 0.0;
  if (D <= 0.0) return lam > 0.0 ? 1.0 - exp(-t / lam) : 1.0;
  double r1 = lam > 0.0 ? t - lam * (1.0 - exp(-t / lam)) : t;
  double r2 = 0.0;
  if (t > D) r2 = lam > 0.0 ? (t - D) - lam * (1.0 - exp(-(t - D) / lam)) : t - D;
  return (r1 - r2) / D;
}

static double ramp_resp(uint32_t qq, const double* lam, const double* k, double D, double t) {
  double y = 0.0;
  for (uint32_t j = 0; j < qq; j++) y += k[j] * ramp_term(lam[j], D, t);
  return y;
}

/* first time the response reaches theta, by bisection to 1e-6 ps */
static double crossing(uint32_t qq, const double* lam, const double* k, double D, double theta) {
  double lmax = 0.0;
  for (uint32_t j = 0; j < qq; j++) if (lam[j] > lmax) lmax = lam[j];
  double lo = 0.0, hi = D + 50.0 * lmax + 1e-3;
  for (int g = 0; g < 60 && ramp_resp(qq, lam, k, D, hi) < theta; g++) hi *= 2.0;
  for (int it = 0; it < 200 && hi - lo > 1e-6; it++) {
    double mid = 0.5 * (lo + hi);
    if (ramp_resp(qq, lam, k, D, mid) >= theta) hi = mid; else lo = mid;
  }
  return 0.5 * (lo + hi);
}

double orc_arnoldi_delay(uint32_t qq, const double* lam, const double* k, double slew, double* out_slew) {
  double D = slew / 0.6;                     /* 20-80 slew of a linear ramp is 0.6 D (reading A1) */
  double t50 = crossing(qq, lam, k, D, 0.5);
  if (out_slew) *out_slew = crossing(qq, lam, k, D, 0.8) - crossing(qq, lam, k, D, 0.2);
  return t50 - 0.5 * D;
}

/* ------------------------------------------------------- sense pairs (O5) */
/* SPEC.md:383 and SURVEY.md §8(c) O5: which (input edge -> output edge) pairs
 * an arc of a given sense propagates. */
static int sense_allows(uint8_t sense, int irf, int orf) {
  switch (sense) {
    case ORC_POS: return irf == orf;
    case ORC_NEG: return irf != orf;
    case ORC_NON: return 1;
    case ORC_RISE_EDGE: return irf == 0;
    case ORC_FALL_EDGE: return irf == 1;
  }
  return 0;
}

/* ----------------------------------------------- O10: top-k path report */
/* Request of a path report (run_update's hook: it runs after the backward
 * pass, on the final arrivals, the recorded arc delays and the endpoint
 * seeds). */
typedef struct {
  int mode;                 /* 0 setup (late), 1 hold (early) */
  uint32_t k, nworst;
  double slack_lt;
  /* outputs (capacities in brackets) */
  uint32_t cap_paths, cap_pins;
  uint32_t n_paths, n_pins;
  uint32_t* path_ptr;       /* [cap_paths + 1] */
  uint32_t* path_pin;       /* [cap_pins] startpoint first */
  uint8_t* path_rf;         /* [cap_pins] */
  double* path_at;          /* [cap_pins] arrival of the path at each of its pins */
  double* path_slack;       /* [cap_paths] */
  uint32_t* path_ep;        /* [cap_paths] */
} orc_path_req;

static int path_report(const orc_design* d, const arcs_t* g, const uint32_t* order, const double* at,
                       const double* elm, const double* dly, const double* seed, orc_path_req* q);

/* ------------------------------------------------- O16: case analysis */
/* SURVEY.md §8(f) row 4; SPEC.md:479-486 (apply_case_analysis), PAPER.md:39,
 * 113 ("case analysis modes"): constants from the case values propagate
 * forward -- a net's sinks take its driver's constant, a cell output whose
 * logic function evaluates to one value for every completion of its
 * non-constant inputs becomes that constant -- in topological order (one
 * pass is the fixpoint: a function depends only on its inputs); a pin with
 * two different constants is an error (6).  Disabled: every arc from or to
 * a constant pin, and every cell arc whose `when` guard is 0 for every
 * completion of the non-constant inputs of its output's function
 * (C1-C4). */
static int fn_eval(const orc_design* d, uint32_t f, const uint8_t* val, uint64_t tt) {
  /* 0 / 1: tt takes that value on every completion; 2: both values occur */
  const uint32_t b = d->fn_in_ptr[f], k = d->fn_in_ptr[f + 1] - b;
  int seen0 = 0, seen1 = 0;
  for (uint32_t m = 0; m < (1u << k); m++) {
    int ok = 1;
    for (uint32_t j = 0; j < k && ok; j++) {
      const uint8_t v = val[d->fn_in[b + j]];
      if (v != 2 && v != ((m >> j) & 1u)) ok = 0;
    }
    if (!ok) continue;
    if ((tt >> m) & 1u) seen1 = 1; else seen0 = 1;
  }
  return seen0 && seen1 ? 2 : (seen1 ? 1 : 0);
}

int orc_case_analysis(const orc_design* d, uint8_t* val, uint8_t* off) {
  const uint32_t P = d->num_pins;
  arcs_t g; memset(&g, 0, sizeof g);
  uint32_t* level = malloc(sizeof(uint32_t) * (P + 1));
  uint32_t* order = malloc(sizeof(uint32_t) * (P + 1));
  uint32_t* fn_of = malloc(sizeof(uint32_t) * (P + 1));
  int st = (!level || !order || !fn_of) ? 2 : build_arcs(d, &g);
  if (!st) st = kahn(d, &g, level, order) ? 1 : 0;
  for (uint32_t p = 0; !st && p < P; p++) { val[p] = 2; fn_of[p] = ORC_NO_PIN; }
  for (uint32_t f = 0; !st && f < d->n_fn; f++) {
    if (d->fn_in_ptr[f + 1] - d->fn_in_ptr[f] > 6) st = 7;
    else fn_of[d->fn_pin[f]] = f;
  }
  for (uint32_t k = 0; !st && k < d->n_case; k++) {
    const uint32_t p = d->case_pin[k];
    const uint8_t v = d->case_val[k] ? 1 : 0;
    if (val[p] != 2 && val[p] != v) st = 6;
    val[p] = v;
  }
  for (uint32_t i = 0; !st && i < P; i++) {
    const uint32_t v = order[i];
    for (uint32_t x = g.fi_ptr[v]; x < g.fi_ptr[v + 1]; x++) {
      const uint32_t e = g.fi[x];
      if (e >= g.En) continue;                       /* the net arc into a sink */
      const uint8_t c = val[g.from[e]];
      if (c == 2) continue;
      if (val[v] != 2 && val[v] != c) { st = 6; break; }
      val[v] = c;
    }
    if (!st && fn_of[v] != ORC_NO_PIN) {
      const int c = fn_eval(d, fn_of[v], val, d->fn_tt[fn_of[v]]);
      if (c != 2) {
        if (val[v] != 2 && val[v] != c) st = 6;
        else val[v] = (uint8_t)c;
      }
    }
  }
  for (uint32_t e = 0; !st && e < g.E; e++) {
    uint8_t o = val[g.from[e]] != 2 || val[g.to[e]] != 2;
    if (!o && e >= g.En && d->arc_when) {
      const uint32_t f = fn_of[g.to[e]];
      if (f != ORC_NO_PIN && fn_eval(d, f, val, d->arc_when[g.cell[e]]) == 0) o = 1;
    }
    off[e] = o;
  }
  free_arcs(&g); free(level); free(order); free(fn_of);
  return st;
}

static int has_case(const orc_design* d) { return d->n_case || d->arc_when; }

/* --------------------------------------------------------- O4-O8: update */
/* O15 handoff of one tag's pass at the -through pins (see run_tagged):
 * dst[p] = the pass whose tag this pass's tag advances to at pin p
 * (ORC_NO_PIN: none), thr[p] = p belongs to some -through segment; hand_at /
 * hand_sl [n_tags][P][4] collect the arrivals handed to each pass, rhand
 * [n_tags][P][4] the required times each pass computes at its through pins. */
typedef struct {
  uint32_t cur, P;
  int fwd_only;
  const uint32_t* dst;
  const uint8_t* thr;
  double *hand_at, *hand_sl, *rhand;
} orc_thr;

static int run_update(const orc_design* d, double* at, double* slew, double* rat, double* slack,
                      double res[4], uint32_t* ep_pin, double* ep_ws, uint32_t* n_ep_out, orc_path_req* pq,
                      const uint8_t* seed_on, const double* ep_ovr, const orc_thr* th);
static int run_tagged(const orc_design* d, double* at, double* slew, double* rat, double* slack,
                      double res[4], uint32_t* ep_pin, double* ep_ws, uint32_t* n_ep_out);


/* --------------------------------------- O13: -from / -to timing exceptions */
/* SURVEY.md §8(f) row 4 (reduced: no case analysis)
 * ("false paths, multi-cycle paths ... can significantly complicate the data
 * structures and states in timing propagation"); the tag model of
 * a path's tag is its launch clock and the segment bits of
 * the exceptions' -from / -through lists it has matched so far (O15 below);
 * each tag is propagated on its own (the startpoints of that tag seeded, the
 * others undefined; at -through pins arrivals move on to the advanced tag,
 * O15) and per endpoint the exceptions the tag fully matches are resolved
 * (X1-X6):
 *   late check: false path > max delay v (RAT_L = v) > multicycle N (capture
 *   at N T: RAT_L + (N-1) T); early check: false path > min delay v (RAT_E =
 *   v) > multicycle N (hold edge (N-1) T: RAT_E + (N-1) T); among exceptions
 *   of one kind the first listed wins.  Results: per pin the early / late
 *   extreme over tags of AT / slew / RAT and the minimum slack; per endpoint
 *   the worst slack over tags (a false path contributes none).
 * ep_ovr per pin: {late mode, late value, early mode, early value}, mode 0:
 * shift by the value, 1: replace by it, 2: no seed (false path). */
static void exc_apply(const double* o, double* rl, double* re) {
  if (o[0] == 2) *rl = INF; else if (o[0] == 1) *rl = o[1]; else *rl += o[1];
  if (o[2] == 2) *re = -INF; else if (o[2] == 1) *re = o[3]; else *re += o[3];
}

static int in_list(const uint32_t* a, uint32_t lo, uint32_t hi, uint32_t p) {
  for (uint32_t i = lo; i < hi; i++) if (a[i] == p) return 1;
  return 0;
}

enum { EXC_FALSE = 0, EXC_MULTICYCLE = 1, EXC_MAX = 2, EXC_MIN = 3 };

/* O14: setup / hold relationships between a launch clock of period TL and a
 * capture clock of period TC (rising edges at multiples of the period; the
 * "bounded hyperperiod" of SPEC.md:504 = the first 1000 launch edges,
 * DESIGN.md X7): for launch edge a the setup capture edge is the first
 * capture edge strictly after a, the hold edge the capture edge before it;
 * setup = the smallest (capture - launch), hold = the largest (hold edge -
 * launch).  One clock: setup T, hold 0. */
static void clk_rel(double TL, double TC, double* rs, double* rh) {
  double s = INF, h = -INF;
  for (int i = 0; i < 1000; i++) {
    const double a = i * TL;
    const double nxt = (floor(a / TC) + 1.0) * TC;
    if (nxt - a < s) s = nxt - a;
    if (nxt - TC - a > h) h = nxt - TC - a;
  }
  *rs = s;
  *rh = h;
}

/* O15: -through ("tags
 * advance their automaton bits at nodes belonging to a next-eligible
 * segment"; "multiple -through patterns that eliminate only
 * paths that go through a predefined pin sequence").  Exception e has the
 * ordered segments [from (if listed), through_1 .. through_m], one tag bit
 * each (bits base_e ..); a path's bits of e are always a prefix of its
 * segments.  At its startpoint a path sets e's from bit if the startpoint is
 * in the -from list; at every pin, while the next segment of e holds the pin,
 * its bit is set (one pin may match consecutive segments, X8); an
 * exception with a -from list that the startpoint missed never advances.
 * The exception holds for a path when all its bits are set (and the endpoint
 * is in its -to list).  adv() is that step. */
typedef struct {
  uint32_t base[32], nseg[32], has_from[32], total;
} segmap;

static int seg_map(const orc_design* d, segmap* m) {
  m->total = 0;
  for (uint32_t e = 0; e < d->n_exc; e++) {
    m->has_from[e] = d->exc_from_ptr[e + 1] > d->exc_from_ptr[e];
    m->nseg[e] = m->has_from[e] + (d->exc_thr_ptr ? d->exc_thr_ptr[e + 1] - d->exc_thr_ptr[e] : 0);
    m->base[e] = m->total;
    m->total += m->nseg[e];
  }
  return m->total <= 32;
}

/* does segment k of exception e hold pin p */
static int seg_has(const orc_design* d, const segmap* m, uint32_t e, uint32_t k, uint32_t p) {
  if (m->has_from[e] && k == 0) return in_list(d->exc_from, d->exc_from_ptr[e], d->exc_from_ptr[e + 1], p);
  const uint32_t sg = d->exc_thr_ptr[e] + k - m->has_from[e];
  return in_list(d->exc_seg, d->exc_seg_ptr[sg], d->exc_seg_ptr[sg + 1], p);
}

static uint32_t adv(const orc_design* d, const segmap* m, uint32_t bits, uint32_t p, int start) {
  for (uint32_t e = 0; e < d->n_exc; e++) {
    uint32_t k = 0;
    while (k < m->nseg[e] && ((bits >> (m->base[e] + k)) & 1u)) k++;
    if (m->has_from[e] && k == 0) {
      if (!start || !seg_has(d, m, e, 0, p)) continue;
      bits |= 1u << m->base[e];
      k = 1;
    }
    while (k < m->nseg[e] && seg_has(d, m, e, k, p)) {
      bits |= 1u << (m->base[e] + k);
      k++;
    }
  }
  return bits;
}

static int full(const segmap* m, uint32_t e, uint32_t bits) {
  const uint32_t mask = m->nseg[e] >= 32 ? 0xFFFFFFFFu : ((1u << m->nseg[e]) - 1u);
  return ((bits >> m->base[e]) & mask) == mask;
}

static int popc32(uint32_t x) {
  int n = 0;
  for (; x; x &= x - 1) n++;
  return n;
}

static int run_tagged(const orc_design* d, double* at, double* slew, double* rat, double* slack,
                      double res[4], uint32_t* ep_pin, double* ep_ws, uint32_t* n_ep_out) {
  const uint32_t P = d->num_pins, E = d->n_exc;
  if (E > 32) return 5;
  segmap m;
  if (!seg_map(d, &m)) return 5;
  /* step 1: the tag of every pin that could be a startpoint: its launch
   * clock (bits 32+) and its segment bits after the startpoint (bits 0..31) */
  uint64_t* tag = calloc(P + 1, sizeof(uint64_t));
  for (uint32_t p = 0; p < P; p++) {
    tag[p] = adv(d, &m, 0u, p, 1);
    if (d->n_clk) tag[p] |= (uint64_t)d->pin_clk[p] << 32;
  }
  /* step 2: the distinct tags of the startpoints, in pin order */
  uint64_t tags[64];
  uint32_t T = 0;
  int bad = 0;
  for (uint32_t p = 0; p < P; p++) {
    int sp = d->pin_role[p] == ORC_FF_CK;
    for (uint32_t k = 0; k < d->n_pi && !sp; k++) sp = d->pi_pin[k] == p;
    if (!sp) continue;
    uint32_t j = 0;
    while (j < T && tags[j] != tag[p]) j++;
    if (j == T) { if (T == 64) { bad = 1; break; } tags[T++] = tag[p]; }
  }
  if (T == 0) tags[T++] = 0;
  /* O15: the tags reached by advancing at -through pins (closure), ordered
   * by the number of set bits: a tag only advances to tags after it */
  uint8_t* thr = calloc(P + 1, 1);
  int any_thr = 0;
  if (d->exc_thr_ptr)
    for (uint32_t e = 0; e < E; e++)
      for (uint32_t sg = d->exc_thr_ptr[e]; sg < d->exc_thr_ptr[e + 1]; sg++)
        for (uint32_t i = d->exc_seg_ptr[sg]; i < d->exc_seg_ptr[sg + 1]; i++) { thr[d->exc_seg[i]] = 1; any_thr = 1; }
  for (uint32_t i = 0; i < T && !bad; i++)
    for (uint32_t p = 0; p < P && !bad; p++) {
      if (!thr[p]) continue;
      const uint64_t t2 = (tags[i] & ~0xFFFFFFFFull) | adv(d, &m, (uint32_t)tags[i], p, 0);
      uint32_t j = 0;
      while (j < T && tags[j] != t2) j++;
      if (j == T) { if (T == 64) bad = 1; else tags[T++] = t2; }
    }
  for (uint32_t i = 1; i < T; i++)            /* stable insertion sort by set bits */
    for (uint32_t j = i; j > 0 && popc32((uint32_t)tags[j - 1]) > popc32((uint32_t)tags[j]); j--) {
      const uint64_t x = tags[j]; tags[j] = tags[j - 1]; tags[j - 1] = x;
    }
  int st = bad ? 5 : 0;
  const size_t P4 = 4 * (size_t)(P + 1);
  double *t_at = malloc(sizeof(double) * P4), *t_sl = malloc(sizeof(double) * P4);
  double *t_rat = malloc(sizeof(double) * P4), *t_sk = malloc(sizeof(double) * P4);
  double* ovr = malloc(sizeof(double) * P4 * (T ? T : 1));
  uint8_t* on = malloc((size_t)(P + 1) * (T ? T : 1));
  uint32_t n_ep_max = d->n_po + d->num_checks + 1, n_ep = 0;
  uint32_t* t_ep = malloc(sizeof(uint32_t) * n_ep_max);
  double* t_ws = malloc(sizeof(double) * 2 * n_ep_max);
  double* m_ws = malloc(sizeof(double) * 2 * n_ep_max);
  double t_res[4];
  /* O15 handoff buffers (tags x pins) and each pass's destination at every
   * through pin */
  const size_t TP4 = (size_t)T * P4;
  uint32_t* dst = any_thr ? malloc(sizeof(uint32_t) * (size_t)T * (P + 1)) : NULL;
  double* h_at = any_thr ? malloc(sizeof(double) * TP4) : NULL;
  double* h_sl = any_thr ? malloc(sizeof(double) * TP4) : NULL;
  double* h_rat = any_thr ? calloc(TP4, sizeof(double)) : NULL;
  if (any_thr) {
    for (size_t i = 0; i < TP4; i++) h_at[i] = h_sl[i] = (i & 3) < 2 ? INF : -INF;
    for (uint32_t j = 0; j < T; j++)
      for (uint32_t p = 0; p < P; p++) {
        uint32_t to = ORC_NO_PIN;
        if (thr[p]) {
          const uint64_t t2 = (tags[j] & ~0xFFFFFFFFull) | adv(d, &m, (uint32_t)tags[j], p, 0);
          if (t2 != tags[j])
            for (uint32_t k = 0; k < T; k++) if (tags[k] == t2) to = k;
        }
        dst[(size_t)j * (P + 1) + p] = to;
      }
  }
  for (uint32_t j = 0; j < T && !st; j++) {
    /* step 3: tag j: its startpoints seeded; each endpoint's exception */
    uint8_t* onj = on + (size_t)j * (P + 1);
    for (uint32_t p = 0; p < P; p++) onj[p] = tag[p] == tags[j];
    const uint32_t lclk = (uint32_t)(tags[j] >> 32);
    for (uint32_t p = 0; p < P; p++) {
      double* o = ovr + P4 * j + 4 * (size_t)p;
      o[0] = o[1] = o[2] = o[3] = 0.0;
      /* O14: the capture clock of endpoint p (a PO's own, a D pin's register
       * clock) and the relationship to this tag's launch clock; the base
       * seeds assume the single clock `period` (setup T, hold 0) */
      double Tcap = d->period;
      if (d->n_clk) {
        uint32_t cc = d->pin_clk[p];
        for (uint32_t c = 0; c < d->num_checks; c++)
          if (d->chk_d[c] == p) { cc = d->pin_clk[d->chk_ck[c]]; break; }
        Tcap = d->clk_period[cc];
        double rs, rh;
        clk_rel(d->clk_period[lclk], Tcap, &rs, &rh);
        o[1] = rs - d->period;
        o[3] = rh;
      }
      int lf = -1, lm = -1, lc = -1, ef = -1, em = -1, ec = -1;
      for (uint32_t e = 0; e < E; e++) {
        const int has_to = d->exc_to_ptr[e + 1] > d->exc_to_ptr[e];
        if (!full(&m, e, (uint32_t)tags[j])) continue;
        if (has_to && !in_list(d->exc_to, d->exc_to_ptr[e], d->exc_to_ptr[e + 1], p)) continue;
        switch (d->exc_kind[e]) {
          case EXC_FALSE: if (lf < 0) lf = (int)e; if (ef < 0) ef = (int)e; break;
          case EXC_MAX: if (lm < 0) lm = (int)e; break;
          case EXC_MIN: if (em < 0) em = (int)e; break;
          case EXC_MULTICYCLE: if (lc < 0) lc = (int)e; if (ec < 0) ec = (int)e; break;
        }
      }
      if (lf >= 0) o[0] = 2;
      else if (lm >= 0) { o[0] = 1; o[1] = d->exc_value[lm]; }
      else if (lc >= 0) o[1] += (d->exc_value[lc] - 1.0) * Tcap;
      if (ef >= 0) o[2] = 2;
      else if (em >= 0) { o[2] = 1; o[3] = d->exc_value[em]; }
      else if (ec >= 0) o[3] += (d->exc_value[ec] - 1.0) * Tcap;
    }
  }
  /* O15: a first sweep of the forwards in tag order collects every pass's
   * handed-over arrivals; the full passes then run in reverse tag order so
   * that the required times a pass takes over at its through pins exist */
  if (any_thr)
    for (uint32_t j = 0; j < T && !st; j++) {
      orc_thr th = {j, P, 1, dst + (size_t)j * (P + 1), thr, h_at, h_sl, h_rat};
      st = run_update(d, t_at, t_sl, t_rat, t_sk, t_res, t_ep, t_ws, &n_ep, NULL, on + (size_t)j * (P + 1),
                      ovr + P4 * j, &th);
    }
  for (uint32_t jj = 0; jj < T && !st; jj++) {
    const uint32_t j = any_thr ? T - 1 - jj : jj;
    orc_thr th = {j, P, 0, any_thr ? dst + (size_t)j * (P + 1) : NULL, thr, h_at, h_sl, h_rat};
    st = run_update(d, t_at, t_sl, t_rat, t_sk, t_res, t_ep, t_ws, &n_ep, NULL, on + (size_t)j * (P + 1),
                    ovr + P4 * j, any_thr ? &th : NULL);
    if (st) break;
    /* step 4: merge over tags */
    for (size_t i = 0; i < 4 * (size_t)P; i++) {
      const int e = (i & 3) < 2;            /* early component */
      if (jj == 0) { at[i] = t_at[i]; if (slew) slew[i] = t_sl[i]; if (rat) rat[i] = t_rat[i]; if (slack) slack[i] = t_sk[i]; continue; }
      at[i] = e ? fmin(at[i], t_at[i]) : fmax(at[i], t_at[i]);
      if (slew) slew[i] = e ? fmin(slew[i], t_sl[i]) : fmax(slew[i], t_sl[i]);
      if (rat) rat[i] = e ? fmax(rat[i], t_rat[i]) : fmin(rat[i], t_rat[i]);
      if (slack) slack[i] = fmin(slack[i], t_sk[i]);
    }
    for (uint32_t k = 0; k < 2 * n_ep; k++) m_ws[k] = jj == 0 ? t_ws[k] : fmin(m_ws[k], t_ws[k]);
  }
  if (!st) {
    double ws = INF, tns = 0.0, wh = INF, tnh = 0.0;
    for (uint32_t k = 0; k < n_ep; k++) {
      const double s = m_ws[2 * k], h = m_ws[2 * k + 1];
      if (s < ws) ws = s;
      if (s < 0) tns += s;
      if (h < wh) wh = h;
      if (h < 0) tnh += h;
      if (ep_pin) ep_pin[k] = t_ep[k];
      if (ep_ws) { ep_ws[2 * k] = s; ep_ws[2 * k + 1] = h; }
    }
    res[0] = ws; res[1] = tns; res[2] = wh; res[3] = tnh;
    if (n_ep_out) *n_ep_out = n_ep;
  }
  free(tag); free(t_at); free(t_sl); free(t_rat); free(t_sk); free(ovr); free(on);
  free(t_ep); free(t_ws); free(m_ws); free(thr); free(dst); free(h_at); free(h_sl); free(h_rat);
  return st;
}

int orc_update(const orc_design* d, double* at, double* slew, double* rat, double* slack,
               double res[4], uint32_t* ep_pin, double* ep_ws, uint32_t* n_ep_out) {
  if (d->n_exc || d->n_clk) return run_tagged(d, at, slew, rat, slack, res, ep_pin, ep_ws, n_ep_out);
  return run_update(d, at, slew, rat, slack, res, ep_pin, ep_ws, n_ep_out, NULL, NULL, NULL, NULL);
}

int orc_paths(const orc_design* d, int mode, uint32_t k, uint32_t nworst, double slack_lt, uint32_t cap_paths,
              uint32_t cap_pins, uint32_t* n_paths, uint32_t* n_pins, uint32_t* path_ptr, uint32_t* path_pin,
              uint8_t* path_rf, double* path_at, double* path_slack, uint32_t* path_ep) {
  orc_path_req q;
  memset(&q, 0, sizeof q);
  q.mode = mode; q.k = k; q.nworst = nworst; q.slack_lt = slack_lt;
  q.cap_paths = cap_paths; q.cap_pins = cap_pins;
  q.path_ptr = path_ptr; q.path_pin = path_pin; q.path_rf = path_rf; q.path_at = path_at;
  q.path_slack = path_slack; q.path_ep = path_ep;
  double res[4];
  uint32_t P = d->num_pins;
  double* at = malloc(sizeof(double) * 4 * (size_t)(P + 1));
  if (!at) return 2;
  if (d->n_exc || d->n_clk) { free(at); return 4; }   /* path reports: one clock, no exceptions (X6) */
  int st = run_update(d, at, NULL, NULL, NULL, res, NULL, NULL, NULL, &q, NULL, NULL, NULL);
  free(at);
  *n_paths = q.n_paths;
  *n_pins = q.n_pins;
  return st;
}

static int run_update(const orc_design* d, double* at, double* slew, double* rat, double* slack,
                      double res[4], uint32_t* ep_pin, double* ep_ws, uint32_t* n_ep_out, orc_path_req* pq,
                      const uint8_t* seed_on, const double* ep_ovr, const orc_thr* th) {
  const uint32_t P = d->num_pins;
  const double LN9 = log(9.0);
  arcs_t g; memset(&g, 0, sizeof g);
  /* O16: the arcs case analysis disables are left out of the graph */
  uint8_t* off = NULL;
  if (has_case(d)) {
    uint8_t* cval = malloc(P + 1);
    off = malloc((size_t)(d->net_ptr[d->num_nets] - d->num_nets) + d->num_arcs + 1);
    const int cst = (!cval || !off) ? 2 : orc_case_analysis(d, cval, off);
    free(cval);
    if (cst) { free(off); return cst; }
  }
  const int bst = build_arcs_off(d, &g, off);
  free(off);
  if (bst) { free_arcs(&g); return 2; }
  uint32_t* level = malloc(sizeof(uint32_t) * (P + 1));
  uint32_t* order = malloc(sizeof(uint32_t) * (P + 1));
  double* load = malloc(sizeof(double) * (d->num_nets + 1));
  double* elm = malloc(sizeof(double) * (P + 1));
  double* drv_load = calloc(P + 1, sizeof(double));  /* load seen by a net's driver pin */
  double* dly = malloc(sizeof(double) * (8 * (size_t)d->num_arcs + 1)); /* d_el(a, irf->orf) */
  double* own_slew = slew ? NULL : malloc(sizeof(double) * 4 * (size_t)(P + 1));
  double* own_rat = rat ? NULL : malloc(sizeof(double) * 4 * (size_t)(P + 1));
  double* own_slack = slack ? NULL : malloc(sizeof(double) * 4 * (size_t)(P + 1));
  uint8_t* is_ep = calloc(P + 1, 1);
  /* O12 (net_model 1): per sink pin its net's reduced model: order (0: Elmore
   * fallback or lumped net), time constants, residues; and the per-component
   * net-arc delays the forward used (the backward reuses them) */
  const int arn = d->net_model == 1;
  const uint32_t aq = arn ? (d->arnoldi_q ? d->arnoldi_q : 4) : 1;
  uint32_t* a_qq = arn ? calloc(P + 1, sizeof(uint32_t)) : NULL;
  double* a_lam = arn ? calloc((size_t)(P + 1) * aq, sizeof(double)) : NULL;
  double* a_res = arn ? calloc((size_t)(P + 1) * aq, sizeof(double)) : NULL;
  double* ndly = arn ? calloc(4 * (size_t)(P + 1), sizeof(double)) : NULL;
  int st = 0;
  if (!slew) slew = own_slew;
  if (!rat) rat = own_rat;
  if (!slack) slack = own_slack;
  if (!level || !order || !load || !elm || !drv_load || !dly || !slew || !rat || !slack || !is_ep ||
      (arn && (!a_qq || !a_lam || !a_res || !ndly))) {
    st = 2; goto done;
  }
  if (arn && pq) { st = 4; goto done; }     /* path reports: Elmore model only (A7) */
  if (kahn(d, &g, level, order)) { st = 1; goto done; }

  /* O3 */
  orc_rc(d, load, elm);
  for (uint32_t n = 0; n < d->num_nets; n++) drv_load[d->net_pins[d->net_ptr[n]]] = load[n];
  if (arn) {                                 /* O12: one reduced model per net with RC nodes */
    double* po_ld = calloc(P + 1, sizeof(double));
    for (uint32_t k = 0; k < d->n_po; k++) po_ld[d->po_pin[k]] += d->po_load[k];
    uint32_t maxn = 1;
    for (uint32_t n = 0; n < d->num_nets; n++)
      if (d->rc_ptr[n + 1] - d->rc_ptr[n] > maxn) maxn = d->rc_ptr[n + 1] - d->rc_ptr[n];
    double* cap = malloc(sizeof(double) * maxn);
    double* lam = malloc(sizeof(double) * aq);
    double* rsd = malloc(sizeof(double) * (size_t)maxn * aq);
    for (uint32_t n = 0; n < d->num_nets; n++) {
      uint32_t b = d->rc_ptr[n], m = d->rc_ptr[n + 1] - b;
      if (m == 0) continue;                  /* lumped: zero wire delay, the Elmore path */
      for (uint32_t i = 0; i < m; i++) {
        uint32_t p = d->rc_node_pin[b + i];
        cap[i] = d->rc_cap[b + i] + (p != ORC_NO_PIN ? d->pin_cap[p] + po_ld[p] : 0.0);
      }
      int qq = orc_arnoldi_reduce(m, d->rc_parent + b, d->rc_res + b, cap, aq, lam, rsd);
      if (qq < 0) continue;                  /* unstable: Elmore fallback */
      for (uint32_t i = 1; i < m; i++) {
        uint32_t p = d->rc_node_pin[b + i];
        if (p == ORC_NO_PIN) continue;
        a_qq[p] = (uint32_t)qq;
        for (uint32_t k = 0; k < aq; k++) {
          a_lam[(size_t)p * aq + k] = k < (uint32_t)qq ? lam[k] : 0.0;
          a_res[(size_t)p * aq + k] = rsd[(size_t)i * aq + k];
        }
      }
    }
    free(cap); free(lam); free(rsd); free(po_ld);
  }

  /* O4 seeds: everything undefined, then PIs and ideal-clock CK pins. */
  for (uint32_t p = 0; p < P; p++) {
    for (int rf = 0; rf < 2; rf++) {
      at[4 * p + Q(0, rf)] = INF;   slew[4 * p + Q(0, rf)] = INF;
      at[4 * p + Q(1, rf)] = -INF;  slew[4 * p + Q(1, rf)] = -INF;
    }
  }
  for (uint32_t k = 0; k < d->n_pi; k++) {
    uint32_t p = d->pi_pin[k];
    if (g.fi_ptr[p + 1] != g.fi_ptr[p]) continue;
    if (seed_on && !seed_on[p]) continue;    /* O13: a startpoint of another tag */
    for (int q = 0; q < 4; q++) { at[4 * p + q] = d->pi_at[4 * k + q]; slew[4 * p + q] = d->pi_slew[4 * k + q]; }
  }
  for (uint32_t p = 0; p < P; p++) {
    if (d->pin_role[p] != ORC_FF_CK || g.fi_ptr[p + 1] != g.fi_ptr[p]) continue;
    if (seed_on && !seed_on[p]) continue;
    /* ideal clock, rising edge at 0, waveform (0, T/2); with
     * several clocks the period of the pin's own clock (O14) */
    const double Tc = d->n_clk ? (double)d->clk_period[d->pin_clk[p]] : d->period;
    at[4 * p + Q(0, 0)] = 0.0; at[4 * p + Q(0, 1)] = Tc / 2;
    at[4 * p + Q(1, 0)] = 0.0; at[4 * p + Q(1, 1)] = Tc / 2;
    for (int q = 0; q < 4; q++) slew[4 * p + q] = d->clock_slew;
  }

  /* O5 forward in topological order. */
  for (uint32_t k = 0; k < P; k++) {
    uint32_t v = order[k];
    if (g.fi_ptr[v + 1] == g.fi_ptr[v]) continue;
    for (uint32_t x = g.fi_ptr[v]; x < g.fi_ptr[v + 1]; x++) {
      uint32_t e = g.fi[x], u = g.from[e];
      for (int el = 0; el < 2; el++) {
        for (int irf = 0; irf < 2; irf++) {
          double a_in = at[4 * u + Q(el, irf)];
          if (!isfinite(a_in)) continue;
          double s_in = slew[4 * u + Q(el, irf)];
          for (int orf = 0; orf < 2; orf++) {
            double ca, cs;
            if (e < g.En && arn && a_qq[v]) {   /* net arc, Arnoldi (O12) */
              if (irf != orf) continue;
              double os;
              double dn = orc_arnoldi_delay(a_qq[v], a_lam + (size_t)v * aq, a_res + (size_t)v * aq, s_in, &os);
              ndly[4 * (size_t)v + Q(el, orf)] = dn;
              ca = a_in + dn;
              cs = os;
            } else if (e < g.En) {         /* net arc: positive unate, Elmore */
              if (irf != orf) continue;
              double imp = LN9 * elm[v];   /* SPEC.md:418 PERI */
              ca = a_in + elm[v];
              cs = sqrt(s_in * s_in + imp * imp);
            } else {                       /* cell arc: NLDM */
              uint32_t a = g.cell[e];
              if (!sense_allows(d->arc_sense[a], irf, orf)) continue;
              uint32_t tb = d->arc_tab[a];
              double ld = drv_load[v];
              double dd = lut_id(d, tb + (uint32_t)orf, s_in, ld);        /* cell_rise/fall */
              double ss = lut_id(d, tb + 2 + (uint32_t)orf, s_in, ld);    /* rise/fall_tr */
              if (dd < 0) dd = 0;
              if (ss < 0) ss = 0;
              dly[8 * (size_t)a + 4 * el + 2 * irf + orf] = dd;
              ca = a_in + dd;
              cs = ss;
            }
            /* merge: early takes min, late takes max, AT and slew independently */
            double* pa = &at[4 * v + Q(el, orf)];
            double* ps = &slew[4 * v + Q(el, orf)];
            if (el == 0) { if (ca < *pa) *pa = ca; if (cs < *ps) *ps = cs; }
            else         { if (ca > *pa) *pa = ca; if (cs > *ps) *ps = cs; }
          }
        }
      }
    }
    /* O15: at a -through pin this tag's arrivals either move on to the tag
     * it advances to (handed to that later pass, undefined here) or, if the
     * tag is final at v, take in what earlier passes handed to it */
    if (th && th->thr[v]) {
      const uint32_t to = th->dst[v];
      double* ha = (to != ORC_NO_PIN ? th->hand_at + ((size_t)to * th->P + v) * 4 : th->hand_at + ((size_t)th->cur * th->P + v) * 4);
      double* hs = (to != ORC_NO_PIN ? th->hand_sl + ((size_t)to * th->P + v) * 4 : th->hand_sl + ((size_t)th->cur * th->P + v) * 4);
      for (int q = 0; q < 4; q++) {
        double* pa = &at[4 * v + q];
        double* ps = &slew[4 * v + q];
        if (to != ORC_NO_PIN) {
          if (q < 2) { if (*pa < ha[q]) ha[q] = *pa; if (*ps < hs[q]) hs[q] = *ps; }
          else       { if (*pa > ha[q]) ha[q] = *pa; if (*ps > hs[q]) hs[q] = *ps; }
          *pa = *ps = q < 2 ? INF : -INF;
        } else {
          if (q < 2) { if (ha[q] < *pa) *pa = ha[q]; if (hs[q] < *ps) *ps = hs[q]; }
          else       { if (ha[q] > *pa) *pa = ha[q]; if (hs[q] > *ps) *ps = hs[q]; }
        }
      }
    }
  }
  if (th && th->fwd_only) goto done;

  /* O7 endpoint seeds then backward in reverse order. */
  for (uint32_t p = 0; p < P; p++) {
    for (int rf = 0; rf < 2; rf++) { rat[4 * p + Q(0, rf)] = -INF; rat[4 * p + Q(1, rf)] = INF; }
  }
  for (uint32_t k = 0; k < d->n_po; k++) {
    uint32_t p = d->po_pin[k];
    is_ep[p] = 1;
    for (int rf = 0; rf < 2; rf++) {
      double rl = d->period - d->po_out_max[2 * k + rf];
      double re = -(double)d->po_out_min[2 * k + rf];
      if (ep_ovr) exc_apply(ep_ovr + 4 * (size_t)p, &rl, &re);
      if (rl < rat[4 * p + Q(1, rf)]) rat[4 * p + Q(1, rf)] = rl;
      if (re > rat[4 * p + Q(0, rf)]) rat[4 * p + Q(0, rf)] = re;
    }
  }
  for (uint32_t c = 0; c < d->num_checks; c++) {
    uint32_t p = d->chk_d[c], tb = d->chk_tab[c];
    is_ep[p] = 1;
    for (int rf = 0; rf < 2; rf++) {
      if (isfinite(at[4 * p + Q(1, rf)])) {   /* setup: index_1 data slew, index_2 clock slew */
        double rl = d->period - lut_id(d, tb + (uint32_t)rf, slew[4 * p + Q(1, rf)], d->clock_slew);
        double dummy = -INF;
        if (ep_ovr) exc_apply(ep_ovr + 4 * (size_t)p, &rl, &dummy);
        if (rl < rat[4 * p + Q(1, rf)]) rat[4 * p + Q(1, rf)] = rl;
      }
      if (isfinite(at[4 * p + Q(0, rf)])) {   /* hold */
        double re = lut_id(d, tb + 2 + (uint32_t)rf, slew[4 * p + Q(0, rf)], d->clock_slew);
        double dummy = INF;
        if (ep_ovr) exc_apply(ep_ovr + 4 * (size_t)p, &dummy, &re);
        if (re > rat[4 * p + Q(0, rf)]) rat[4 * p + Q(0, rf)] = re;
      }
    }
  }
  if (pq) {   /* O10 needs each endpoint's own seed (its check), before the backward */
    double* seed = malloc(sizeof(double) * 4 * (size_t)(P + 1));
    if (!seed) { st = 2; goto done; }
    memcpy(seed, rat, sizeof(double) * 4 * (size_t)P);
    for (uint32_t p = 0; p < P; p++)
      if (!is_ep[p]) for (int q = 0; q < 4; q++) seed[4 * p + q] = q < 2 ? -INF : INF;
    st = path_report(d, &g, order, at, elm, dly, seed, pq);
    free(seed);
    goto done;
  }
  for (uint32_t k = P; k-- > 0;) {
    uint32_t u = order[k];
    for (uint32_t x = g.fo_ptr[u]; x < g.fo_ptr[u + 1]; x++) {
      uint32_t e = g.fo[x], v = g.to[e];
      for (int el = 0; el < 2; el++) {
        for (int irf = 0; irf < 2; irf++) {
          if (!isfinite(at[4 * u + Q(el, irf)])) continue;   /* only arcs O5 used */
          for (int orf = 0; orf < 2; orf++) {
            double dd;
            if (e < g.En) { if (irf != orf) continue; dd = arn && a_qq[v] ? ndly[4 * (size_t)v + Q(el, orf)] : elm[v]; }
            else {
              uint32_t a = g.cell[e];
              if (!sense_allows(d->arc_sense[a], irf, orf)) continue;
              dd = dly[8 * (size_t)a + 4 * el + 2 * irf + orf];
            }
            double cand = rat[4 * v + Q(el, orf)] - dd;
            double* pr = &rat[4 * u + Q(el, irf)];
            if (el == 1) { if (cand < *pr) *pr = cand; }   /* late: min */
            else         { if (cand > *pr) *pr = cand; }   /* early: max */
          }
        }
      }
    }
    /* O15: at a -through pin the required times of the tag this one
     * advances to (its paths continue as that tag); a final tag records
     * its own for the earlier passes */
    if (th && th->thr[u]) {
      const uint32_t to = th->dst[u];
      for (int q = 0; q < 4; q++) {
        if (to != ORC_NO_PIN) rat[4 * u + q] = th->rhand[((size_t)to * th->P + u) * 4 + q];
        else th->rhand[((size_t)th->cur * th->P + u) * 4 + q] = rat[4 * u + q];
      }
    }
  }

  /* O8 slack, WNS, TNS */
  for (uint32_t p = 0; p < P; p++) {
    for (int rf = 0; rf < 2; rf++) {
      double al = at[4 * p + Q(1, rf)], rl = rat[4 * p + Q(1, rf)];
      double ae = at[4 * p + Q(0, rf)], re = rat[4 * p + Q(0, rf)];
      slack[4 * p + Q(1, rf)] = (isfinite(al) && isfinite(rl)) ? rl - al : INF;
      slack[4 * p + Q(0, rf)] = (isfinite(ae) && isfinite(re)) ? ae - re : INF;
    }
  }
  {
    double wns_s = INF, tns_s = 0.0, wns_h = INF, tns_h = 0.0;
    uint32_t ne = 0;
    for (uint32_t p = 0; p < P; p++) {
      if (!is_ep[p]) continue;
      double ws = slack[4 * p + Q(1, 0)] < slack[4 * p + Q(1, 1)] ? slack[4 * p + Q(1, 0)] : slack[4 * p + Q(1, 1)];
      double wh = slack[4 * p + Q(0, 0)] < slack[4 * p + Q(0, 1)] ? slack[4 * p + Q(0, 0)] : slack[4 * p + Q(0, 1)];
      if (ws < wns_s) wns_s = ws;
      if (wh < wns_h) wns_h = wh;
      if (ws < 0) tns_s += ws;
      if (wh < 0) tns_h += wh;
      if (ep_pin) ep_pin[ne] = p;
      if (ep_ws) { ep_ws[2 * ne] = ws; ep_ws[2 * ne + 1] = wh; }
      ne++;
    }
    res[0] = wns_s; res[1] = tns_s; res[2] = wns_h; res[3] = tns_h;
    if (n_ep_out) *n_ep_out = ne;
  }

done:
  free_arcs(&g);
  free(level); free(order); free(load); free(elm); free(drv_load); free(dly);
  free(own_slew); free(own_rat); free(own_slack); free(is_ep);
  free(a_qq); free(a_lam); free(a_res); free(ndly);
  return st;
}

/* ----------------------------------------------- O10: top-k path report */
/* SURVEY.md §8(f) row 3; PAPER.md:187-190 ("top-k path reports ... controlled
 * with top-k, per-endpoint report limit, and slack-less-than thresholds ...
 * flattened CSR-based path pin arrays with slacks").
 * Readings (P1-P4): a path is a sequence of (pin, transition)
 * nodes from a startpoint with a defined arrival to an endpoint with a
 * defined seed, along enabled arcs with the transition pairs their sense
 * allows; its arrival is the startpoint's arrival plus the delays the update
 * used on its arcs (graph-based: recorded cell delays, Elmore net delays);
 * setup slack = seed_L - arrival_L, hold slack = arrival_E - seed_E, the
 * seed being the endpoint's own required time (its check / output delay).
 * Report order: slack, then endpoint pin id, then the node sequence read
 * backwards from the endpoint ((pin, rf) lexicographic).  Selection walks
 * that order keeping at most nworst paths per endpoint, slack < slack_lt,
 * k paths in all.
 * Plain dynamic program: the m = min(nworst, k) first partial paths into
 * every (pin, rf) in that order, in topological order, each extending a
 * partial path of a fan-in (u, irf) by the arc's delay -- a path among the m
 * first into (v, rf) has its prefix among the m first into its predecessor,
 * so the lists are exact.  Ties between equal arrivals at a node compare
 * the predecessor (pin, rf) and then its rank there, which is the backward
 * sequence order. */
typedef struct {
  double a;                 /* arrival of the partial path at this node */
  uint32_t pin;             /* predecessor pin (ORC_NO_PIN at a startpoint) */
  uint32_t rf;              /* predecessor transition */
  uint32_t rank;            /* predecessor's rank in its list */
} pent;

static int g_late;          /* comparator mode (single-threaded oracle) */

static int cmp_pent(const void* x, const void* y) {
  const pent* a = (const pent*)x;
  const pent* b = (const pent*)y;
  if (a->a != b->a) return g_late ? (a->a > b->a ? -1 : 1) : (a->a < b->a ? -1 : 1);
  if (a->pin != b->pin) return a->pin < b->pin ? -1 : 1;
  if (a->rf != b->rf) return a->rf < b->rf ? -1 : 1;
  return a->rank < b->rank ? -1 : (a->rank > b->rank ? 1 : 0);
}

typedef struct {
  double slack;
  uint32_t ep, rf, rank;
} pcand;

static int cmp_pcand(const void* x, const void* y) {
  const pcand* a = (const pcand*)x;
  const pcand* b = (const pcand*)y;
  if (a->slack != b->slack) return a->slack < b->slack ? -1 : 1;
  if (a->ep != b->ep) return a->ep < b->ep ? -1 : 1;
  if (a->rf != b->rf) return a->rf < b->rf ? -1 : 1;
  return a->rank < b->rank ? -1 : (a->rank > b->rank ? 1 : 0);
}

static int path_report(const orc_design* d, const arcs_t* g, const uint32_t* order, const double* at,
                       const double* elm, const double* dly, const double* seed, orc_path_req* q) {
  const uint32_t P = d->num_pins;
  const int late = q->mode == 0, el = late ? 1 : 0;
  const uint32_t m = q->nworst < q->k ? q->nworst : q->k;
  q->n_paths = q->n_pins = 0;
  if (m == 0) return 0;
  pent* L = malloc(sizeof(pent) * 2 * (size_t)P * m + 1);
  uint32_t* cnt = calloc(2 * (size_t)P + 1, sizeof(uint32_t));
  uint32_t maxfi = 1;
  for (uint32_t v = 0; v < P; v++) {
    uint32_t f = g->fi_ptr[v + 1] - g->fi_ptr[v];
    if (f > maxfi) maxfi = f;
  }
  pent* cand = malloc(sizeof(pent) * 2 * (size_t)maxfi * m + 1);
  if (!L || !cnt || !cand) { free(L); free(cnt); free(cand); return 2; }
  g_late = late;
  /* the m first partial paths into every (pin, rf), in topological order */
  for (uint32_t k = 0; k < P; k++) {
    const uint32_t v = order[k];
    for (int rf = 0; rf < 2; rf++) {
      pent* lv = L + ((size_t)v * 2 + rf) * m;
      uint32_t nc = 0;
      if (g->fi_ptr[v + 1] == g->fi_ptr[v]) {            /* startpoint: its own arrival */
        if (isfinite(at[4 * v + Q(el, rf)])) {
          lv[0].a = at[4 * v + Q(el, rf)]; lv[0].pin = ORC_NO_PIN; lv[0].rf = 0; lv[0].rank = 0;
          cnt[2 * v + rf] = 1;
        }
        continue;
      }
      for (uint32_t x = g->fi_ptr[v]; x < g->fi_ptr[v + 1]; x++) {
        const uint32_t e = g->fi[x], u = g->from[e];
        for (int irf = 0; irf < 2; irf++) {
          double dd;
          if (e < g->En) {                                 /* net arc: positive unate, Elmore */
            if (irf != rf) continue;
            dd = elm[v];
          } else {
            const uint32_t a = g->cell[e];
            if (!sense_allows(d->arc_sense[a], irf, rf)) continue;
            dd = dly[8 * (size_t)a + 4 * el + 2 * irf + rf];
          }
          const pent* lu = L + ((size_t)u * 2 + irf) * m;
          for (uint32_t j = 0; j < cnt[2 * u + irf]; j++) {
            cand[nc].a = lu[j].a + dd; cand[nc].pin = u; cand[nc].rf = (uint32_t)irf; cand[nc].rank = j;
            nc++;
          }
        }
      }
      qsort(cand, nc, sizeof(pent), cmp_pent);
      if (nc > m) nc = m;
      memcpy(lv, cand, sizeof(pent) * nc);
      cnt[2 * v + rf] = nc;
    }
  }
  /* endpoint candidates, in report order */
  size_t ncand = 0;
  for (uint32_t p = 0; p < P; p++)
    for (int rf = 0; rf < 2; rf++) ncand += cnt[2 * p + rf];
  pcand* pc = malloc(sizeof(pcand) * (ncand + 1));
  uint32_t* kept = calloc(P + 1, sizeof(uint32_t));
  uint32_t* chain = malloc(sizeof(uint32_t) * 3 * (size_t)(P + 1));
  if (!pc || !kept || !chain) { free(L); free(cnt); free(cand); free(pc); free(kept); free(chain); return 2; }
  size_t n = 0;
  for (uint32_t p = 0; p < P; p++) {
    for (int rf = 0; rf < 2; rf++) {
      const double sd = seed[4 * p + Q(el, rf)];
      if (!isfinite(sd)) continue;                       /* not an endpoint, or no seed */
      const pent* lp = L + ((size_t)p * 2 + rf) * m;
      for (uint32_t j = 0; j < cnt[2 * p + rf]; j++) {
        pc[n].slack = late ? sd - lp[j].a : lp[j].a - sd;
        pc[n].ep = p; pc[n].rf = (uint32_t)rf; pc[n].rank = j;
        n++;
      }
    }
  }
  qsort(pc, n, sizeof(pcand), cmp_pcand);
  int st = 0;
  for (size_t i = 0; i < n && q->n_paths < q->k; i++) {
    if (!(pc[i].slack < q->slack_lt)) break;
    if (kept[pc[i].ep] >= q->nworst) continue;
    kept[pc[i].ep]++;
    /* the node chain, endpoint first */
    uint32_t len = 0, v = pc[i].ep, rf = pc[i].rf, r = pc[i].rank;
    for (;;) {
      chain[3 * len] = v; chain[3 * len + 1] = rf; chain[3 * len + 2] = r;
      len++;
      const pent* e = L + ((size_t)v * 2 + rf) * m + r;
      if (e->pin == ORC_NO_PIN) break;
      v = e->pin; rf = e->rf; r = e->rank;
    }
    if (q->n_paths + 1 > q->cap_paths || q->n_pins + len > q->cap_pins) { st = 3; break; }
    q->path_ptr[q->n_paths] = q->n_pins;
    for (uint32_t t = 0; t < len; t++) {                 /* startpoint first */
      const uint32_t* c = chain + 3 * (len - 1 - t);
      q->path_pin[q->n_pins + t] = c[0];
      q->path_rf[q->n_pins + t] = (uint8_t)c[1];
      q->path_at[q->n_pins + t] = L[((size_t)c[0] * 2 + c[1]) * m + c[2]].a;
    }
    q->n_pins += len;
    q->path_slack[q->n_paths] = pc[i].slack;
    q->path_ep[q->n_paths] = pc[i].ep;
    q->n_paths++;
    q->path_ptr[q->n_paths] = q->n_pins;
  }
  free(L); free(cnt); free(cand); free(pc); free(kept); free(chain);
  return st;
}

/* ------------------------------------------------- O11: built-in Steiner RC */
/* SURVEY.md §8(f) row 2; PAPER.md:178-179 ("A placer only needs to provide
 * HeteroSTA with pin positions and unit resistance/capacitance values along
 * x/y directions"); the construction is SPEC.md:322-331 with its decisions
 * SPEC.md:338-343 (FLUTE's tables are out of scope there too):
 *   1. a net's pins: the driver, then its sinks sorted by pin id;
 *   2. rectilinear minimum spanning tree by Prim from the driver, Manhattan
 *      distance, the next pin = smallest distance to the tree, ties by the
 *      smaller pin id; a pin's tree parent = the tree pin that first gave it
 *      its final distance (strict improvement only: DESIGN.md reading S2);
 *   3. each tree edge parent -> child embedded as an L, horizontal leg first
 *      from the parent (reading S3): one Steiner node at (x_child, y_parent)
 *      when both legs are non-zero;
 *   4. a leg of length L in direction d: resistance L * unit_res_d, and
 *      L * unit_cap_d split half to each end node; zero resistances clamped to
 *      1e-6 kOhm.
 * Distances (the MST decisions) are fp32, as on the device (S1);
 * resistances and capacitances are accumulated in fp64 and stored as float.
 * Output in the sta_set_rc_tree layout: net n owns nodes [rc_ptr[n],
 * rc_ptr[n+1]), node 0 the driver (parent -1), parents local and < child;
 * nodes in Prim order, each Steiner node right before its pin.  Capacity of
 * the node arrays: 2 * net_ptr[N] - N suffices.  Returns the node count. */
static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

static float mdist(const float* x, const float* y, uint32_t a, uint32_t b) {
  return fabsf(x[a] - x[b]) + fabsf(y[a] - y[b]);
}

uint32_t orc_steiner(uint32_t N, const uint32_t* net_ptr, const uint32_t* net_pins, const float* x,
                     const float* y, double rx, double ry, double cx, double cy, uint32_t* rc_ptr,
                     int32_t* parent, uint32_t* node_pin, float* res, float* cap) {
  uint32_t nn = 0, maxn = 1;
  for (uint32_t n = 0; n < N; ++n)
    if (net_ptr[n + 1] - net_ptr[n] > maxn) maxn = net_ptr[n + 1] - net_ptr[n];
  uint32_t* pin = malloc(sizeof(uint32_t) * maxn);     /* step 1: driver, sinks by id */
  uint32_t* par = malloc(sizeof(uint32_t) * maxn);     /* tree parent (index into pin) */
  uint32_t* node_of = malloc(sizeof(uint32_t) * maxn); /* local node of each pin */
  char* in_tree = malloc(maxn);
  float* key = malloc(sizeof(float) * maxn);
  double* c = malloc(sizeof(double) * 2 * maxn);       /* node caps of the net */
  for (uint32_t n = 0; n < N; ++n) {
    const uint32_t m = net_ptr[n + 1] - net_ptr[n], base = nn;
    rc_ptr[n] = nn;
    for (uint32_t k = 0; k < m; ++k) pin[k] = net_pins[net_ptr[n] + k];
    if (m > 1) qsort(pin + 1, m - 1, sizeof(uint32_t), cmp_u32);
    /* step 2: Prim */
    for (uint32_t k = 0; k < m; ++k) {
      in_tree[k] = k == 0;
      key[k] = k ? mdist(x, y, pin[0], pin[k]) : 0.f;
      par[k] = 0;
    }
    uint32_t local = 0;
    parent[base] = -1;
    node_pin[base] = pin[0];
    res[base] = 0.f;
    c[0] = 0.0;
    node_of[0] = local++;
    for (uint32_t step = 1; step < m; ++step) {
      uint32_t best = 0;
      for (uint32_t k = 1; k < m; ++k) {
        if (in_tree[k]) continue;
        if (!best || key[k] < key[best] || (key[k] == key[best] && pin[k] < pin[best])) best = k;
      }
      in_tree[best] = 1;
      /* step 3: emit the edge par[best] -> best as an L, horizontal leg first */
      const uint32_t p = par[best], u = pin[p], v = pin[best];
      const float dx = fabsf(x[v] - x[u]), dy = fabsf(y[v] - y[u]);
      uint32_t up = node_of[p];
      if (dx != 0.f && dy != 0.f) {                    /* Steiner bend at (x_v, y_u) */
        const uint32_t b = local++;
        parent[base + b] = (int32_t)up;
        node_pin[base + b] = ORC_NO_PIN;
        res[base + b] = (float)((double)dx * rx > 0 ? (double)dx * rx : 1e-6);
        c[up] += 0.5 * dx * cx;
        c[b] = 0.5 * dx * cx + 0.5 * dy * cy;
        up = b;
        const uint32_t w = local++;
        parent[base + w] = (int32_t)up;
        node_pin[base + w] = v;
        res[base + w] = (float)((double)dy * ry > 0 ? (double)dy * ry : 1e-6);
        c[w] = 0.5 * dy * cy;
        node_of[best] = w;
      } else {                                         /* one straight leg (or none) */
        const double L_r = dy == 0.f ? (double)dx * rx : (double)dy * ry;
        const double L_c = dy == 0.f ? (double)dx * cx : (double)dy * cy;
        const uint32_t w = local++;
        parent[base + w] = (int32_t)up;
        node_pin[base + w] = v;
        res[base + w] = (float)(L_r > 0 ? L_r : 1e-6);
        c[up] += 0.5 * L_c;
        c[w] = 0.5 * L_c;
        node_of[best] = w;
      }
      /* Prim key update with the new tree pin */
      for (uint32_t k = 1; k < m; ++k) {
        if (in_tree[k]) continue;
        const float d = mdist(x, y, v, pin[k]);
        if (d < key[k]) {
          key[k] = d;
          par[k] = best;
        }
      }
    }
    for (uint32_t k = 0; k < local; ++k) cap[base + k] = (float)c[k];
    nn += local;
  }
  rc_ptr[N] = nn;
  free(pin); free(par); free(node_of); free(in_tree); free(key); free(c);
  return nn;
}
