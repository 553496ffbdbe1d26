/*
 * sta_oracle.h -- plain, slow, single-thread fp64 CPU oracle of one full
 * graph-based STA timing update (HeteroSTA, arxiv 2511.11660).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2511_11660_b200/csrc, include/sta.h).
 *
 * What it computes follows SURVEY.md §8(c) steps O1-O9 (textbook max/min-plus
 * STA; the paper names the reports -- "WNS/TNS, pin slacks", PAPER.md:187 --
 * but not the formulas, which come from SPEC.md:371-532).  Every readings the
 * paper leaves open is listed in DESIGN.md §2.
 *
 * Layout of per-pin quantities: double[P][4] in (early_rise, early_fall,
 * late_rise, late_fall) order, indexed by the caller's pin id.
 */
#ifndef STA_ORACLE_H
#define STA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_POS = 0, ORC_NEG = 1, ORC_NON = 2, ORC_RISE_EDGE = 3, ORC_FALL_EDGE = 4 };
enum { ORC_INTERNAL = 0, ORC_PI = 1, ORC_PO = 2, ORC_FF_CK = 3, ORC_FF_D = 4 };
#define ORC_NO_PIN 0xFFFFFFFFu

typedef struct {
  /* netlist */
  uint32_t num_pins;
  const float* pin_cap;      /* [P] fF */
  const uint8_t* pin_role;   /* [P] */
  uint32_t num_nets;
  const uint32_t* net_ptr;   /* [N+1] */
  const uint32_t* net_pins;  /* driver first */
  uint32_t num_arcs;
  const uint32_t* arc_from;
  const uint32_t* arc_to;
  const uint8_t* arc_sense;
  const uint32_t* arc_tab;   /* base of cell_rise, cell_fall, rise_tr, fall_tr */
  uint32_t num_checks;
  const uint32_t* chk_d;
  const uint32_t* chk_ck;
  const uint32_t* chk_tab;   /* base of setup_r, setup_f, hold_r, hold_f */
  /* one corner's NLDM table pool */
  uint32_t num_tables;
  const uint8_t* tab_n1;
  const uint8_t* tab_n2;
  const uint32_t* tab_off;
  const float* tab_data;
  /* one corner's RC trees */
  const uint32_t* rc_ptr;    /* [N+1] */
  const int32_t* rc_parent;  /* local parent, -1 at node 0 */
  const uint32_t* rc_node_pin;
  const float* rc_res;       /* kOhm, edge parent->i */
  const float* rc_cap;       /* fF, wire cap at node i */
  /* constraints: one ideal clock */
  double period;
  double clock_slew;
  uint32_t n_pi;
  const uint32_t* pi_pin;
  const float* pi_at;        /* [n_pi][4] */
  const float* pi_slew;      /* [n_pi][4] */
  uint32_t n_po;
  const uint32_t* po_pin;
  const float* po_out_max;   /* [n_po][2] rise, fall */
  const float* po_out_min;   /* [n_po][2] */
  const float* po_load;      /* [n_po] fF */
  /* net-arc delay model: 0 Elmore (O3), 1 Arnoldi
   * reduced-order model of order arnoldi_q (O12) */
  int32_t net_model;
  uint32_t arnoldi_q;
  /* -from / -to timing exceptions: kind 0 false
   * path, 1 multicycle (value N), 2 max delay (value ps), 3 min delay (value
   * ps); CSR lists of startpoint / endpoint pins (an empty list: any) */
  uint32_t n_exc;
  const uint8_t* exc_kind;
  const float* exc_value;
  const uint32_t* exc_from_ptr;
  const uint32_t* exc_from;
  const uint32_t* exc_to_ptr;
  const uint32_t* exc_to;
  /* multiple ideal clocks (row f4, O14): n_clk periods; pin_clk[P] = the
   * clock of each FF_CK pin, the launch clock of each PI, the capture clock
   * of each PO (n_clk = 0: the single clock `period`) */
  uint32_t n_clk;
  const float* clk_period;
  const uint32_t* pin_clk;
  /* -through segments (row f4, O15): exception i's ordered
   * through segments are the segment ids exc_thr_ptr[i] .. exc_thr_ptr[i+1];
   * segment s holds the pins exc_seg[exc_seg_ptr[s] .. exc_seg_ptr[s+1]).
   * exc_thr_ptr NULL: no exception has -through. */
  const uint32_t* exc_thr_ptr;
  const uint32_t* exc_seg_ptr;
  const uint32_t* exc_seg;
  /* case analysis (row f4, O16): logic functions of cell
   * output pins -- pin fn_pin[i] = truth table fn_tt[i] over the pins
   * fn_in[fn_in_ptr[i] .. fn_in_ptr[i+1]) (<= 6; input j = bit j of the
   * table index); optional `when` guards per cell arc, arc_when[a] a truth
   * table over the inputs of fn(arc_to[a]) (all ones: no guard; NULL: no
   * guards); constants case_pin[k] = case_val[k] (0 / 1).  n_fn = n_case = 0
   * and arc_when NULL: no case analysis. */
  uint32_t n_fn;
  const uint32_t* fn_pin;
  const uint32_t* fn_in_ptr;
  const uint32_t* fn_in;
  const uint64_t* fn_tt;
  const uint64_t* arc_when;
  uint32_t n_case;
  const uint32_t* case_pin;
  const uint8_t* case_val;
} orc_design;

/* O16: case analysis alone -- val[P] (0, 1, 2 = not constant) and, per
 * canonical arc (net arcs net by net, then cell arcs),
 * off[E] = 1 where the arc is disabled.  Returns 0, 6 on contradictory
 * constants, 7 on a function with more than 6 inputs, 2 on allocation. */
int orc_case_analysis(const orc_design* d, uint8_t* val, uint8_t* off);

/* O6: NLDM bilinear lookup, fp64.  `tab` points at
 * index_1[n1], index_2[n2], values[n1][n2]. */
double orc_lut(uint32_t n1, uint32_t n2, const float* tab, double s, double c);

/* O2: Kahn levelization over net + cell arcs.
 * level[P], perm[P] (stable sort by (level, pin id)).  Returns 0, or 1 on a
 * combinational cycle. */
int orc_levelize(const orc_design* d, uint32_t* level, uint32_t* perm, uint32_t* num_levels);

/* O3: per-net Elmore.  load[N] = total net cap (fF),
 * elm[P] = Elmore delay of the net arc into each sink pin (0 for non-sinks). */
void orc_rc(const orc_design* d, double* load, double* elm);

/* O1-O8: full update.  at/slew/rat/slack: double[P][4] (may be NULL except
 * at); res[4] = {WNS_setup, TNS_setup, WNS_hold, TNS_hold};
 * ep_pin/ep_ws (optional, [n_ep] and [n_ep][2]) receive the endpoints in
 * increasing pin id with their worst setup/hold slack.  Returns 0, 1 on a
 * cycle, 2 on allocation failure.  *n_ep receives the endpoint count. */
int orc_update(const orc_design* d, double* at, double* slew, double* rat, double* slack,
               double res[4], uint32_t* ep_pin, double* ep_ws, uint32_t* n_ep);

/* O10: top-k path report (the
 * readings are in sta_oracle.c and DESIGN.md).  mode 0 setup, 1 hold; k >= 1
 * paths in all, nworst >= 1 per endpoint, slack < slack_lt.  CSR output:
 * path i = pins path_pin[path_ptr[i] .. path_ptr[i+1]) (startpoint first) with
 * their transitions (0 rise, 1 fall) and the path's arrival at each;
 * path_slack / path_ep per path, in report order.  Returns 0, 1 on a cycle,
 * 2 on allocation failure, 3 when a capacity is too small. */
int orc_paths(const orc_design* d, int mode, uint32_t k, uint32_t nworst, double slack_lt, uint32_t cap_paths,
              uint32_t cap_pins, uint32_t* n_paths, uint32_t* n_pins, uint32_t* path_ptr, uint32_t* path_pin,
              uint8_t* path_rf, double* path_at, double* path_slack, uint32_t* path_ep);

/* O11: built-in Steiner RC from pin positions (
 * PAPER.md:178-179): rectilinear MST by Prim from the
 * driver (fp32 Manhattan distances, ties by smaller pin id), L-embedded edges
 * (horizontal leg first from the parent), half-split leg caps.  Writes the
 * sta_set_rc_tree / sta_set_rc_values arrays (rc_ptr[N+1]; parent, node_pin,
 * res, cap with capacity >= 2 * net_ptr[N] - N) and returns the node count. */
uint32_t orc_steiner(uint32_t N, const uint32_t* net_ptr, const uint32_t* net_pins, const float* x,
                     const float* y, double rx, double ry, double cx, double cy, uint32_t* rc_ptr,
                     int32_t* parent, uint32_t* node_pin, float* res, float* cap);

/* O12: Arnoldi reduced-order net model (PAPER.md:182-183,
 * 209; readings A1-A7 in DESIGN.md).
 * orc_arnoldi_reduce: one net's RC tree (m nodes, node 0 the driven root,
 * parent[i] < i local, res[i] of the edge parent -> i, cap[i] the node's total
 * grounded cap incl. pin caps): Lanczos in the C-inner product on A = G^-1 C
 * from the start vector G^-1 b = 1, each A application one O(m) tree solve,
 * full reorthogonalisation, order <= q (breakdown truncates).  Writes the
 * reduced time constants lam[k] = -1/pole_k (>= 0) and per-node residues
 * resid[i*q + k] (H_i(s) = sum_k resid / (1 + s lam_k), sum_k resid = 1).
 * Returns the achieved order, or -1 if the model is unstable (a negative
 * time constant: callers fall back to Elmore).
 * orc_arnoldi_delay: the response of the reduced model to a saturated ramp
 * of 20-80 slew `slew` (duration slew / 0.6): delay = t50(out) - t50(in) and
 * *out_slew = t80 - t20 of the output, crossings by bisection to 1e-6 ps. */
int orc_arnoldi_reduce(uint32_t m, const int32_t* parent, const float* res, const double* cap, uint32_t q,
                       double* lam, double* resid);
double orc_arnoldi_delay(uint32_t qq, const double* lam, const double* k, double slew, double* out_slew);

#ifdef __cplusplus
}
#endif
#endif
