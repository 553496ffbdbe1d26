/*
 * sta.h -- C ABI of the B200-native graph-based STA hot path
 *          (HeteroSTA, arxiv 2511.11660, re-designed for sm_100a).
 *
 * The paper's boundary is a "zero-overhead flattened heterogeneous API"
 * (PAPER.md:39, 131-134): the netlist arrives as CSR arrays (PAPER.md:166-171,
 * "accepts external net and cell CSR arrays directly ... eliminates the need to
 * ... maintain pin indices mappings"), parasitics as a flattened RC structure
 * "on either CPU or GPU", reports are "WNS/TNS, pin slacks"
 * and "all output arrays can be on CPU or GPU at user's option"
 * (PAPER.md:191); the deliverable is a ".so" plus "C header files"
 * (PAPER.md:198).  Every entry point below is one of those calls.
 *
 * Units: ps, fF, kOhm (kOhm * fF = ps).  Ids are the caller's 0-based ids and
 * are never re-indexed: every per-pin input and output is indexed by the
 * caller's pin id.  Per-pin timing quantities are float[4] in the order
 * (early_rise, early_fall, late_rise, late_fall).
 *
 * Memory: each pointer argument is tagged by an sta_mem flag.  STA_MEM_HOST
 * pointers are read (or written) before the call returns; the caller may free
 * them afterwards.  STA_MEM_DEVICE pointers are CUDA device pointers on the
 * ctx's device; inputs are copied device-to-device in stream order, except
 * sta_set_rc_values which BORROWS them (zero copy, see there).  The library
 * never hands out memory; outputs go to caller buffers.
 *
 * Errors: every call returns an sta_status; nothing throws across the ABI.
 * sta_last_error(ctx) names the offending index ("net 17: offsets not
 * monotone").  A CUDA failure poisons the ctx: every later call except
 * sta_destroy / sta_last_error returns STA_ERR_CUDA.
 *
 * Async: sta_update_timing only enqueues work on the ctx stream.  Calls that
 * write HOST buffers synchronize the stream; calls that write DEVICE buffers
 * are stream ordered.
 *
 * Threading: a ctx is used by one host thread at a time; there is no global
 * state, so independent ctxs may run concurrently.
 */
#ifndef STA_H
#define STA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define STA_API __attribute__((visibility("default")))
#else
#define STA_API
#endif

typedef struct sta_ctx_s* sta_ctx;

typedef enum {
  STA_OK = 0,
  STA_ERR_ARG = 1,         /* NULL pointer, bad count, enum or corner index, role mismatch */
  STA_ERR_CSR = 2,         /* CSR offsets not starting at 0, not monotone, empty net */
  STA_ERR_ID = 3,          /* pin / table id out of range */
  STA_ERR_MULTIDRIVER = 4, /* pin in two nets, or driven by a net and a cell arc */
  STA_ERR_CYCLE = 5,       /* combinational cycle through net + cell arcs */
  STA_ERR_LUT = 6,         /* table size outside 1..8, axes not strictly ascending, non-finite */
  STA_ERR_RC = 7,          /* RC tree malformed, or R/C negative or non-finite */
  STA_ERR_ORDER = 8,       /* call order violated (see sta_update_timing) */
  STA_ERR_CUDA = 9,        /* CUDA runtime failure; ctx poisoned */
  STA_ERR_OOM = 10         /* device or host allocation failed */
} sta_status;

typedef enum { STA_MEM_HOST = 0, STA_MEM_DEVICE = 1 } sta_mem;

/* Timing sense of a cell arc. */
typedef enum {
  STA_POS_UNATE = 0,   /* r->r, f->f */
  STA_NEG_UNATE = 1,   /* r->f, f->r */
  STA_NON_UNATE = 2,   /* all four (late: worst, early: best) */
  STA_RISE_EDGE = 3,   /* clock-to-Q of a rising-edge register: r->r, r->f */
  STA_FALL_EDGE = 4    /* f->r, f->f */
} sta_sense;

/* Pin roles.  PI and FF_CK pins must have no fan-in.  FF_CK pins are ideal
 * clock sources: arrival (0, T/2) for (rise, fall), slew = clock_slew
 * (SPEC.md:542).  FF_D pins are the data pins of check arcs. */
typedef enum {
  STA_PIN_INTERNAL = 0, STA_PIN_PI = 1, STA_PIN_PO = 2, STA_PIN_FF_CK = 3, STA_PIN_FF_D = 4
} sta_pin_role;

#define STA_NO_PIN 0xFFFFFFFFu

/* ------------------------------------------------------------- lifecycle */

/* Create a context on `cuda_device` for `num_corners` >= 1 analysis corners.
 * `cuda_stream` is a cudaStream_t to enqueue on, or NULL for a stream the ctx
 * creates and owns.  *out receives the handle. */
STA_API sta_status sta_create(int cuda_device, uint32_t num_corners, void* cuda_stream, sta_ctx* out);

/* Synchronize and release every resource of ctx.  NULL is a no-op. */
STA_API sta_status sta_destroy(sta_ctx ctx);

/* Message of the last failed call on ctx (valid until the next call). */
STA_API const char* sta_last_error(sta_ctx ctx);

/* Static name of a status code. */
STA_API const char* sta_status_string(sta_status st);

/* ---------------------------------------------------------------- inputs */

/* Flattened netlist.
 *  - num_pins P, pin_cap[P] (fF, input pin capacitance), pin_role[P].
 *  - nets: net_ptr[N+1] offsets into net_pins; net n = net_pins[net_ptr[n] ..
 *    net_ptr[n+1]); its FIRST entry is the driver, the rest are sinks.  Every
 *    net has a driver; a pin belongs to at most one net.  Each sink gets one
 *    net arc (driver -> sink), positive unate.
 *  - cell arcs a < num_arcs: arc_from[a] -> arc_to[a] with arc_sense[a] and
 *    arc_tab[a] = id of the first of 4 consecutive tables (cell_rise,
 *    cell_fall, rise_transition, fall_transition).  A cell-arc target must not
 *    also be a net sink.
 *  - checks c < num_checks: data pin chk_d[c] (role FF_D), clock pin
 *    chk_ck[c] (role FF_CK), chk_tab[c] = first of 4 tables (setup_rise,
 *    setup_fall, hold_rise, hold_fall), indexed by (data slew, clock slew).
 *    Checks create endpoints, not graph edges.
 *  - num_tables: size of every corner's table pool; every table id used above
 *    (+3) must be < num_tables.
 * Arrays are all HOST or all DEVICE (`mem`); arrays of a zero count may be NULL. */
typedef struct {
  sta_mem mem;
  uint32_t num_pins;
  const float* pin_cap;
  const uint8_t* pin_role;
  uint32_t num_nets;
  const uint32_t* net_ptr;
  const uint32_t* net_pins;
  uint32_t num_arcs;
  const uint32_t* arc_from;
  const uint32_t* arc_to;
  const uint8_t* arc_sense;
  const uint32_t* arc_tab;
  uint32_t num_checks;
  const uint32_t* chk_d;
  const uint32_t* chk_ck;
  const uint32_t* chk_tab;
  uint32_t num_tables;
} sta_graph_desc;

/* Validate the netlist, levelize it (longest-path pin levels over net + cell
 * arcs) and build the device-resident timing graph.  Runs
 * once per design; resets every library / RC / constraint input.
 * Errors: STA_ERR_ARG, STA_ERR_CSR, STA_ERR_ID, STA_ERR_MULTIDRIVER,
 * STA_ERR_CYCLE, STA_ERR_OOM, STA_ERR_CUDA. */
STA_API sta_status sta_load_graph(sta_ctx ctx, const sta_graph_desc* desc);

/* NLDM table pool of one corner (SPEC.md:30-45 Lut2D).
 * Table t: n1[t], n2[t] in 1..8, data[off[t] ...] = index_1[n1] (input slew
 * ps; data slew for constraint tables), index_2[n2] (load fF; clock slew for
 * constraint tables), values[n1][n2] row-major (ps).  Axes strictly
 * ascending.  Corners may use different axes (pool sizes may differ).
 * Copied (small).  Errors: STA_ERR_ARG, STA_ERR_LUT. */
STA_API sta_status sta_set_library(sta_ctx ctx, uint32_t corner, sta_mem mem, uint32_t num_tables,
                           const uint8_t* n1, const uint8_t* n2, const uint32_t* off,
                           const float* data, uint32_t data_len);

/* RC tree topology, shared by all corners ("a set of predefined
 * CSR structures").  Net n owns nodes
 * [rc_ptr[n], rc_ptr[n+1]) (rc_ptr[N] = num_nodes).  Within a net, node 0 is
 * the driver (parent -1), parent[i] is a LOCAL index < i, node_pin[i] is a
 * pin of that net or STA_NO_PIN (Steiner/wire node).  If a net has nodes,
 * each of its sinks maps to exactly one node and node 0 maps to the driver or
 * STA_NO_PIN.  A net without nodes is lumped (load = its pin caps + PO
 * loads, zero wire delay).  Copied.  Errors: STA_ERR_ORDER (no graph),
 * STA_ERR_ARG, STA_ERR_CSR, STA_ERR_RC. */
STA_API sta_status sta_set_rc_tree(sta_ctx ctx, sta_mem mem, const uint32_t* rc_ptr, uint32_t num_nodes,
                           const int32_t* parent, const uint32_t* node_pin);

/* Built-in Steiner RC estimation from pin positions (
 * "A placer only needs to provide HeteroSTA with pin
 * positions and unit resistance/capacitance values along x/y directions";
 * construction SPEC.md:322-331 with its decisions SPEC.md:338-343).  For
 * every net of the loaded graph: its pins (driver, then sinks by pin id) are
 * joined by a rectilinear minimum spanning tree (Prim from the driver, fp32
 * Manhattan distances, ties by the smaller pin id), every tree edge is
 * embedded as an L (horizontal leg first from the parent, one Steiner node
 * at the bend when both legs are non-zero), a leg of length L along x/y has
 * resistance L * res_x/res_y (zero clamped to 1e-6 kOhm) and puts
 * L * cap_x/cap_y / 2 on each end node.  Runs on the device (one warp or
 * block per net); Prim is O(m^2) in the net's pin count m.
 *  - pin_x[P], pin_y[P]: positions (distance units), finite, in `mem`
 *    memory; units: all >= 0 and finite.
 *  - outputs, in `mem` memory, in the layout sta_set_rc_tree /
 *    sta_set_rc_values take: rc_ptr[N+1]; parent, node_pin, res, cap of
 *    node_capacity entries, which must be >= 2 * (pins on nets) - N (the
 *    largest possible node count); *num_nodes (host) receives the count.
 *  Nodes of a net are in Prim order, each Steiner node right before its
 *  pin; node 0 is the driver.  The call synchronizes the ctx stream.
 * Errors: STA_ERR_ORDER (no graph), STA_ERR_ARG (capacity, units, NULL
 * outputs, non-finite host positions), STA_ERR_CUDA. */
typedef struct {
  float res_x, res_y;   /* kOhm per distance unit */
  float cap_x, cap_y;   /* fF per distance unit */
} sta_steiner_units;

STA_API sta_status sta_build_steiner(sta_ctx ctx, sta_mem mem, const float* pin_x, const float* pin_y,
                             const sta_steiner_units* units, uint32_t node_capacity, uint32_t* rc_ptr,
                             int32_t* parent, uint32_t* node_pin, float* res, float* cap,
                             uint32_t* num_nodes);

/* Net-arc delay model of the next updates (
 * "The Elmore model is the fastest yet not accurate
 * enough in late design stages, where Arnoldi might be a better option";
 * SPEC.md:398-418).  STA_NET_ELMORE (default): Elmore delay, PERI slew.
 * STA_NET_ARNOLDI: per net and corner a Lanczos (Arnoldi on the symmetric
 * RC-tree pencil) reduced-order model of order q (1..4) is built on the
 * device every update; a sink's delay and slew are the response of that
 * model to a saturated ramp of the driver's 20-80 slew (delay = 50% crossing
 * minus the input's, slew = 20-80 crossing difference), evaluated wherever
 * the sink's arrival is needed; an unstable model falls back to Elmore for
 * its net.  Readings A1-A7 in DESIGN.md.  The top-k path report is Elmore
 * only (sta_report_paths returns STA_ERR_ORDER under Arnoldi).
 * Errors: STA_ERR_ARG (model, q). */
typedef enum { STA_NET_ELMORE = 0, STA_NET_ARNOLDI = 1 } sta_net_model;
STA_API sta_status sta_set_net_model(sta_ctx ctx, sta_net_model model, uint32_t q);

/* Timing exceptions ("false
 * paths, multi-cycle paths, case analysis, and cross clock region paths ...
 * complicate the data structures and states in timing propagation"; PAPER.md:
 * 250: "-through patterns that eliminate only paths that go through a
 * predefined pin sequence"; the tag model of SPEC.md:465-509; case
 * analysis: sta_set_case_analysis).  Exception i: kind[i] (STA_EXC_*), value[i] (multicycle:
 * N >= 1; max / min delay: ps), startpoint pins from_pins[from_ptr[i] ..
 * from_ptr[i+1]), endpoint pins to_pins[to_ptr[i] .. to_ptr[i+1]) (an empty
 * list: any) and, if thr_ptr is not NULL, the ordered -through segments
 * thr_ptr[i] .. thr_ptr[i+1], segment g holding the pins
 * seg_pins[seg_ptr[g] .. seg_ptr[g+1]) (non-empty).  A path matches
 * exception i when its startpoint is in the -from list and it passes a pin
 * of every -through segment in order (X8: one pin may match
 * consecutive segments).  A path's tag is its launch clock and the matched
 * prefix of every exception's segments (one bit per segment); tags advance
 * at -through pins; every tag is propagated as its own pass (RC shared; with
 * -through a forward sweep hands the arrivals of advancing tags on, then
 * full passes in reverse order take the required times back), and per
 * endpoint and tag the fully matched exceptions are resolved: setup (late):
 * false path > max delay (RAT_L = value) > multicycle (capture at N T); hold
 * (early): false path > min delay (RAT_E = value) > multicycle (hold edge
 * (N-1) T); the first listed of a kind wins.  Reports merge the tags: per
 * pin the early / late extreme of AT, slew, RAT and the minimum slack; per
 * endpoint the worst slack over tags (false paths contribute none) for
 * WNS / TNS.  num = 0 clears.  At most 32 exceptions, 32 segments (-from
 * lists and -through segments) and 32 tags.  The top-k path report needs no
 * exceptions (STA_ERR_ORDER).  Arrays in `mem`, copied.  Errors:
 * STA_ERR_ORDER (no graph), STA_ERR_ARG (kinds, values, limits), STA_ERR_CSR
 * (offsets, empty segment), STA_ERR_ID (pin out of range). */
typedef enum { STA_EXC_FALSE_PATH = 0, STA_EXC_MULTICYCLE = 1, STA_EXC_MAX_DELAY = 2,
               STA_EXC_MIN_DELAY = 3 } sta_exception_kind;
typedef struct {
  sta_mem mem;
  uint32_t num;
  const uint8_t* kind;
  const float* value;
  const uint32_t* from_ptr;
  const uint32_t* from_pins;
  const uint32_t* to_ptr;
  const uint32_t* to_pins;
  const uint32_t* thr_ptr;    /* [num + 1] or NULL: no -through */
  const uint32_t* seg_ptr;    /* [thr_ptr[num] + 1] */
  const uint32_t* seg_pins;
} sta_exceptions;
STA_API sta_status sta_set_exceptions(sta_ctx ctx, const sta_exceptions* ex);

/* Case analysis ("case analysis
 * modes", apply_case_analysis).  Logic functions of cell
 * output pins: pin fn_pin[i] = truth table fn_tt[i] over the pins
 * fn_in[fn_in_ptr[i] .. fn_in_ptr[i+1]) (at most 6; bit m of the table is
 * the output when input j has the value of bit j of m); arc_when (NULL: no
 * guards) = per cell arc a truth table over the inputs of the function of
 * arc_to[a] (all ones: no guard); constants case_pin[k] = case_val[k] (0 /
 * 1).  Constants are carried over nets (a sink takes its driver's constant)
 * and through the functions (an output is constant when its function takes
 * one value for every completion of its non-constant inputs), in
 * topological order; every arc from or to a constant pin and every cell arc
 * whose guard is false for every completion is disabled: nothing
 * propagates over it in either direction (a pin whose fan-in is all
 * disabled has no arrival, C1-C4).  num_fn = num_case = 0 and
 * arc_when NULL clear.  Arrays in `mem`, copied; applied at the next
 * update.  Errors: STA_ERR_ORDER (no graph), STA_ERR_ID (pin out of range),
 * STA_ERR_CSR (offsets), STA_ERR_ARG (more than 6 inputs, a pin with two
 * functions, values other than 0 / 1; contradictory constants on a pin are
 * reported by the next sta_update_timing). */
typedef struct {
  sta_mem mem;
  uint32_t num_fn;
  const uint32_t* fn_pin;     /* [num_fn] */
  const uint32_t* fn_in_ptr;  /* [num_fn + 1] */
  const uint32_t* fn_in;
  const uint64_t* fn_tt;      /* [num_fn] */
  const uint64_t* arc_when;   /* [num_arcs] or NULL */
  uint32_t num_case;
  const uint32_t* case_pin;   /* [num_case] */
  const uint8_t* case_val;    /* [num_case] 0 / 1 */
} sta_case_analysis;
STA_API sta_status sta_set_case_analysis(sta_ctx ctx, const sta_case_analysis* ca);

/* Multiple ideal clocks ("cross clock region
 * paths"; the relationship rule of SPEC.md:504).  Clock k:
 * period_ps[k], rising edges at multiples of the period, waveform (0, T/2).
 * pin_clk[P]: the clock of each FF_CK pin (its register), the launch clock
 * of each PI (the input delay's clock) and the capture clock of each PO
 * (the output delay's clock); other entries are ignored.  Startpoints are
 * tagged by their launch clock (and their -from exceptions) and propagated
 * per tag; an endpoint's setup edge is the first capture edge after the
 * launch edge, its hold edge the capture edge before that, taken over the
 * first 1000 launch edges (the most restrictive pair); multicycle shifts use
 * the capture period.  num_clocks = 0: one clock, the constraints' period.
 * At most 16 clocks.  Arrays in `mem`, copied.  Errors: STA_ERR_ORDER,
 * STA_ERR_ARG, STA_ERR_ID. */
typedef struct {
  sta_mem mem;
  uint32_t num_clocks;
  const float* period_ps;
  const uint32_t* pin_clk;
} sta_clocks;
STA_API sta_status sta_set_clocks(sta_ctx ctx, const sta_clocks* clk);

/* Per-corner RC values: res[i] = resistance of the edge parent -> i (kOhm,
 * ignored at node 0), cap[i] = wire capacitance to ground at node i (fF);
 * both num_nodes long, >= 0 and finite.  HOST: copied into ctx-owned device
 * buffers before the call returns (page-locked buffers move by DMA at link
 * speed); the ctx keeps two buffer pairs per corner and copies on its own
 * copy stream into the pair no enqueued update reads, so the copy of the
 * next iteration's values runs beside an update still in flight; the next
 * update is ordered after the copy.  DEVICE: BORROWED, zero copy -- the caller keeps both
 * arrays alive and unmodified until the next sta_update_timing has completed
 * on the ctx stream; the call itself never blocks the host (the pointer pair
 * is published by a stream-ordered one-thread kernel), so the next
 * iteration's inputs can be produced while an update runs.  In both cases the
 * values are validated on the device by the RC kernels: a bad value is
 * reported as STA_ERR_RC by the next synchronizing call.  This is the
 * per-iteration call of an optimization loop. */
STA_API sta_status sta_set_rc_values(sta_ctx ctx, uint32_t corner, sta_mem mem, const float* res,
                             const float* cap);

/* One ideal clock plus port constraints.
 *  - period_ps > 0 (setup capture edge), clock_slew_ps >= 0.
 *  - PIs: pi_pin[k] (role PI), pi_at[k][4], pi_slew[k][4] (finite).  A PI pin
 *    not listed is an undefined source (no arrival).
 *  - POs: po_pin[k] (role PO), po_out_max[k][2], po_out_min[k][2]
 *    (rise, fall output delays), po_load_ff[k] added to the PO pin's node cap.
 * All arrays HOST or DEVICE per `mem`; copied.  Errors: STA_ERR_ORDER,
 * STA_ERR_ARG, STA_ERR_ID. */
typedef struct {
  sta_mem mem;
  float period_ps;
  float clock_slew_ps;
  uint32_t n_pi;
  const uint32_t* pi_pin;
  const float* pi_at;
  const float* pi_slew;
  uint32_t n_po;
  const uint32_t* po_pin;
  const float* po_out_max;
  const float* po_out_min;
  const float* po_load_ff;
} sta_constraints;
STA_API sta_status sta_set_constraints(sta_ctx ctx, const sta_constraints* cons);

/* --------------------------------------------------------------- update */

/* One full timing update for every corner of ctx, enqueued on the ctx
 * stream: Elmore RC and loads, forward AT/slew with NLDM cell delays, endpoint
 * required-time seeds, backward RAT, per-pin slack, WNS/TNS (SURVEY.md §8(a)
 * a1-a5).  Up to 8 corners are traversed by the same kernel launches (their
 * level-by-level wavefronts advance together).  Requires sta_load_graph, sta_set_rc_tree, sta_set_constraints and,
 * for every corner, sta_set_library and sta_set_rc_values (else
 * STA_ERR_ORDER).  Asynchronous: errors of the kernels surface at the next
 * synchronizing call. */
STA_API sta_status sta_update_timing(sta_ctx ctx);

/* ------------------------------------------------------------- reports */

/* Results of `corner` after the last update.
 *  - res4 (may be NULL): double[4] {WNS_setup, TNS_setup, WNS_hold, TNS_hold}
 *    in ps, in `mem` memory.  WNS = min over endpoints (PO pins and check data
 *    pins) of the worst (over rise/fall) slack, +inf if none is constrained;
 *    TNS = sum over endpoints of min(0, worst slack), accumulated in fp64
 *    (SPEC.md:515-523, 547).  HOST: synchronizes and reports deferred errors;
 *    DEVICE: stream ordered (for a device-side allreduce across ranks).
 *  - pin_slack (may be NULL): float[P][4] per pin (hold rise, hold fall, setup
 *    rise, setup fall) = (AT_E - RAT_E, AT_E - RAT_E, RAT_L - AT_L, RAT_L -
 *    AT_L), +inf where either side is undefined, in `mem` memory. */
STA_API sta_status sta_report_slack(sta_ctx ctx, uint32_t corner, double* res4, float* pin_slack,
                            sta_mem mem);

/* Full per-pin state of `corner` (any pointer may be NULL): at, slew, rat as
 * float[P][4].  Undefined components are +inf (early) / -inf (late) for at
 * and slew and -inf (early) / +inf (late) for rat. */
STA_API sta_status sta_get_timing(sta_ctx ctx, uint32_t corner, float* at, float* slew, float* rat,
                          sta_mem mem);

/* Delay-calculation results of `corner` (either pointer may be NULL):
 * net_load[N] (fF, the NLDM load of each net's driver) and pin_elm[P] (the
 * Elmore delay of the net arc into each sink pin, 0 for non-sinks). */
STA_API sta_status sta_get_rc(sta_ctx ctx, uint32_t corner, float* net_load, float* pin_elm,
                      sta_mem mem);

/* Levelization of the loaded graph: level[P] = longest-path depth of each
 * pin (0 without fan-in), perm[P] = pins stably sorted by (level, pin id),
 * *num_levels = max level + 1 (HOST).  level/perm may be NULL. */
STA_API sta_status sta_get_levels(sta_ctx ctx, uint32_t* level, uint32_t* perm, uint32_t* num_levels,
                          sta_mem mem);

/* Top-k path report of `corner` after the last update (
 * "top-k path reports ... controlled with top-k,
 * per-endpoint report limit, and slack-less-than thresholds ... flattened
 * CSR-based path pin arrays with slacks").  A path is a sequence of
 * (pin, transition) from a startpoint with an arrival (PI, ideal clock pin)
 * to an endpoint (PO, checked data pin) along enabled arcs; its arrival is
 * the startpoint's plus the delays the update used on its arcs (graph-based);
 * setup slack = the endpoint's own required time (check / output delay) -
 * arrival (late), hold slack = arrival - required (early).  Paths are
 * reported in the order (slack, endpoint pin id, the (pin, transition)
 * sequence read backwards from the endpoint), keeping slack < slack_lt, at
 * most nworst per endpoint, k in all (1 <= min(k, nworst) <= 255).
 * The first setup path's slack is the worst endpoint slack.
 * Output (in `mem` memory; capacities cap_paths >= k and cap_pins, e.g.
 * k * (num_levels + 1)): path i has pins path_pin[path_ptr[i] ..
 * path_ptr[i + 1]) startpoint first, their transitions path_rf (0 rise,
 * 1 fall) and the path's arrival at each (path_at, ps); path_slack[i],
 * path_ep[i] (endpoint pin).  If the pins do not fit, STA_ERR_ARG with
 * n_paths / n_pins set to the sizes needed.  Synchronizes. */
typedef struct {
  uint32_t mode;        /* 0 setup (late), 1 hold (early) */
  uint32_t k;           /* paths in all */
  uint32_t nworst;      /* paths per endpoint */
  float slack_lt;       /* report slack < slack_lt only (INFINITY: all) */
} sta_path_query;
typedef struct {
  uint32_t cap_paths, cap_pins;  /* in */
  uint32_t n_paths, n_pins;      /* out */
  uint32_t* path_ptr;            /* [cap_paths + 1] */
  uint32_t* path_pin;            /* [cap_pins] */
  uint8_t* path_rf;              /* [cap_pins] */
  float* path_at;                /* [cap_pins] */
  float* path_slack;             /* [cap_paths] */
  uint32_t* path_ep;             /* [cap_paths] */
} sta_path_set;
STA_API sta_status sta_report_paths(sta_ctx ctx, uint32_t corner, const sta_path_query* q, sta_path_set* out,
                                    sta_mem mem);

/* Counters describing the loaded graph and the last update. */
typedef struct {
  uint32_t num_pins, num_nets, num_net_arcs, num_cell_arcs, num_checks, num_endpoints;
  uint32_t num_levels;       /* pin levels */
  uint32_t num_stages;       /* gate stages the kernels step through */
  uint32_t num_pull_pins;    /* pins evaluated over cell arcs (stage pins) */
  uint32_t num_sink_pins;    /* net sinks */
  uint32_t num_heavy_drivers;
  uint32_t kernels_per_update; /* kernel launches of one sta_update_timing */
  uint32_t lut_smem_bytes;   /* largest per-launch NLDM image staged in shared memory (0: global lookups) */
  uint64_t device_bytes;     /* device memory held by ctx */
} sta_info;
STA_API sta_status sta_get_info(sta_ctx ctx, sta_info* out);

/* Block until all work enqueued on the ctx stream is done; returns any
 * deferred kernel error (STA_ERR_CUDA, STA_ERR_RC). */
STA_API sta_status sta_synchronize(sta_ctx ctx);

/* ------------------------------------------------------------ profiling */

/* Per-phase device time of sta_update_timing, measured with CUDA events on the
 * ctx stream around each phase's kernels (used by bench.py's roofline).
 * Phases: 0 = RC/Elmore (a1), 1 = forward AT/slew (a2), 2 = backward RAT +
 * slack (a3-a5 per pin), 3 = WNS/TNS reduction (a5), 4 = whole update. */
#define STA_NUM_PHASES 5
typedef struct {
  double ms[STA_NUM_PHASES];        /* accumulated milliseconds */
  uint32_t launches[STA_NUM_PHASES];/* accumulated kernel launches */
  uint32_t updates;                 /* updates accumulated */
} sta_profile;

/* enable != 0: start (and zero) accumulation; 0: stop. */
STA_API sta_status sta_profile_enable(sta_ctx ctx, int enable);
/* Synchronizes, then copies the accumulated profile. */
STA_API sta_status sta_profile_read(sta_ctx ctx, sta_profile* out);

#ifdef __cplusplus
}
#endif
#endif /* STA_H */
