// sta_internal.h -- device data layout shared by the host engine (sta_api.cpp)
// and the sm_100a kernels (sta_kernels.cu).  See DESIGN.md §5 for the layout.
//
// Internal pin numbering (built once by sta_load_graph):
//   * "pull pins" -- pins without a net arc into them (cell outputs, sources):
//     internal ids [0, NP), sorted by (gate stage, user id).  A pull pin is
//     evaluated by pulling over its cell-arc fan-in.
//   * "sinks" -- net sinks (exactly one fan-in: the net arc): internal ids
//     [NP, P), grouped by driver in driver order, in net order.  A sink is a
//     pure function of its driver (AT + Elmore, PERI slew): its arrival and
//     slew are never stored, every consumer recomputes them from the driver's
//     record with the same instructions (pull-through).
//   Gate stage: 0 for pins without fan-in, else 1 + max over cell fan-in
//   (u -> v) of stage(driver(u)) (stage(u) if u is itself a pull pin).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sta {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kSeedClock = 0xFFFFFFFEu;   // stage-0 seed: ideal clock pin
constexpr uint32_t kSeedMark = 0xFFFFFFFDu;    // forward term slot: seed pin
constexpr uint32_t kHeavyMark = 0xFFFFFFFCu;   // forward term slot: pin with many terms
constexpr uint32_t kTile = 32;                 // backward: sinks per warp tile (lane = sink)
constexpr uint32_t kBNet = 1024;               // RC tier B: nets of 33..1024 nodes, one block tile
constexpr uint32_t kChunk = 256;               // stage id padding; readiness group of the persistent kernels
constexpr uint32_t kWarpUnit = 32;             // persistent kernels: items per warp unit
constexpr uint32_t kFwdUnitTerms = 8;          // forward warp unit: fan-in terms (4 lanes each)
// Persistent kernels: ONE block per SM holding all of the SM's warps, so the
// staged NLDM pools of every corner of a batch exist once per SM (8 corners of
// LIB-SYN = 190 KB).  Warps per SM are the register budget tuned on C3 (the
// forward's short per-lane chains want many warps, the backward's one-lane-per-
// sink chains want registers): 32 forward warps (<= 64 registers), 24 backward
// warps (<= 85 registers); more forward warps measured slower (r2 sweep).
#ifndef STA_FWD_THREADS
#define STA_FWD_THREADS 1024
#endif
constexpr int kFwdThreads = STA_FWD_THREADS;    // forward persistent kernel block size
#ifndef STA_FWD_MINB
#define STA_FWD_MINB 1
#endif
constexpr int kFwdMinBlocks = STA_FWD_MINB;
#ifndef STA_BWD_THREADS
#define STA_BWD_THREADS 768
#endif
constexpr int kBwdThreads = STA_BWD_THREADS;    // backward persistent kernel block size
#ifndef STA_BWD_MINB
#define STA_BWD_MINB 1
#endif
constexpr int kBwdMinBlocks = STA_BWD_MINB;
#ifndef STA_BWD_SPIN_FIRST
#define STA_BWD_SPIN_FIRST 0                    // wait on the first fan-out pin before loading the arrival
#endif
#ifndef STA_FWD_PF
#define STA_FWD_PF 1                            // forward: prefetch term slots 2 and RC results 1 unit ahead
#endif
#ifndef STA_FWD_RECPF
#define STA_FWD_RECPF 1                         // forward: next unit's record words loaded speculatively
#endif
#ifndef STA_MERGE_BOUND
#define STA_MERGE_BOUND 0                       // 1: merge rounds bounded by the longest run in the warp (measured slower)
#endif
#ifndef STA_BWD_PIPE
#define STA_BWD_PIPE 1                          // backward: next unit's fan-out records: 1 registers, 2 TMA (slower, r2)
#endif
constexpr uint32_t kMaxBatch = 8;               // corners traversed by one launch
// backward persistent kernel: per-warp TMA staging buffer of the next unit's
// fan-out records (1 KB) and its mbarrier, after the LUT image
constexpr size_t kBwdExtraSmem = STA_BWD_PIPE == 2 ? (size_t)(kBwdThreads / 32) * (1024 + 8) : 0;

// Device NLDM table pool (built by sta_set_library), shared-memory friendly:
//   * table t: a block of kTabStride = 65 floats at t * 65: word 0 = offset
//     (as int) of its axis template, words 1..64 = values v[8][8] row-major,
//     rows >= n1 / columns >= n2 replicating the last row / column (so a
//     1-wide axis interpolates by 0).  The odd stride spreads lanes that read
//     the same entry of different tables over different shared-memory banks.
//   * axis templates (deduplicated, 16-byte aligned), 48 floats: for index_1
//     then index_2: sx[8] search thresholds (sx[k] = x[k] for 1 <= k <= n-2,
//     +inf otherwise -> segment i = #{k : sx[k] <= s}), x[8] (padded with the
//     last value), rx[8] = 1 / (x[k+1] - x[k]) (0 past the end), fp32.
//     Tables of one library template share one record (warp broadcast).
constexpr int kTabStride = 65;
constexpr int kTmplStride = 48;

// arc info word: sense (3 bits) | first table id << 3
__host__ __device__ inline uint32_t pack_info(uint32_t sense, uint32_t tab) { return sense | (tab << 3); }

struct EpRec {          // one timing endpoint
  uint32_t po;          // index into the PO constraint arrays or kNone
  uint32_t chk_tab;     // first of (setup_r, setup_f, hold_r, hold_f) or kNone
};

// Topology shared by all corners (device pointers).
struct Topo {
  uint32_t P, NP, NS, S, N, n_ep, n_pi, n_po, n0;   // P: caller pins; NP: pull ids incl. padding
  // forward: fan-in terms of pull pins (heavy pins and tests; the kernels read fterm)
  const uint32_t* fi_src;    // record to read (driver of u, or u if u is a pull pin)
  const uint32_t* fi_hop;    // sink index of u (net hop to apply) or kNone
  const uint32_t* fi_info;
  const uint32_t* sink_ptr;  // [NP+1] sinks of each pull pin (sink index space)
  const uint32_t* sink_drv;  // [NS]
  const uint32_t* seed;      // [pins of stage 0]: PI index, kSeedClock or kNone
  // backward: cell fan-out arcs of sinks / pull pins (ranges in sinkrec / pullrec)
  const uint32_t* sfo_dst;   // pull pin
  const uint32_t* sfo_info;
  const uint32_t* pfo_dst;
  const uint32_t* pfo_info;
  const EpRec* ep;           // [n_ep]
  const uint32_t* nosink;    // pull pins without sinks, by stage
  const uint32_t* heavy_nchunk; // [n_heavy] tiles of each heavy driver
  const uint32_t* heavy_base;   // [n_heavy] first partial slot of each heavy driver
  // propagation work units (sta_kernels.cu), lists in dependency order
  // forward warp unit u = term slots [kFwdUnitTerms u, kFwdUnitTerms (u + 1)):
  //   {src, hop, info, pin}: a fan-in term of pull pin `pin` (record src,
  //     sink hop or kNone, sense | table << 3)
  //   {kNone, kNone, 0, kNone}: padding
  //   {kSeedMark, 0, 0, pin or kNone}: stage-0 pin (seed)
  //   {kHeavyMark, term0, nterms, pin} in every slot but slot 1 = {kHeavyMark,
  //     first delay slot, 0, 0}: one pin with more than kFwdUnitTerms terms
  //     (fi_* arrays), looped over by the warp
  // the delay slot of a term is its unit slot (heavy pins: past the units)
  const uint4* fterm;
  uint32_t n_fwu;
  // backward warp units, descending stage: {k0, k1, kNone, 0}: sinks [k0, k1)
  // (<= kTile, a light driver never split); {k0, k1, heavy slot, 2 + partial
  // slot}: one tile of a driver with more than kTile sinks; {x0, x1, 0, 1}:
  // sink-less pull pins [x0, x1) (<= kTile; internal ids of a stage put
  // drivers first, so a stage's sink-less pins are contiguous)
  const uint4* bwu;
  uint32_t n_bwu;
  uint32_t n_bwu_static;         // units [0, n_bwu_static) statically assigned; the rest (stage 0,
                                 // no dependencies among them) handed out by a ticket counter
  // backward fan-out records, two uint4 per sink (sinkfo) / pull pin (pullfo):
  //   a = {driver | has-pullfo-work << 31 (sinks; 0 for pull pins), nfo = cell fan-out terms, f0 =
  //        first term in sfo_* / pfo_*, endpoint index or kNone}
  //   b = non-endpoints: {dst, sense | delay slot << 3} of the first two fan-out terms (kNone
  //       dst if absent); endpoints: {check table or kNone, PO index or
  //       kNone, 0, 0} and the fan-out is read from sfo_* / pfo_*
  const uint4* sinkfo;
  const uint4* pullfo;
  const float4* po_seed;         // [n_po] {-out_min_r, -out_min_f, T - out_max_r, T - out_max_f}
  // constraints
  const float4* pi_at;       // [n_pi]
  const float4* pi_slew;
  const float2* po_out_max;  // [n_po]
  const float2* po_out_min;
  float period, clock_slew;
  // RC: nets in driver order j; each net's nodes in DFS preorder ("internal
  // nodes", subtree of position p = [p, end(p))), grouped by tier (A: 1..32
  // nodes, B: 33..kBNet, C: larger), each group in driver order.
  const uint32_t* net_drv;   // [N] internal pull id of the driver
  const float* net_lumped;   // [N] lumped load (nets without RC nodes)
  // per internal RC node: meta = pos | parent pos << 8 (0xFF: root) | end << 16
  // (tier A); tag = sink index, driver | 0x80000000 at the root, or kNone;
  // scap = pin cap + PO load at the node (R / Cw stay in the caller's order)
  const uint4* rc_node;      // [tier A + B nodes] {meta, tag, caller node (tier B) or caller
                             //  offset in the warp tile (tier A), scap bits} packed
  uint32_t n_wtiles;         // warp tiles of nets with 1..32 nodes (no net straddles a tile; the
                             // tile's caller nodes are one contiguous range)
  const uint4* wtiles;       // {first internal node, node count, first caller node, 0}
  // tier B: nets with 33..kBNet nodes, whole nets in block tiles of <= kBNet
  // contiguous nodes; their node_meta is pos | parent pos << 10 (0x7FF: root) | end << 21
  uint32_t n_btiles;
  const uint2* btiles;       // {first internal node, node count}
  uint32_t n_lumped;
  const uint32_t* lumped_j;  // nets without RC nodes
  uint32_t nC;               // nets with > kBNet nodes (tier C)
  // tier C (nets > kBNet nodes): segmented prefix sums over ONE global
  // preorder array of their nodes (each net contiguous, DFS preorder inside,
  // the net's root its segment head) and over its Euler event sequence
  // (enter / exit of every node, 2 per node; a net whose root sits at
  // position g0 owns events [2 g0, 2 g0 + 2 m), its first event entering the
  // root).  With Sx / Si the segmented exclusive / inclusive sums of the node
  // caps, Cdown(g) = Si[end(g) - 1] - Sx[g]; with w = R Cdown, event values
  // +w(a) at enter(a), -w(a) at exit(a) and H their segmented inclusive sum,
  // elm(g) = H[enter(g)] (the ancestors-or-self of g are exactly the nodes
  // entered and not yet exited there).
  uint32_t nCn;               // tier-C nodes
  const uint4* tc_node;       // [nCn] {caller node id, tag (as node_tag), end (global position one
                              //  past the subtree), rc_scap bits}
  const uint2* tc_ev;         // [2 nCn] {node position of each event | 0x80000000 for an exit,
                              //  the node's tag for an enter event, kNone for an exit}
  // outputs to user order
  const uint32_t* int_of_user; // [P]
  const uint32_t* drv_of_net;  // [N] user net -> internal driver
  // NEXT row f1: net-arc delay model (0 Elmore, 1 Arnoldi reduced order
  // arn_q <= 4; sta_arnoldi.cu / sta_arnoldi.cuh).  Arnoldi layout over the
  // internal RC nodes (each net contiguous in DFS preorder):
  uint32_t net_model, arn_q;
  uint32_t n_arn_nets;
  const uint4* arn_nets;      // {first internal node, nodes (0: lumped net), internal driver, 0}
  const uint4* arn_node;      // [n_rc] {caller node id, internal parent or kNone at the root,
                              //  subtree end (internal), sink index or kNone}
  const float* arn_scap;      // [n_rc] pin + PO cap at the node
  // NEXT row f4 (reduced): endpoint overrides of the tag this pass propagates
  // (nullptr: no exceptions), per endpoint {late mode, late value bits,
  // early mode, early value bits}; mode 0 shift, 1 replace, 2 no seed
  const uint4* ep_ovr;
  uint32_t n_arn_big;
  const uint32_t* arn_big;    // indices (into arn_nets) of the nets of more than 1024 RC nodes
  uint64_t n_rc_nodes;
  // row f4: -through exception segments (the oracle's O15; X8).
  // The pins of any -through segment are "through slots" 0 .. n_thr-1;
  // thr_pull [NP] / thr_sink [NS]: slot of a pull pin / sink or kNone
  // (nullptr: no -through, the kernels' non-THR instantiations run).  This
  // pass (tag thr_cur): thr_dst [n_thr] = the pass its tag advances to at the
  // slot's pin (its arrivals there are handed over, its required times taken
  // from that pass) or kNone (final there: it takes in the arrivals handed
  // to it and records its required times).  thr_sk [n_thr_sk]: {sink, slot}
  // of the sink slots (the handoff of sink arrivals, thr_capture_kernel).
  const uint32_t* thr_pull;
  const uint32_t* thr_sink;
  const uint32_t* thr_dst;
  const uint2* thr_sk;
  uint32_t n_thr, n_thr_sk, thr_cur;
};

// Per-corner device state.
struct CornerDev {
  uint4* rec;         // [4 NP]: tagged forward records of pull pins (sta_kernels.cu: ld_ll)
  uint4* rat_ll;      // [2 NP]: tagged required times of pull pins
  float4* at4;        // [NP]: untagged copy of the pull pins' arrival times, written by the
                      // forward next to the tagged record, read by the backward (which runs
                      // after the forward kernel: no readiness tags needed; 16 B instead of 64 B)
  uint32_t* epoch;    // [1] tag of the current update (advanced by reduce_kernel)
  float4* tdel;       // [delay slots] cell-arc delays of each fan-in term, (el, orf) order,
                      // written by the forward, read by the backward
  float4* rat;        // [P]: required times of sinks (ids >= NP; pull pins use rat_ll)
  float4* slack;      // [P]
  float* elm;         // [NS] Elmore delay of each sink's net arc
  float* load;        // [NP] NLDM load seen by each pull pin (0 if no net)
  float2* ep_ws;      // [n_ep] worst setup / hold slack per endpoint
  double* res;        // [4]
  double* red_part;   // [kRedBlocks * 4] reduction partials
  uint32_t* red_cnt;  // [2] last-block counter, backward tail ticket (reset by reduce_kernel)
  float4* heavy_part; // [heavy tiles] partial required time of each heavy-driver tile
  uint32_t* heavy_cnt;// [n_heavy] finished tiles (self-resetting)
  const float* lut;   // table records (kTabStride floats each)
  uint32_t lut_n4;    // float4s of this corner's pool
  uint32_t lut_off4;  // float4 offset of this corner's pool in a batch's shared-memory image
  const float* const* rc_vals;  // device {res, cap} pointer pair (user node order)
  double* scratch;    // tier-C scratch (tierC_scratch)
  uint32_t* err_flag; // nonzero: bad RC value seen
  float4* m_pin;      // exceptions (row f4): [4][NP + NS] internal order, at / slew / rat / slack merged over tags
  float2* m_ep_ws;    // [n_ep] worst setup / hold slack per endpoint merged over tags
  float4* arn_lam;    // [NP] Arnoldi time constants of the net each pull pin drives (x < 0: Elmore)
  float4* arn_res;    // [NS] residues of each sink
  double* arn_scr;    // [(arn_q + 4) n_rc] Lanczos scratch
  unsigned long long* trace;  // optional (STA_TRACE): per warp unit {start, ready, end} ns
  // row f4 -through handoff (Topo::thr_*), [tags][n_thr] each: arrivals / slews
  // handed to a pass at its final through pins (merged, early min / late
  // max), required times each pass computes at its final through pins
  float4* thr_hat;
  float4* thr_hsl;
  float4* thr_hrat;
};

// The corners one launch traverses.  Persistent kernels bind warp w to corner
// w % K and walk that corner's unit list with stride W / K, so the K corners'
// wavefronts advance together: one dependent-latency chain serves all K (a
// corner's stage-to-stage latency is paid once per batch, not once per
// corner), and the K warps reading the same unit's topology meet in L2.
struct Batch {
  CornerDev c[kMaxBatch];
  uint32_t K;
  uint32_t smem_f4;   // float4s of the staged LUT image (the K pools back to back); 0: global
};

#ifndef STA_RED_BLOCKS
#define STA_RED_BLOCKS (4 * 148)
#endif
constexpr int kRedBlocks = STA_RED_BLOCKS;    // reduce_kernel blocks per corner (fixed: bitwise reproducible)

// ---- launchers (sta_kernels.cu); all enqueue on `s` with programmatic
// dependent launch, return cudaGetLastError().  Every launch covers the
// corners of batch b (grid.y = corner for the data-parallel kernels).
// RC of nets with <= kBNet nodes and lumped nets; tier C (nets > kBNet nodes) is
// independent of it and is enqueued on a second stream (2 launches)
cudaError_t launch_rc(const Topo& t, const Batch& b, uint32_t wgrid, cudaStream_t s);
cudaError_t launch_rc_tierC(const Topo& t, const Batch& b, cudaStream_t s);
// tier-C scratch: Si [nCn] (double), block aggregates of the node and the
// event scans [nbn + nbe] (double), their flags [nbn + nbe] (u32 {has head,
// epoch}) and the two tile tickets (u32, zero-initialised, monotonic)
#ifndef STA_TC_TILE
#define STA_TC_TILE 2048
#endif
constexpr uint32_t kTcTile = STA_TC_TILE;       // elements per tier-C block (256 threads x 8)
__host__ __device__ inline uint32_t tierC_blocks(uint64_t n) { return (uint32_t)((n + kTcTile - 1) / kTcTile); }
__host__ __device__ inline size_t tierC_scratch_scan(uint32_t nCn) {
  const size_t nb = (size_t)tierC_blocks(nCn) + tierC_blocks(2ull * nCn);
  return (size_t)nCn + nb + (nb + 2 + 1) / 2 + 1;
}
// ... followed by w [nCn] (double): R(g) Cdown(g) of every tier-C node (0 at a root)
__host__ __device__ inline size_t tierC_scratch(uint32_t nCn) { return tierC_scratch_scan(nCn) + nCn; }
uint32_t rc_warp_grid();                        // co-resident grid of the tier-A kernel (per corner)
// units [u0, u1) of one gate stage (one launch per stage, grid.y = corner)
cudaError_t launch_fwd_stage(const Topo& t, const Batch& b, uint32_t u0, uint32_t u1, cudaStream_t s);
cudaError_t launch_bwd_stage(const Topo& t, const Batch& b, uint32_t u0, uint32_t u1, cudaStream_t s);
cudaError_t set_lut_smem_limit(size_t bytes);
// persistent (cooperative, sync-free dataflow) forward / backward passes;
// grid = co-resident blocks (one per SM).  persistent_grid returns 0 if unsupported.
uint32_t persistent_grid(uint32_t smem_f4, int which);
cudaError_t launch_fwd_persistent(const Topo& t, const Batch& b, uint32_t grid, cudaStream_t s);
cudaError_t launch_bwd_persistent(const Topo& t, const Batch& b, uint32_t grid, cudaStream_t s);
constexpr size_t kLutSmemMax = 200 * 1024;   // larger batch images stay in global memory
                                             // (+ kBwdExtraSmem stays under the 227 KB per block)
cudaError_t launch_reduce(const Topo& t, const Batch& b, cudaStream_t s);
cudaError_t launch_gather_pins(const Topo& t, const CornerDev& c, int what, float4* dst, cudaStream_t s);
cudaError_t launch_gather_rc(const Topo& t, const CornerDev& c, float* net_load, float* pin_elm, cudaStream_t s);
cudaError_t launch_init_corner(const Topo& t, const CornerDev& c, uint32_t n_heavy, cudaStream_t s);
cudaError_t launch_set_ptrs(const float* const* dst, const float* a, const float* b, cudaStream_t s);

// ---- row f3: top-k path report (sta_kernels.cu, path_*_kernel)
struct PathEnt {        // one partial path into a (pull pin, transition)
  float a;              // its arrival there
  uint32_t term;        // the fan-in term it came through (kNone: startpoint)
  uint32_t rr;          // input transition << 31 | rank in the source's list
};
struct PathArgs {
  uint32_t mode, m;                 // 0 setup (late), 1 hold (early); list length
  PathEnt* lists;                   // [NP][2][m]
  uint8_t* cnt;                     // [NP][2]
  const uint32_t* fi_p;             // [NP + 1] fan-in terms of each pull pin
  const uint32_t* fi_slot;          // [terms] delay slot (tdel) of each term
  const uint32_t* uoi;              // [NP + NS] internal id -> user pin id
  const uint32_t* ep_int;           // [n_ep] internal id of each endpoint
  unsigned long long* cand_key;     // [n_ep * m] (orderable slack << 32 | user id)
  uint32_t* cand_ref;               // [n_ep * m] endpoint index
  uint32_t* cand_sub;               // [n_ep * m] transition << 31 | rank
  float* cand_slack;                // [n_ep * m]
  const uint32_t* sorted_ref;       // report order
  const uint32_t* sorted_sub;
  const float* sorted_slack;
  uint32_t* path_ptr;               // outputs (device)
  uint32_t* path_pin;
  uint8_t* path_rf;
  float* path_at;
  float* path_slack;
  uint32_t* path_ep;
};
// Enqueue the report on s and return the selected path and pin counts
// (synchronizes s).  pin capacity of pa.path_* = cap_pins; if the pins do
// not fit, only the counts are returned (*fits = false).
cudaError_t run_path_report(const Topo& t, const CornerDev& c, PathArgs pa, const uint32_t* stage_ptr, uint32_t S,
                            uint32_t k, float slack_lt, uint32_t cap_pins, uint32_t* n_paths, uint32_t* n_pins,
                            bool* fits, cudaStream_t s);

// ---- row a0 on the device (sta_levelize.cu): cell-arc fan-in / fan-out CSR
// (segments in arc id order), Kahn-frontier levels over net + cell arcs and
// perm = pins stably sorted by (level, id).  Device pointers; synchronizes s.
cudaError_t levelize_device(uint32_t P, uint32_t N, uint32_t A, const uint32_t* net_ptr, const uint32_t* net_pins,
                            const uint32_t* arc_from, const uint32_t* arc_to, uint32_t* level, uint32_t* perm,
                            uint32_t* fi_ptr, uint32_t* fi_ids, uint32_t* fo_ptr, uint32_t* fo_ids,
                            uint32_t* num_levels, uint32_t* cycle_pin, cudaStream_t s);

// ---- NEXT row f4: merge one tag's results into the merged arrays
cudaError_t launch_merge_tag(const Topo& t, const CornerDev& c, int first, cudaStream_t s);
// -through handoff: reset every pass's handed arrivals (start of an update),
// hand this pass's sink arrivals at its advancing through sinks to their
// passes (after its forward), advance the record epoch (after a forward-only
// pass: the next forward must not see this pass's records as current)
cudaError_t launch_thr_reset(const Topo& t, const Batch& b, uint32_t n_tags, cudaStream_t s);
cudaError_t launch_thr_capture(const Topo& t, const Batch& b, cudaStream_t s);
cudaError_t launch_bump_epoch(const Batch& b, cudaStream_t s);

// ---- NEXT row f1: Arnoldi reduced-order models of every net (sta_arnoldi.cu)
cudaError_t launch_arn_reduce(const Topo& t, const Batch& b, cudaStream_t s);

// ---- NEXT row f2: built-in Steiner RC from pin positions (sta_steiner.cu)
struct SteinerArgs {
  const uint32_t* net_ptr;        // [N + 1] the graph's net CSR offsets
  const uint32_t* spins;          // [net_ptr[N]] per net: driver, then sinks by pin id
  const float* x;                 // [P] pin positions
  const float* y;
  float rx, ry, cx, cy;           // unit R (kOhm) / C (fF) per distance unit along x / y
  uint32_t* ord;                  // [net_ptr[N]] Prim order (position in spins of the k-th tree pin)
  uint32_t* ppos;                 // [net_ptr[N]] Prim position of its tree parent (kNone at the root)
  uint32_t* nodeix;               // [net_ptr[N]] local node of the k-th tree pin
  uint32_t* cnt;                  // [N + 1] nodes per net (cnt[N] = 0)
  float4* scratch;                // [net_ptr[N]] per-pin Prim state of nets too large for shared memory
  uint32_t* rc_ptr;               // outputs (sta_set_rc_tree / sta_set_rc_values layout)
  int32_t* parent;
  uint32_t* node_pin;
  float* res;
  float* cap;
};
// Enqueue the construction on s.  warp_nets: nets of 2..32 pins; smem_nets:
// 33..steiner_smem_pins() pins (max_smem_pins = their largest); big_nets:
// larger (max_big_pins = their largest: one 8-CTA cluster per net up to
// 102,400 pins, one block with a global scratch beyond).  scan_tmp:
// steiner_scan_bytes(N) bytes.
cudaError_t run_steiner(const SteinerArgs& a, uint32_t N, const uint32_t* warp_nets, uint32_t n_warp,
                        const uint32_t* smem_nets, uint32_t n_smem, const uint32_t* big_nets, uint32_t n_big,
                        uint32_t max_smem_pins, uint32_t max_big_pins, void* scan_tmp, size_t scan_bytes,
                        cudaStream_t s);
size_t steiner_scan_bytes(uint32_t N);
uint32_t steiner_smem_pins();

}  // namespace sta
