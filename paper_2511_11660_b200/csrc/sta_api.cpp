// sta_api.cpp -- the C ABI of include/sta.h: validation, the host-side
// plan of the timing graph (levels, gate stages, internal numbering, CSR
// arrays, RC schedules), device memory and the update launcher.
//
// Every arithmetic step of the timing update runs in sta_kernels.cu; this file
// only arranges data (integer bookkeeping) and enqueues kernels.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <limits>
#include <new>
#include <string>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sta.h"
#include "sta_internal.h"

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: API ranges for nsys / ncu timelines

using sta::kNone;
using u32 = uint32_t;
using u64 = uint64_t;

namespace {

// NVTX range of one API call (visible in an nsys / ncu --nvtx timeline)
struct Nvtx {
  explicit Nvtx(const char* n) { nvtxRangePushA(n); }
  ~Nvtx() { nvtxRangePop(); }
};

// STA_TIMING=1: host phase times of sta_load_graph / sta_set_rc_tree on stderr
struct PhaseTimer {
  bool on = std::getenv("STA_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[sta timing] %-28s %9.1f ms\n", what,
                 std::chrono::duration<double, std::milli>(t1 - t0).count());
    t0 = t1;
  }
};

// Host parallel-for over [0, n) in T contiguous chunks f(lo, hi, t) (the
// planner's loops are memory-latency bound and scale with host threads).  f
// must not throw.
unsigned host_threads() {
  static const unsigned T = [] {
    if (const char* e = std::getenv("STA_HOST_THREADS")) return (unsigned)std::max(1, std::atoi(e));
    return std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 32u);
  }();
  return T;
}
template <class F>
void par_chunks(uint64_t n, F&& f) {
  const unsigned T = n < 65536 ? 1u : host_threads();
  if (T == 1) {
    f((uint64_t)0, n, 0u);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (unsigned t = 0; t < T; ++t) th.emplace_back([&f, n, t, T] { f(n * t / T, n * (t + 1) / T, t); });
  for (auto& x : th) x.join();
}
// Host parallel loop over a sequence of dependent phases: T threads run
// f(phase, lo, hi) on their chunk of [0, n(phase)) for every phase in order,
// with a barrier between phases (one thread team for all phases instead of
// one spawn per phase).  f must not throw.
template <class N, class F>
void par_phases(uint32_t phases, N&& n_of, F&& f) {
  const unsigned T = host_threads();
  if (T == 1) {
    for (uint32_t ph = 0; ph < phases; ++ph) f(ph, (uint64_t)0, (uint64_t)n_of(ph));
    return;
  }
  std::mutex mu;
  std::condition_variable cv;
  unsigned arrived = 0, gen = 0;
  auto barrier = [&] {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned g = gen;
    if (++arrived == T) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  };
  std::vector<std::thread> th;
  th.reserve(T);
  for (unsigned t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      for (uint32_t ph = 0; ph < phases; ++ph) {
        const uint64_t n = n_of(ph);
        f(ph, n * t / T, n * (t + 1) / T);
        barrier();
      }
    });
  for (auto& x : th) x.join();
}

// in-place exclusive prefix sum; returns the total
template <class T>
T excl_prefix(std::vector<T>& v) {
  T run = 0;
  for (T& x : v) {
    const T y = x;
    x = run;
    run += y;
  }
  return run;
}

struct StaError {
  sta_status st;
  std::string msg;
};

[[noreturn]] void fail(sta_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  throw StaError{st, buf};
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) fail(STA_ERR_OOM, "%s: %s", what, cudaGetErrorString(e));
    fail(STA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  }
}

// device allocations grouped by lifetime scope
struct Arena {
  std::vector<void*> ptrs;
  uint64_t bytes = 0;
  template <class T>
  T* alloc(size_t n) {
    if (n == 0) n = 1;
    void* p = nullptr;
    ck(cudaMalloc(&p, n * sizeof(T)), "cudaMalloc");
    ptrs.push_back(p);
    bytes += n * sizeof(T);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v, cudaStream_t s) {
    T* p = alloc<T>(v.size());
    if (!v.empty()) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s), "H2D");
    return p;
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
    bytes = 0;
  }
};

// copy caller input (HOST or DEVICE) into a host vector
template <class T>
std::vector<T> fetch(const T* p, size_t n, sta_mem mem, const char* name, cudaStream_t s) {
  std::vector<T> v(n);
  if (n == 0) return v;
  if (!p) fail(STA_ERR_ARG, "%s: NULL pointer for %zu elements", name, n);
  if (mem == STA_MEM_HOST) {
    std::memcpy(v.data(), p, n * sizeof(T));
  } else if (mem == STA_MEM_DEVICE) {
    // stream ordered: after every kernel the caller queued on the ctx stream
    ck(cudaMemcpyAsync(v.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s), name);
    ck(cudaStreamSynchronize(s), name);
  } else {
    fail(STA_ERR_ARG, "%s: bad sta_mem %d", name, (int)mem);
  }
  return v;
}

// the top-k path report's device scratch (row f3), kept across reports
struct PathScratch {
  Arena a;
  u32 m = 0, cp = 0, cq = 0;
  sta::PathEnt* lists = nullptr;
  uint8_t* cnt = nullptr;
  unsigned long long* key = nullptr;
  u32 *ref = nullptr, *sub = nullptr, *pptr = nullptr, *ppin = nullptr, *pep = nullptr;
  float *sl = nullptr, *pat = nullptr, *psl = nullptr;
  uint8_t* prf = nullptr;
};

struct CornerState {
  bool lib = false, rcv = false;
  Arena lib_arena, rc_arena, state_arena, ptr_arena;
  const float* rc_res = nullptr;   // active R / Cw arrays (owned or borrowed)
  const float* rc_cap = nullptr;
  // STA_MEM_HOST values: two owned {R, Cw} buffers, written alternately on the
  // copy stream; free_ev[b] = the point of the ctx stream after which buffer b
  // is no longer read (recorded when the other buffer becomes current)
  // row f4 -through: forward results of every tag's pass (index = pass; pass
  // 0 = dev.rec / at4 / tdel), so the reverse sweep needs no second forward
  std::vector<uint4*> p_rec;
  std::vector<float4*> p_at4, p_tdel;
  float* hbuf[2][2] = {{nullptr, nullptr}, {nullptr, nullptr}};
  int hcur = -1;                   // the current owned buffer (-1: borrowed or none)
  cudaEvent_t free_ev[2] = {nullptr, nullptr};
  bool free_rec[2] = {false, false};
  size_t lut_bytes = 0;                  // device table pool size
  sta::CornerDev dev{};
};

}  // namespace

struct sta_ctx_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t side = nullptr;    // tier-C RC branch (forked from / joined to `stream`)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr;
  cudaStream_t copy = nullptr;    // host RC values: H2D beside a running update (double-buffered)
  cudaEvent_t copy_ev = nullptr;
  u32 K = 1;
  std::string err;
  bool poisoned = false;
  bool has_graph = false, has_tree = false, has_cons = false, prepared = false;

  // ---- host copy of the netlist (validated)
  u32 P = 0, N = 0, A = 0, C = 0, T = 0;
  std::vector<float> pin_cap;
  std::vector<uint8_t> pin_role;
  std::vector<u32> net_ptr, net_pins, arc_from, arc_to, arc_tab, chk_d, chk_ck, chk_tab;
  std::vector<uint8_t> arc_sense;
  std::vector<u32> pin_net;       // net of each pin or kNone
  std::vector<uint8_t> is_sink;   // pin is a net sink (not driver)
  std::vector<u32> chk_of_pin;    // check index of a data pin or kNone

  // ---- plan
  std::vector<u32> level, perm;
  u32 num_levels = 0;
  std::vector<u32> stage, int_of_user, user_of_int;
  u32 NP = 0, NS = 0, S = 0, n0 = 0, Pi = 0;   // NP includes stage padding; Pi = NP + NS
  std::vector<u32> pull_stage_ptr, sink_stage_ptr, tile_stage_ptr, nosink_stage_ptr, sink_ptr;
  std::vector<u32> drv_of_net;    // user net -> internal driver id
  u32 n_heavy = 0, n_heavy_parts = 0, n_fwu = 0, n_bwu = 0, n_dslots = 0;
  std::vector<u32> sfo_p, pfo_p, sink_drv;      // host copies for prepare()
  std::vector<u32> sfo_dst, sfo_info, pfo_dst, pfo_info;
  std::vector<u32> fwu_stage_ptr;                // [S + 1] forward units of each stage
  std::vector<u32> fi_p_h, fi_slot_h, ep_int_h;  // path report: term ranges, delay slots, endpoint ids
  Arena path_arena;                              // path report: their device copies + user_of_int
  PathScratch path_scratch;                      // path report: lists, candidates, host-destination outputs
  // row f4 (reduced): -from / -to exceptions; per startpoint tag a seed array
  // and endpoint overrides (prepare)
  std::vector<float> clk_period;                 // multiple ideal clocks (row f4; empty: one clock)
  std::vector<u32> pin_clk;
  std::vector<uint8_t> exc_kind;
  std::vector<float> exc_value;
  std::vector<u32> exc_from_ptr, exc_from, exc_to_ptr, exc_to;
  std::vector<u32> exc_thr_ptr, exc_seg_ptr, exc_seg;   // -through segments (empty: none)
  Arena exc_arena;
  std::vector<const u32*> exc_seed_d;
  std::vector<const uint4*> exc_ovr_d;
  std::vector<const u32*> exc_thr_dst_d;         // per pass: thr_dst (with -through)
  u32 n_thr = 0;                                 // through slots (pins of -through segments)
  // row f4: case analysis (sta_set_case_analysis): logic functions, when
  // guards, constants; applied in prepare() by patched copies of the term
  // arrays (disabled forward terms read the always-undefined pull pin U,
  // disabled backward terms carry bit 31, killed sinks bit 31 of the count)
  std::vector<u32> fn_pin, fn_in_ptr, fn_in, case_pin;
  std::vector<uint64_t> fn_tt, arc_when;
  std::vector<uint8_t> case_val;
  bool case_on = false;
  u32 undef_pin = kNone;                         // U: internal id of a stage-0 padding pull pin
  std::vector<uint4> fterm_h;                    // host copies of the plan's term arrays
  std::vector<u32> fi_src_h, fi_hop_h, arc_term_h;
  const uint4* fterm_d0 = nullptr;               // the plan's own device arrays
  const u32 *fi_src_d0 = nullptr, *fi_hop_d0 = nullptr, *sfo_info_d0 = nullptr, *pfo_info_d0 = nullptr;
  std::vector<uint8_t> case_sink_kill;           // [NS] (prepare)
  Arena case_arena;
  int net_model = 0;                             // row f1: 0 Elmore, 1 Arnoldi (order arn_q)
  u32 arn_q = 4;
  Arena arn_arena;                               // Arnoldi layout (prepare)
  Arena steiner_arena;                           // Steiner RC (row f2): static plan + scratch, lazily
  bool steiner_ready = false;
  const u32 *st_net_ptr = nullptr, *st_spins = nullptr, *st_warp = nullptr, *st_smem = nullptr, *st_big = nullptr;
  u32 st_n_warp = 0, st_n_smem = 0, st_n_big = 0, st_max_smem = 0, st_max_big = 0;
  sta::SteinerArgs st_args{};
  void* st_scan = nullptr;
  size_t st_scan_bytes = 0;
  const u32 *fi_p_d = nullptr, *fi_slot_d = nullptr, *ep_int_d = nullptr, *uoi_d = nullptr;
  std::vector<u32> bwu_stage_lo, bwu_stage_hi;   // [S] backward units of each stage (descending list)

  // ---- RC tree (host)
  std::vector<u32> rc_ptr, rc_node_pin;
  std::vector<int32_t> rc_parent;
  u32 n_rc = 0;
  u32 big_total = 0;              // tier-C nodes
  std::vector<u32> node_user;     // internal RC node -> caller node id
  std::vector<u32> node_meta_h, node_tag_h;   // host copies (packed node records, prepare())
  std::vector<u32> node_z_h;      // rc_node .z: caller offset in the warp tile (tier A) / caller id (B)
  std::vector<u32> tc_end_h;      // tier-C node: global position one past its subtree
  u32 n_rc_ab = 0;                // internal RC nodes of tiers A and B (they come first)
  std::vector<u32> rc_net_j;      // net j (driver order) -> internal driver id

  // ---- constraints (host)
  float period = 0, clock_slew = 0;
  std::vector<u32> pi_pin, po_pin;
  std::vector<float> pi_at, pi_slew, po_out_max, po_out_min, po_load;
  u32 n_ep = 0;

  // ---- device
  Arena graph_arena, tree_arena, cons_arena, tmp_arena;
  sta::Topo topo{};
  std::vector<CornerState> corners;

  // ---- profiling
  bool prof = false;
  sta_profile profile{};
  cudaEvent_t ev[STA_NUM_PHASES * 2] = {};
  u32 launches_per_update = 0;
  u32 smem_f4 = 0;                // largest batch LUT image staged in shared memory (float4s; 0: global)
  u32 wgrid = 0;                  // co-resident grid of the tier-A RC kernel
  // the update as one CUDA graph (captured lazily, invalidated by any input
  // change except sta_set_rc_values, which only rewrites a device-side
  // pointer pair)
  cudaGraphExec_t gexec = nullptr;
  bool use_graph = true;
  // forward / backward as persistent cooperative dataflow kernels (default)
  // or one launch per gate stage (STA_STAGE_KERNELS=1, or no cooperative launch)
  bool use_persistent = true;
  std::string trace_path;         // STA_TRACE (debug)
  std::vector<u32> fwu_stage_h;   // stage of each forward warp unit (trace labels)
  std::vector<u32> bwu_stage_h;   // stage of each backward warp unit (trace labels)
  std::vector<u32> bwu_kind_h;    // 0 light tile, 1 heavy tile, 2 sink-less pins (trace labels)
  u32 pgrid = 0, pgrid_b = 0;     // co-resident grids (forward, backward)
};

namespace {

void invalidate_graph(sta_ctx c) {
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  c->gexec = nullptr;
}

void prof_mark(sta_ctx c, int idx) {
  if (c->prof) ck(cudaEventRecord(c->ev[idx], c->stream), "cudaEventRecord");
}

// ------------------------------------------------------------ validation
void validate_graph(sta_ctx c) {
  const u32 P = c->P;
  for (u32 p = 0; p < P; ++p) {
    if (c->pin_role[p] > STA_PIN_FF_D) fail(STA_ERR_ARG, "pin %u: bad role %u", p, c->pin_role[p]);
    if (!std::isfinite(c->pin_cap[p]) || c->pin_cap[p] < 0) fail(STA_ERR_ARG, "pin %u: bad pin_cap", p);
  }
  if (c->N) {
    if (c->net_ptr[0] != 0) fail(STA_ERR_CSR, "net_ptr[0] = %u, expected 0", c->net_ptr[0]);
    for (u32 n = 0; n < c->N; ++n)
      if (c->net_ptr[n + 1] <= c->net_ptr[n])
        fail(STA_ERR_CSR, "net %u: offsets not monotone or empty net (no driver)", n);
  }
  c->pin_net.assign(P, kNone);
  c->is_sink.assign(P, 0);
  for (u32 n = 0; n < c->N; ++n) {
    for (u32 k = c->net_ptr[n]; k < c->net_ptr[n + 1]; ++k) {
      const u32 p = c->net_pins[k];
      if (p >= P) fail(STA_ERR_ID, "net %u: pin id %u out of range", n, p);
      if (c->pin_net[p] != kNone) fail(STA_ERR_MULTIDRIVER, "pin %u: in nets %u and %u", p, c->pin_net[p], n);
      c->pin_net[p] = n;
      c->is_sink[p] = k != c->net_ptr[n];
    }
  }
  for (u32 a = 0; a < c->A; ++a) {
    const u32 f = c->arc_from[a], t = c->arc_to[a];
    if (f >= P || t >= P) fail(STA_ERR_ID, "arc %u: pin id out of range", a);
    if (c->arc_sense[a] > STA_FALL_EDGE) fail(STA_ERR_ARG, "arc %u: bad sense %u", a, c->arc_sense[a]);
    if ((uint64_t)c->arc_tab[a] + 3 >= c->T) fail(STA_ERR_ID, "arc %u: table id %u out of range", a, c->arc_tab[a]);
    if (c->is_sink[t]) fail(STA_ERR_MULTIDRIVER, "pin %u: driven by net %u and by cell arc %u", t, c->pin_net[t], a);
    if (f == t) fail(STA_ERR_CYCLE, "cycle through pin %u (self arc %u)", f, a);
  }
  c->chk_of_pin.assign(P, kNone);
  for (u32 k = 0; k < c->C; ++k) {
    const u32 d = c->chk_d[k], ckp = c->chk_ck[k];
    if (d >= P || ckp >= P) fail(STA_ERR_ID, "check %u: pin id out of range", k);
    if (c->pin_role[d] != STA_PIN_FF_D) fail(STA_ERR_ARG, "check %u: data pin %u does not have role FF_D", k, d);
    if (c->pin_role[ckp] != STA_PIN_FF_CK) fail(STA_ERR_ARG, "check %u: clock pin %u does not have role FF_CK", k, ckp);
    if ((uint64_t)c->chk_tab[k] + 3 >= c->T) fail(STA_ERR_ID, "check %u: table id %u out of range", k, c->chk_tab[k]);
    if (c->chk_of_pin[d] != kNone) fail(STA_ERR_ARG, "pin %u: two checks (%u, %u)", d, c->chk_of_pin[d], k);
    c->chk_of_pin[d] = k;
  }
  for (u32 p = 0; p < P; ++p)
    if ((c->pin_role[p] == STA_PIN_PI || c->pin_role[p] == STA_PIN_FF_CK) && c->is_sink[p])
      fail(STA_ERR_ARG, "pin %u: role %s must not have fan-in", p, c->pin_role[p] == STA_PIN_PI ? "PI" : "FF_CK");
}

// CSR of arcs grouped by key (stable in arc id order)
void group_arcs(const std::vector<u32>& key, u32 P, std::vector<u32>& ptr, std::vector<u32>& ids) {
  ptr.assign(P + 1, 0);
  for (u32 k : key) ptr[k + 1]++;
  for (u32 p = 0; p < P; ++p) ptr[p + 1] += ptr[p];
  ids.resize(key.size());
  std::vector<u32> fill(ptr.begin(), ptr.end() - 1);
  for (u32 a = 0; a < key.size(); ++a) ids[fill[key[a]]++] = a;
}

// ------------------------------------------------------------------ plan
void build_plan(sta_ctx c) {
  const u32 P = c->P;
  PhaseTimer tm;
  // row a0 on the device (sta_levelize.cu): cell-arc CSR by target / source,
  // Kahn-frontier levels, perm = stable sort by (level, id)
  std::vector<u32> fi_ptr(P + 1), fi_ids(c->A), fo_ptr(P + 1), fo_ids(c->A);
  c->level.assign(P, 0);
  c->perm.assign(P, 0);
  {
    Arena a;
    cudaStream_t s = c->stream;
    try {
      const u32* d_np = a.upload(c->net_ptr, s);
      const u32* d_pins = a.upload(c->net_pins, s);
      const u32* d_from = a.upload(c->arc_from, s);
      const u32* d_to = a.upload(c->arc_to, s);
      u32* d_level = a.alloc<u32>(P);
      u32* d_perm = a.alloc<u32>(P);
      u32* d_fip = a.alloc<u32>(P + 1);
      u32* d_fii = a.alloc<u32>(c->A);
      u32* d_fop = a.alloc<u32>(P + 1);
      u32* d_foi = a.alloc<u32>(c->A);
      u32 cyc = kNone;
      ck(sta::levelize_device(P, c->N, c->A, d_np, d_pins, d_from, d_to, d_level, d_perm, d_fip, d_fii, d_fop, d_foi,
                              &c->num_levels, &cyc, s), "levelize kernels");
      if (cyc != kNone) fail(STA_ERR_CYCLE, "combinational cycle through pin %u", cyc);
      ck(cudaMemcpyAsync(c->level.data(), d_level, 4ull * P, cudaMemcpyDeviceToHost, s), "D2H level");
      ck(cudaMemcpyAsync(c->perm.data(), d_perm, 4ull * P, cudaMemcpyDeviceToHost, s), "D2H perm");
      ck(cudaMemcpyAsync(fi_ptr.data(), d_fip, 4ull * (P + 1), cudaMemcpyDeviceToHost, s), "D2H csr");
      ck(cudaMemcpyAsync(fo_ptr.data(), d_fop, 4ull * (P + 1), cudaMemcpyDeviceToHost, s), "D2H csr");
      if (c->A) {
        ck(cudaMemcpyAsync(fi_ids.data(), d_fii, 4ull * c->A, cudaMemcpyDeviceToHost, s), "D2H csr");
        ck(cudaMemcpyAsync(fo_ids.data(), d_foi, 4ull * c->A, cudaMemcpyDeviceToHost, s), "D2H csr");
      }
      ck(cudaStreamSynchronize(s), "levelize");
    } catch (...) {
      cudaStreamSynchronize(s);
      a.release();
      throw;
    }
    cudaStreamSynchronize(s);
    a.release();
  }
  tm.mark("plan: device levelize + CSR");
  for (u32 p = 0; p < P; ++p)
    if (c->pin_role[p] == STA_PIN_PI || c->pin_role[p] == STA_PIN_FF_CK)
      if (fi_ptr[p + 1] != fi_ptr[p])
        fail(STA_ERR_ARG, "pin %u: role %s must not have fan-in", p, c->pin_role[p] == STA_PIN_PI ? "PI" : "FF_CK");
  auto driver_of = [&](u32 p) { return c->net_pins[c->net_ptr[c->pin_net[p]]]; };

  // gate stages in pin-level order (the pins of one level are independent)
  c->stage.assign(P, 0);
  {
    std::vector<u32> lptr(c->num_levels + 1, 0);
    for (u32 p = 0; p < P; ++p) lptr[c->level[p] + 1]++;
    for (u32 l = 0; l < c->num_levels; ++l) lptr[l + 1] += lptr[l];
    par_phases(c->num_levels, [&](uint32_t l) { return (uint64_t)(lptr[l + 1] - lptr[l]); },
               [&](uint32_t l, uint64_t lo, uint64_t hi) {
      for (uint64_t j = lptr[l] + lo; j < lptr[l] + hi; ++j) {
        const u32 p = c->perm[j];
        if (c->is_sink[p]) {
          c->stage[p] = c->stage[driver_of(p)];
        } else if (fi_ptr[p + 1] != fi_ptr[p]) {
          u32 st = 0;
          for (u32 x = fi_ptr[p]; x < fi_ptr[p + 1]; ++x) st = std::max(st, c->stage[c->arc_from[fi_ids[x]]] + 1);
          c->stage[p] = st;
        }
      }
    });
  }

  // internal numbering: pull pins by (stage, id); sinks grouped by driver
  u32 NP = 0, S = 0;
  u32 NS = 0;
  for (u32 p = 0; p < P; ++p) {
    if (!c->is_sink[p]) S = std::max(S, c->stage[p] + 1);
    else ++NS;
  }
  c->S = S;
  // each stage's pull pins start on a kChunk boundary (padding ids are inert
  // dummies), so the chunk of a pin is id / kChunk for the persistent kernels
  std::vector<u32> stage_cnt(S, 0);
  for (u32 p = 0; p < P; ++p)
    if (!c->is_sink[p]) stage_cnt[c->stage[p]]++;
  c->pull_stage_ptr.assign(S + 1, 0);
  for (u32 s = 0; s < S; ++s)
    // (stage 0 keeps at least one padding id: the always-undefined source U
    // that case analysis points its disabled forward terms at)
    c->pull_stage_ptr[s + 1] = c->pull_stage_ptr[s] + (stage_cnt[s] + (s == 0) + sta::kChunk - 1) / sta::kChunk * sta::kChunk;
  NP = c->pull_stage_ptr[S];
  c->NP = NP;
  c->NS = NS;
  c->Pi = NP + NS;
  c->n0 = S ? c->pull_stage_ptr[1] : 0;
  c->undef_pin = S ? c->pull_stage_ptr[1] - 1 : kNone;
  c->int_of_user.assign(P, kNone);
  c->user_of_int.assign(c->Pi, kNone);
  {
    // within a stage: drivers of nets with an endpoint sink (PO / check data
    // pin), other drivers of nets with sinks, then sink-less pins (each
    // class by user id): the backward's sink-less units are ranges, and its
    // endpoint-seed lookups (divergent work) concentrate in few warps
    std::vector<u32> fill(c->pull_stage_ptr.begin(), c->pull_stage_ptr.end());
    auto pin_class = [&](u32 p) {
      const u32 n = c->pin_net[p];
      if (n == kNone || c->net_ptr[n + 1] - c->net_ptr[n] <= 1) return 2;
      for (u32 x = c->net_ptr[n] + 1; x < c->net_ptr[n + 1]; ++x) {
        const u32 q = c->net_pins[x];
        if (c->pin_role[q] == STA_PIN_PO || c->pin_role[q] == STA_PIN_FF_D || c->chk_of_pin[q] != kNone) return 0;
      }
      return 1;
    };
    std::vector<uint8_t> cls(P, 0);
    par_chunks(P, [&](uint64_t lo, uint64_t hi, unsigned) {
      for (uint64_t p = lo; p < hi; ++p)
        if (!c->is_sink[p]) cls[p] = (uint8_t)pin_class((u32)p);
    });
    // position of pull pin p: its stage's base, then the pins of lower
    // classes of the stage, then those of its class with a smaller id --
    // counted per (class, stage, id chunk) so the chunks fill in parallel
    const unsigned T = P < 65536 ? 1u : host_threads();
    std::vector<u32> cnt((size_t)T * 3 * S, 0);   // [class][stage][chunk]
    auto at = [&](u32 cl, u32 st, unsigned t) -> u32& { return cnt[((size_t)cl * S + st) * T + t]; };
    par_chunks(P, [&](uint64_t lo, uint64_t hi, unsigned t) {
      for (uint64_t p = lo; p < hi; ++p)
        if (!c->is_sink[p]) at(cls[p], c->stage[p], t)++;
    });
    for (u32 st = 0; st < S; ++st) {
      u32 run = c->pull_stage_ptr[st];
      for (u32 cl = 0; cl < 3; ++cl)
        for (unsigned t = 0; t < T; ++t) {
          const u32 y = at(cl, st, t);
          at(cl, st, t) = run;
          run += y;
        }
    }
    par_chunks(P, [&](uint64_t lo, uint64_t hi, unsigned t) {
      for (uint64_t p = lo; p < hi; ++p)
        if (!c->is_sink[p]) {
          const u32 i = at(cls[p], c->stage[p], t)++;
          c->int_of_user[p] = i;
          c->user_of_int[i] = (u32)p;
        }
    });
    (void)fill;
  }
  c->sink_ptr.assign(NP + 1, 0);
  c->drv_of_net.assign(c->N, kNone);
  par_chunks(NP, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t i = lo; i < hi; ++i) {
      const u32 p = c->user_of_int[i];
      const u32 n = p == kNone ? kNone : c->pin_net[p];
      c->sink_ptr[i] = n == kNone ? 0 : c->net_ptr[n + 1] - c->net_ptr[n] - 1;
    }
  });
  excl_prefix(c->sink_ptr);
  par_chunks(NP, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t i = lo; i < hi; ++i) {
      const u32 p = c->user_of_int[i];
      if (p == kNone) continue;               // padding
      const u32 n = c->pin_net[p];
      if (n == kNone) continue;
      c->drv_of_net[n] = (u32)i;              // p is the driver of n
      u32 k = c->sink_ptr[i];
      for (u32 x = c->net_ptr[n] + 1; x < c->net_ptr[n + 1]; ++x, ++k) {
        const u32 sp = c->net_pins[x];
        c->int_of_user[sp] = NP + k;
        c->user_of_int[NP + k] = sp;
      }
    }
  });
  c->sink_stage_ptr.assign(S + 1, 0);
  for (u32 s = 0; s <= S; ++s) c->sink_stage_ptr[s] = c->sink_ptr[c->pull_stage_ptr[s]];

  tm.mark("plan: stages + numbering");
  // A non-unate arc's (irf -> orf) pairs are the union of the positive- and
  // negative-unate pairs, so it becomes two terms with the same
  // tables; every kernel item then evaluates exactly one pair per output edge
  // (no divergent second pass).  Min / max merges are order-free, so results
  // are unchanged.
  auto n_terms = [&](u32 a) { return c->arc_sense[a] == STA_NON_UNATE ? 2u : 1u; };
  auto term_info = [&](u32 a, u32 q) {
    const u32 sense = c->arc_sense[a] == STA_NON_UNATE ? (q ? STA_NEG_UNATE : STA_POS_UNATE) : c->arc_sense[a];
    return sta::pack_info(sense, c->arc_tab[a]);
  };

  // forward fan-in terms of pull pins (cell arcs, arc id order): counted,
  // prefix-summed, then filled in parallel
  std::vector<u32> fi_p(NP + 1, 0), arc_term(c->A, kNone);
  par_chunks(NP, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t i = lo; i < hi; ++i) {
      const u32 p = c->user_of_int[i];
      u32 n = 0;
      if (p != kNone)
        for (u32 x = fi_ptr[p]; x < fi_ptr[p + 1]; ++x) n += n_terms(fi_ids[x]);
      fi_p[i] = n;
    }
  });
  const u32 n_fi = excl_prefix(fi_p);
  std::vector<u32> fi_src(n_fi), fi_hop(n_fi), fi_info(n_fi);
  par_chunks(NP, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t i = lo; i < hi; ++i) {
      const u32 p = c->user_of_int[i];
      if (p == kNone) continue;
      u32 e = fi_p[i];
      for (u32 x = fi_ptr[p]; x < fi_ptr[p + 1]; ++x) {
        const u32 a = fi_ids[x], u = c->arc_from[a];
        arc_term[a] = e;
        for (u32 q = 0; q < n_terms(a); ++q, ++e) {
          if (c->is_sink[u]) {
            fi_src[e] = c->int_of_user[driver_of(u)];
            fi_hop[e] = c->int_of_user[u] - NP;
          } else {
            fi_src[e] = c->int_of_user[u];
            fi_hop[e] = kNone;
          }
          fi_info[e] = term_info(a, q);
        }
      }
    }
  });

  // backward: cell fan-out of sinks and of pull pins (same two passes)
  std::vector<u32> sfo_p(c->NS + 1, 0), pfo_p(NP + 1, 0);
  auto fo_count = [&](u32 u) {
    u32 n = 0;
    for (u32 x = fo_ptr[u]; x < fo_ptr[u + 1]; ++x) n += n_terms(fo_ids[x]);
    return n;
  };
  par_chunks(c->NS, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t kk = lo; kk < hi; ++kk) sfo_p[kk] = fo_count(c->user_of_int[NP + kk]);
  });
  par_chunks(NP, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t i = lo; i < hi; ++i) {
      const u32 u = c->user_of_int[i];
      pfo_p[i] = u == kNone ? 0 : fo_count(u);
    }
  });
  const u32 n_sfo = excl_prefix(sfo_p), n_pfo = excl_prefix(pfo_p);
  std::vector<u32> sfo_dst(n_sfo), sfo_info(n_sfo), pfo_dst(n_pfo), pfo_info(n_pfo);
  auto fo_fill = [&](u32 u, u32 e, std::vector<u32>& dst, std::vector<u32>& info) {
    for (u32 x = fo_ptr[u]; x < fo_ptr[u + 1]; ++x) {
      const u32 a = fo_ids[x];
      for (u32 q = 0; q < n_terms(a); ++q, ++e) {
        dst[e] = c->int_of_user[c->arc_to[a]];
        info[e] = arc_term[a] + q;             // term index; becomes sense | delay slot << 3 below
      }
    }
  };
  par_chunks(c->NS, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t kk = lo; kk < hi; ++kk) fo_fill(c->user_of_int[NP + kk], sfo_p[kk], sfo_dst, sfo_info);
  });
  par_chunks(NP, [&](uint64_t lo, uint64_t hi, unsigned) {
    for (uint64_t i = lo; i < hi; ++i)
      if (c->user_of_int[i] != kNone) fo_fill(c->user_of_int[i], pfo_p[i], pfo_dst, pfo_info);
  });

  tm.mark("plan: fan-in / fan-out terms");
  // backward warp tiles per stage: runs of <= 32 consecutive sinks that never
  // split a driver with <= 32 sinks; a driver with more sinks gets its own
  // tiles (heavy slot: atomics + last-tile finish).  Stage pins without sinks
  // are listed separately.
  std::vector<uint2> tiles;
  std::vector<u32> nosink, heavy_nchunk, heavy_base, tile_part;   // tile_part: partial slot of a heavy tile
  u32 n_parts = 0;
  c->tile_stage_ptr.assign(S + 1, 0);
  c->nosink_stage_ptr.assign(S + 1, 0);
  // Work-unit size adapts to the stage: a unit waits for the slowest of its
  // inputs, so small stages (latency-bound) use small units -- down to one
  // driver / pin per warp -- and large stages (throughput-bound) full ones.
  // Target: about half the persistent grid's warps per stage.
  u32 sms = 148;
  {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && n > 0)
      sms = (u32)n;
    cudaGetLastError();
  }
  const u32 fwd_warps = sms * (sta::kFwdThreads / 32) * sta::kFwdMinBlocks, bwd_warps = sms * (sta::kBwdThreads / 32) * sta::kBwdMinBlocks;
  auto unit_cap = [&](u64 items, u32 cap, u32 warps) {
    const u64 per = (items + warps / 2 - 1) / (warps / 2);
    return (u32)std::min<u64>(cap, std::max<u64>(1, per));
  };
  for (u32 s = 0; s < S; ++s) {
    c->tile_stage_ptr[s] = (u32)tiles.size();
    c->nosink_stage_ptr[s] = (u32)nosink.size();
    const u32 tcap = unit_cap(c->sink_ptr[c->pull_stage_ptr[s + 1]] - c->sink_ptr[c->pull_stage_ptr[s]], sta::kTile, bwd_warps);
    u32 cur = kNone, fill = 0;   // open light tile: first sink, lanes used
    for (u32 i = c->pull_stage_ptr[s]; i < c->pull_stage_ptr[s + 1]; ++i) {
      const u32 b = c->sink_ptr[i], n = c->sink_ptr[i + 1] - b;
      if (n == 0) {
        if (c->user_of_int[i] != kNone) nosink.push_back(i);   // padding has no work
        continue;
      }
      if (n > (u32)sta::kTile) {
        cur = kNone;
        const u32 slot = (u32)heavy_nchunk.size();
        const u32 nch = (n + sta::kTile - 1) / sta::kTile;
        heavy_base.push_back(n_parts);
        heavy_nchunk.push_back(nch);
        for (u32 q = 0; q < nch; ++q) {
          tiles.push_back(make_uint2(b + q * sta::kTile, slot));
          tile_part.push_back(n_parts++);
        }
        continue;
      }
      if (cur == kNone || fill + n > tcap) {
        cur = b;
        fill = 0;
        tiles.push_back(make_uint2(b, kNone));
        tile_part.push_back(kNone);
      }
      fill += n;
    }
  }
  c->tile_stage_ptr[S] = (u32)tiles.size();
  c->nosink_stage_ptr[S] = (u32)nosink.size();
  c->n_heavy = (u32)heavy_nchunk.size();
  c->n_heavy_parts = n_parts;

  // persistent-kernel work lists (warp-granular dataflow, sta_kernels.cu):
  // forward units are runs of consecutive pull pins of one stage with <=
  // kFwdUnitTerms fan-in terms (four lanes per term; a pin with more terms
  // is a unit of its own and its warp loops); stage-0 units are <=
  // kFwdUnitTerms seed pins.  Unit u is the kFwdUnitTerms term slots
  // [u kFwdUnitTerms, (u + 1) kFwdUnitTerms) of fterm (layout in
  // sta_internal.h), so a lane's static data is one 16-byte load.  Backward
  // units are one tile of <= kTile sinks, or <= kTile sink-less pins, in
  // descending stage order.  Both lists are in dependency order: every unit
  // depends only on units with a smaller index.
  std::vector<uint4> fterm, bwu;           // forward term slots (kFwdUnitTerms per unit) / backward units
  // delay slot of each fan-in term: its unit slot, or past the unit slots for
  // the terms of heavy pins (the forward stores the term's four delays there,
  // the backward reads them)
  std::vector<u32> term_slot(fi_src.size(), kNone), heavy_units;
  std::vector<u32> fwu_stage, stage_sink_end(S);
  for (u32 s = 0; s < S; ++s) stage_sink_end[s] = c->sink_ptr[c->pull_stage_ptr[s + 1]];
  std::vector<u32> fi_pin(fi_src.size());
  for (u32 i = 0; i < NP; ++i)
    for (u32 e = fi_p[i]; e < fi_p[i + 1]; ++e) fi_pin[e] = i;
  const uint4 pad = make_uint4(kNone, kNone, 0, kNone);
  std::vector<u32> fwu_of_pin(NP, 0);     // forward unit writing each pull pin
  for (u32 s = 0; s < S; ++s) {
    const u32 p0 = c->pull_stage_ptr[s], p1 = c->pull_stage_ptr[s + 1];
    if (s == 0) {                          // seed units: slot = pin
      for (u32 p = p0; p < p1; p += sta::kFwdUnitTerms) {
        u32 n = 0;
        while (n < sta::kFwdUnitTerms && p + n < p1 && c->user_of_int[p + n] != kNone) ++n;
        if (!n) break;                                  // stage padding
        for (u32 x = 0; x < sta::kFwdUnitTerms; ++x) {
          fterm.push_back(make_uint4(sta::kSeedMark, 0, 0, x < n ? p + x : kNone));
          if (x < n) fwu_of_pin[p + x] = (u32)fwu_stage.size();
        }
        fwu_stage.push_back(s);
      }
      // U: a seed slot without a seed, so its record is written (undefined)
      // by every update
      for (u32 x = 0; x < sta::kFwdUnitTerms; ++x)
        fterm.push_back(make_uint4(sta::kSeedMark, 0, 0, x == 0 ? c->undef_pin : kNone));
      fwu_stage.push_back(s);
      continue;
    }
    const u32 fcap = unit_cap(fi_p[p1] - fi_p[p0], sta::kFwdUnitTerms, fwd_warps);
    // the stage's units {first pin, first term, terms}, then ordered by the
    // position of their latest-produced input (units of one stage are
    // independent): warps take units in list order, so a unit's inputs are
    // then most likely complete when its warp reaches it
    std::vector<uint3> su;
    std::vector<u64> key;
    u32 p = p0;
    while (p < p1) {
      while (p < p1 && fi_p[p + 1] == fi_p[p]) ++p;   // stage padding: no work
      if (p == p1) break;
      const u32 q0 = p;
      u32 items = 0;
      while (p < p1) {
        const u32 n = fi_p[p + 1] - fi_p[p];
        if (n == 0 || (items && items + n > fcap)) break;
        items += n;
        ++p;
      }
      su.push_back(make_uint3(q0, fi_p[q0], items));
    }
    // sort keys (parallel: random reads of the producers' unit positions)
    key.resize(su.size());
    par_chunks(su.size(), [&](uint64_t lo, uint64_t hi, unsigned) {
      for (uint64_t x = lo; x < hi; ++x) {
        u32 kmax = 0;
        for (u32 e = su[x].y; e < su[x].y + su[x].z; ++e) kmax = std::max(kmax, fwu_of_pin[fi_src[e]]);
        key[x] = (u64)kmax << 32 | x;
      }
    });
    std::sort(key.begin(), key.end());
    // emission in sorted order: unit r of the stage takes slots [8 (u0 + r), 8 (u0 + r + 1))
    const u32 u0 = (u32)fwu_stage.size();
    const size_t f0 = fterm.size();
    fterm.resize(f0 + (size_t)sta::kFwdUnitTerms * su.size());
    fwu_stage.resize(u0 + su.size(), s);
    std::vector<uint8_t> heavy_flag(su.size(), 0);
    std::atomic<bool> too_large{false};
    par_chunks(su.size(), [&](uint64_t lo, uint64_t hi, unsigned) {
      for (uint64_t r = lo; r < hi; ++r) {
        const uint3 un = su[(u32)key[r]];
        const u32 q0 = un.x, e0 = un.y, items = un.z;
        const u32 upos = u0 + (u32)r;
        uint4* ft = fterm.data() + f0 + (size_t)sta::kFwdUnitTerms * r;
        for (u32 e = e0; e < e0 + items; ++e) fwu_of_pin[fi_pin[e]] = upos;
        if (items > sta::kFwdUnitTerms) {  // one pin with many terms: the warp loops over fi_*
          // slot 0: {mark, first term, terms, pin}; slot 1: {mark, first delay slot}
          // (the delays of these terms live past the unit slots)
          heavy_flag[r] = 1;
          ft[0] = make_uint4(sta::kHeavyMark, e0, items, q0);
          ft[1] = make_uint4(sta::kHeavyMark, 0, 0, 0);
          for (u32 x = 2; x < sta::kFwdUnitTerms; ++x) ft[x] = make_uint4(sta::kHeavyMark, e0, items, q0);
        } else {
          for (u32 x = 0; x < sta::kFwdUnitTerms; ++x) {
            if (x >= items) {
              ft[x] = pad;
              continue;
            }
            const u32 e = e0 + x;
            if (fi_info[e] >> 31) too_large = true;
            term_slot[e] = (u32)(f0 + (size_t)sta::kFwdUnitTerms * r + x);
            ft[x] = make_uint4(fi_src[e], fi_hop[e], fi_info[e], fi_pin[e]);
          }
        }
      }
    });
    if (too_large) fail(STA_ERR_LUT, "table id too large for the forward plan");
    for (size_t r = 0; r < su.size(); ++r)
      if (heavy_flag[r]) heavy_units.push_back((u32)(f0 + (size_t)sta::kFwdUnitTerms * r));
  }
  {
    u32 next = (u32)fterm.size();
    for (u32 h : heavy_units) {
      fterm[h + 1].y = next;
      for (u32 x = 0; x < fterm[h].z; ++x) term_slot[fterm[h].y + x] = next++;
    }
    c->n_dslots = next;
    if (next >= (1u << 29)) fail(STA_ERR_ARG, "forward plan too large (%u term slots)", next);
    for (u32& x : sfo_info) x = (fi_info[x] & 7u) | term_slot[x] << 3;
    for (u32& x : pfo_info) x = (fi_info[x] & 7u) | term_slot[x] << 3;
  }
  tm.mark("plan: forward units");
  c->fwu_stage_ptr.assign(S + 1, 0);
  for (u32 s : fwu_stage) c->fwu_stage_ptr[s + 1]++;
  for (u32 s = 0; s < S; ++s) c->fwu_stage_ptr[s + 1] += c->fwu_stage_ptr[s];
  // backward units per stage (descending), ordered within a stage by the
  // position of the latest unit producing a required time they read (units
  // of one stage are independent), like the forward's
  std::vector<u32> drv_of_sink(c->NS);
  for (u32 i = 0; i < NP; ++i)
    for (u32 x = c->sink_ptr[i]; x < c->sink_ptr[i + 1]; ++x) drv_of_sink[x] = i;
  std::vector<u32> bwu_of_pin(NP, 0);     // backward unit finishing each pull pin
  c->bwu_stage_lo.assign(S, 0);
  c->bwu_stage_hi.assign(S, 0);
  for (u32 s = S; s-- > 0;) {
    c->bwu_stage_lo[s] = (u32)bwu.size();
    std::vector<uint4> su;
    std::vector<u64> key;
    auto reads_pin = [&](u32 i, u32& kmax) {   // pull pin i's direct fan-out
      for (u32 f = pfo_p[i]; f < pfo_p[i + 1]; ++f) kmax = std::max(kmax, bwu_of_pin[pfo_dst[f]]);
    };
    for (u32 x = c->tile_stage_ptr[s]; x < c->tile_stage_ptr[s + 1]; ++x) {
      const u32 k1 = x + 1 < c->tile_stage_ptr[s + 1] ? tiles[x + 1].x : stage_sink_end[s];
      su.push_back(make_uint4(tiles[x].x, k1, tiles[x].y, tile_part[x] == kNone ? 0 : 2 + tile_part[x]));
    }
    const u32 ncap = unit_cap(c->nosink_stage_ptr[s + 1] - c->nosink_stage_ptr[s], sta::kTile, bwd_warps);
    for (u32 x = c->nosink_stage_ptr[s]; x < c->nosink_stage_ptr[s + 1]; x += ncap) {
      const u32 x1 = std::min<u32>(x + ncap, c->nosink_stage_ptr[s + 1]);
      if (nosink[x1 - 1] - nosink[x] != x1 - 1 - x) fail(STA_ERR_ARG, "internal: sink-less pins not contiguous");
      su.push_back(make_uint4(nosink[x], nosink[x1 - 1] + 1, 0, 1));
    }
    // sort keys in parallel (random reads of the producers' unit positions)
    key.resize(su.size());
    par_chunks(su.size(), [&](uint64_t lo, uint64_t hi, unsigned) {
      for (uint64_t x = lo; x < hi; ++x) {
        const uint4 un = su[x];
        u32 kmax = 0;
        if (un.w == 1) {
          for (u32 i = un.x; i < un.y; ++i) reads_pin(i, kmax);
        } else {
          for (u32 k = un.x; k < un.y; ++k) {
            for (u32 f = sfo_p[k]; f < sfo_p[k + 1]; ++f) kmax = std::max(kmax, bwu_of_pin[sfo_dst[f]]);
            if (k == un.x || drv_of_sink[k] != drv_of_sink[k - 1]) reads_pin(drv_of_sink[k], kmax);
          }
        }
        key[x] = (u64)kmax << 32 | x;
      }
    });
    std::sort(key.begin(), key.end());
    for (u64 kk : key) {
      const uint4 un = su[(u32)kk];
      const u32 upos = (u32)bwu.size();
      if (un.w == 1) {
        for (u32 i = un.x; i < un.y; ++i) bwu_of_pin[i] = upos;
      } else {
        for (u32 k = un.x; k < un.y; ++k) bwu_of_pin[drv_of_sink[k]] = std::max(bwu_of_pin[drv_of_sink[k]], upos);
      }
      bwu.push_back(un);
    }
    c->bwu_stage_hi[s] = (u32)bwu.size();
  }
  c->n_fwu = (u32)fwu_stage.size();
  c->n_bwu = (u32)bwu.size();
  c->fwu_stage_h = fwu_stage;
  c->bwu_stage_h.resize(bwu.size());
  c->bwu_kind_h.resize(bwu.size());
  for (size_t x = 0; x < bwu.size(); ++x) c->bwu_kind_h[x] = bwu[x].w == 1 ? 2 : bwu[x].z != kNone ? 1 : 0;
  for (u32 s = 0; s < S; ++s)
    for (u32 x = c->bwu_stage_lo[s]; x < c->bwu_stage_hi[s]; ++x) c->bwu_stage_h[x] = s;

  std::vector<u32>& sink_drv = c->sink_drv;
  sink_drv.assign(c->NS, 0);
  for (u32 i = 0; i < NP; ++i)
    for (u32 x = c->sink_ptr[i]; x < c->sink_ptr[i + 1]; ++x) sink_drv[x] = i;
  c->fi_p_h = fi_p;                        // (the path report's per-pin term ranges / delay slots)
  c->fi_slot_h = term_slot;
  c->sfo_p = sfo_p;
  c->pfo_p = pfo_p;
  c->sfo_dst = sfo_dst;
  c->sfo_info = sfo_info;
  c->pfo_dst = pfo_dst;
  c->pfo_info = pfo_info;

  tm.mark("plan: backward units");
  // upload
  cudaStream_t s = c->stream;
  Arena& g = c->graph_arena;
  sta::Topo& t = c->topo;
  t = sta::Topo{};
  t.P = P; t.NP = NP; t.NS = c->NS; t.S = S; t.N = c->N; t.n0 = c->n0;
  t.fi_src = g.upload(fi_src, s);
  t.fi_hop = g.upload(fi_hop, s);
  t.fi_info = g.upload(fi_info, s);
  t.sink_ptr = g.upload(c->sink_ptr, s);
  t.sink_drv = g.upload(sink_drv, s);
  t.sfo_dst = g.upload(sfo_dst, s);
  t.sfo_info = g.upload(sfo_info, s);
  t.pfo_dst = g.upload(pfo_dst, s);
  t.pfo_info = g.upload(pfo_info, s);
  t.fterm = g.upload(fterm, s);
  // (host copies for case analysis: moved, the uploads above staged them)
  c->fterm_h = std::move(fterm);
  c->fi_src_h = std::move(fi_src);
  c->fi_hop_h = std::move(fi_hop);
  c->arc_term_h = std::move(arc_term);
  t.n_fwu = c->n_fwu;
  t.bwu = g.upload(bwu, s);
  t.n_bwu = c->n_bwu;
  t.n_bwu_static = S ? c->bwu_stage_lo[0] : 0;
  t.nosink = g.upload(nosink, s);
  t.heavy_nchunk = g.upload(heavy_nchunk, s);
  t.heavy_base = g.upload(heavy_base, s);
  t.int_of_user = g.upload(c->int_of_user, s);
  t.drv_of_net = g.upload(c->drv_of_net, s);
  c->fterm_d0 = t.fterm;
  c->fi_src_d0 = t.fi_src;
  c->fi_hop_d0 = t.fi_hop;
  c->sfo_info_d0 = t.sfo_info;
  c->pfo_info_d0 = t.pfo_info;
  ck(cudaStreamSynchronize(s), "plan upload");
  tm.mark("plan: upload");
}

// Row f4: case analysis (the oracle's O16; DESIGN.md
// C1-C4).  Constants from the case values are carried over nets (a sink
// takes its driver's constant) and through the cells' logic functions (an
// output is constant when its function takes one value for every completion
// of its non-constant inputs), pull pins in internal order (gate stage
// order: every input of a stage-s pin is final before it); a pin with two
// constants is an error.  Disabled: cell arcs from / to a constant pin or
// whose when guard is false for every completion, and net arcs from / to a
// constant pin ("killed" sinks).  Returns the disabled cell arcs.
std::vector<uint8_t> case_analysis(sta_ctx c, std::vector<uint8_t>& kill) {
  const u32 P = c->P, NP = c->NP;
  std::vector<uint8_t> val(P, 2), arc_off(c->A, 0);
  std::vector<u32> fn_of(P, kNone);
  for (u32 f = 0; f + 1 < c->fn_in_ptr.size(); ++f) fn_of[c->fn_pin[f]] = f;
  auto eval = [&](u32 f, uint64_t tt) {      // 0 / 1: one value on every completion; 2: both
    const u32 b = c->fn_in_ptr[f], k = c->fn_in_ptr[f + 1] - b;
    bool s0 = false, s1 = false;
    for (u32 m = 0; m < (1u << k); ++m) {
      bool ok = true;
      for (u32 j = 0; j < k && ok; ++j) {
        const uint8_t v = val[c->fn_in[b + j]];
        if (v != 2 && v != ((m >> j) & 1u)) ok = false;
      }
      if (!ok) continue;
      if ((tt >> m) & 1u) s1 = true; else s0 = true;
    }
    return s0 && s1 ? 2 : (s1 ? 1 : 0);
  };
  auto pin_const = [&](u32 p, uint8_t v) {
    if (val[p] != 2 && val[p] != v) fail(STA_ERR_ARG, "case analysis: contradictory constants on pin %u", p);
    val[p] = v;
  };
  for (size_t k = 0; k < c->case_pin.size(); ++k) pin_const(c->case_pin[k], c->case_val[k] ? 1 : 0);
  for (u32 i = 0; i < NP; ++i) {
    const u32 p = c->user_of_int[i];
    if (p == kNone) continue;
    if (fn_of[p] != kNone) {
      const int v = eval(fn_of[p], c->fn_tt[fn_of[p]]);
      if (v != 2) pin_const(p, (uint8_t)v);
    }
    if (val[p] != 2)
      for (u32 k = c->sink_ptr[i]; k < c->sink_ptr[i + 1]; ++k) pin_const(c->user_of_int[NP + k], val[p]);
  }
  kill.assign(c->NS, 0);
  for (u32 k = 0; k < c->NS; ++k)
    kill[k] = val[c->user_of_int[NP + k]] != 2 || val[c->user_of_int[c->sink_drv[k]]] != 2;
  for (u32 a = 0; a < c->A; ++a) {
    const u32 u = c->arc_from[a], v = c->arc_to[a];
    bool off = val[u] != 2 || val[v] != 2;
    if (!off && !c->arc_when.empty() && fn_of[v] != kNone && eval(fn_of[v], c->arc_when[a]) == 0) off = true;
    arc_off[a] = off;
  }
  return arc_off;
}

// RC tree topology: validation and per-net schedules (tree scope)
void build_rc(sta_ctx c) {
  PhaseTimer tm;
  const u32 N = c->N;
  // validation
  if (c->rc_ptr.size() != N + 1) fail(STA_ERR_ARG, "rc_ptr must have num_nets + 1 entries");
  if (N && c->rc_ptr[0] != 0) fail(STA_ERR_CSR, "rc_ptr[0] = %u, expected 0", c->rc_ptr[0]);
  for (u32 n = 0; n < N; ++n)
    if (c->rc_ptr[n + 1] < c->rc_ptr[n]) fail(STA_ERR_CSR, "rc net %u: offsets not monotone", n);
  if (N && c->rc_ptr[N] != c->n_rc) fail(STA_ERR_CSR, "rc_ptr[N] = %u != num_nodes %u", c->rc_ptr[N], c->n_rc);
  std::vector<u32> seen(c->P, 0);
  for (u32 n = 0; n < N; ++n) {
    const u32 b = c->rc_ptr[n], m = c->rc_ptr[n + 1] - b;
    if (!m) continue;
    const u32 drv = c->net_pins[c->net_ptr[n]];
    if (c->rc_parent[b] != -1) fail(STA_ERR_RC, "rc net %u: node 0 must have parent -1", n);
    if (c->rc_node_pin[b] != kNone && c->rc_node_pin[b] != drv)
      fail(STA_ERR_RC, "rc net %u: node 0 maps pin %u, not the driver %u", n, c->rc_node_pin[b], drv);
    for (u32 i = 1; i < m; ++i) {
      const int32_t pa = c->rc_parent[b + i];
      if (pa < 0 || (u32)pa >= i) fail(STA_ERR_RC, "rc net %u node %u: parent %d not in [0, %u)", n, i, pa, i);
      const u32 pin = c->rc_node_pin[b + i];
      if (pin == kNone) continue;
      if (pin >= c->P || c->pin_net[pin] != n || !c->is_sink[pin])
        fail(STA_ERR_RC, "rc net %u node %u: pin %u is not a sink of the net", n, i, pin);
      if (seen[pin]++) fail(STA_ERR_RC, "rc net %u: sink pin %u mapped to two nodes", n, pin);
    }
    for (u32 x = c->net_ptr[n] + 1; x < c->net_ptr[n + 1]; ++x)
      if (!seen[c->net_pins[x]]) fail(STA_ERR_RC, "rc net %u: sink pin %u has no RC node", n, c->net_pins[x]);
  }

  // nets in caller order j; each net's RC nodes renumbered in DFS preorder
  // (children in increasing index order) into "internal nodes", so that a
  // subtree is a contiguous range [pos, end) and the kernels read topology
  // contiguously.  Internal nodes are grouped by tier: nets of 1..32 nodes
  // (warp tiles), then 33..kBNet (block tiles, packed densely), then larger
  // (tier C), each group in net order.  R and Cw stay in the caller's
  // node order (borrowed zero-copy), addressed through node_user.
  struct Group {
    std::vector<u32> user, meta, tag, z;
  } grp[3];
  std::vector<u32> net_drv;
  net_drv.reserve(N);
  std::vector<uint4> wtiles;                // warp tiles of nets with 1..32 nodes
  std::vector<uint2> btiles;                // block tiles of nets with 33..kBNet nodes (group-1 offsets)
  std::vector<u32> lumped_j, tierC;
  std::vector<u32> tc_end, tc_ev;
  auto tier_of = [](u32 m) { return m <= 32 ? 0 : m <= sta::kBNet ? 1 : 2; };
  auto lg = [](u32 x) { u32 r = 0; while ((1u << r) < x) ++r; return r; };
  // (1, parallel) depth of the deepest root path of every tier-A net
  std::vector<uint8_t> depth_lg(N, 0);
  par_chunks(N, [&](uint64_t lo, uint64_t hi, unsigned) {
    std::vector<u32> dp;
    for (uint64_t n = lo; n < hi; ++n) {
      const u32 ub = c->rc_ptr[n], m = c->rc_ptr[n + 1] - ub;
      if (m == 0 || m > 32) continue;
      u32 depth = 0;
      dp.assign(m, 0);
      for (u32 q = 1; q < m; ++q) depth = std::max(depth, dp[q] = dp[(u32)c->rc_parent[ub + q]] + 1);
      depth_lg[n] = (uint8_t)lg(depth);
    }
  });
  // (2, sequential, sizes only) nets in the caller's net order: the caller's
  // R / Cw arrays (borrowed, node order of the caller) are then read nearly
  // contiguously; the scattered 4-byte outputs (load per driver, Elmore per
  // sink) stay in L2.  Group offsets, warp / block tiles.
  std::vector<u32> net_x0(N, kNone), net_tile(N, kNone);
  u32 gsz[3] = {0, 0, 0};
  u32 wt_fill = 0, wt_cend = kNone;         // open warp tile: nodes, caller node one past its last
  for (u32 n = 0; n < N; ++n) {
    const u32 i = c->drv_of_net[n];
    if (i == kNone) continue;
    const u32 j = (u32)net_drv.size();
    const u32 ub = c->rc_ptr[n], m = c->rc_ptr[n + 1] - ub;
    net_drv.push_back(i);
    if (m == 0) {
      lumped_j.push_back(j);
      continue;
    }
    const int tier = tier_of(m);
    const u32 x0 = gsz[tier];
    net_x0[n] = x0;
    gsz[tier] += m;
    if (tier == 0) {
      if (wtiles.empty() || wt_fill + m > 32 || ub != wt_cend) {
        // a warp tile's caller nodes must be one contiguous range (the kernel
        // loads them by lane and permutes with a shuffle)
        wtiles.push_back(make_uint4(x0, 0, ub, 0));
        wt_fill = 0;
      }
      uint4& wt = wtiles.back();
      wt.y += m;
      wt_fill += m;
      wt_cend = ub + m;
      // rounds the warp kernel needs for this tile: ceil(log2) of the
      // largest net (segmented scan) and of the deepest root path (pointer
      // jumping; the root itself carries no resistance)
      wt.w = std::max(wt.w & 0xFFu, lg(m)) | (std::max((wt.w >> 8) & 0xFFu, (u32)depth_lg[n]) << 8);
      net_tile[n] = (u32)wtiles.size() - 1;
    } else if (tier == 1) {
      if (btiles.empty() || btiles.back().y + m > sta::kBNet) btiles.push_back(make_uint2(x0, 0));
      btiles.back().y += m;
    } else {
      tierC.push_back(n);
    }
  }
  for (int g = 0; g < 3; ++g) {
    grp[g].user.resize(gsz[g]);
    grp[g].meta.resize(gsz[g]);
    grp[g].tag.resize(gsz[g]);
    grp[g].z.resize(gsz[g]);
  }
  tc_end.resize(gsz[2]);
  // (3, parallel) each net's nodes renumbered in DFS preorder (children in
  // increasing index order)
  struct Dfs {
    std::vector<u32> cnt, ch, pos, endp, pre;
    std::vector<std::pair<u32, u32>> stack;
    void run(const int32_t* par, u32 m) {
      cnt.assign(m + 1, 0);
      ch.resize(m);
      pos.resize(m);
      endp.resize(m);
      pre.clear();
      for (u32 q = 1; q < m; ++q) cnt[(u32)par[q] + 1]++;
      for (u32 q = 0; q < m; ++q) cnt[q + 1] += cnt[q];
      {
        std::vector<u32> fill(cnt.begin(), cnt.end() - 1);
        for (u32 q = 1; q < m; ++q) ch[fill[(u32)par[q]]++] = q;
      }
      stack.assign(1, {0u, 0u});
      pos[0] = 0;
      pre.push_back(0);
      while (!stack.empty()) {
        const u32 nd = stack.back().first;
        if (cnt[nd] + stack.back().second < cnt[nd + 1]) {
          const u32 cld = ch[cnt[nd] + stack.back().second++];
          pos[cld] = (u32)pre.size();
          pre.push_back(cld);
          stack.push_back({cld, 0u});
        } else {
          endp[pos[nd]] = (u32)pre.size();
          stack.pop_back();
        }
      }
    }
  };
  par_chunks(N, [&](uint64_t lo, uint64_t hi, unsigned) {
    Dfs D;
    for (uint64_t n = lo; n < hi; ++n) {
      const u32 x0 = net_x0[n];
      if (x0 == kNone) continue;
      const u32 i = c->drv_of_net[n];
      const u32 ub = c->rc_ptr[n], m = c->rc_ptr[n + 1] - ub;
      const int tier = tier_of(m);
      Group& G = grp[tier];
      D.run(c->rc_parent.data() + ub, m);
      const u32 zb = tier == 0 ? wtiles[net_tile[n]].z : 0;
      for (u32 t2 = 0; t2 < m; ++t2) {
        const u32 q = D.pre[t2];
        const u32 un = ub + q;
        G.user[x0 + t2] = un;
        G.z[x0 + t2] = un - zb;
        if (tier == 0) {
          const u32 ppos = q ? D.pos[(u32)c->rc_parent[un]] : 0xFFu;
          G.meta[x0 + t2] = t2 | (ppos << 8) | (D.endp[t2] << 16);
        } else if (tier == 1) {
          const u32 ppos = q ? D.pos[(u32)c->rc_parent[un]] : 0x7FFu;
          G.meta[x0 + t2] = t2 | (ppos << 10) | (D.endp[t2] << 21);
        } else {
          G.meta[x0 + t2] = 0;                // tier C: tc_* arrays
          tc_end[x0 + t2] = x0 + D.endp[t2];
        }
        const u32 pin = c->rc_node_pin[un];
        u32 tag = kNone;
        if (t2 == 0) tag = i | 0x80000000u;                      // root: the driver
        else if (pin != kNone && c->is_sink[pin]) tag = c->int_of_user[pin] - c->NP;
        G.tag[x0 + t2] = tag;
      }
    }
  });
  // (4) tier C (> kBNet nodes): one global array of their nodes (each net in
  // preorder, as internally), subtree ends, and the Euler event sequence
  // (before entering position t2: exit every node whose subtree ends there,
  // deepest first; after the last node: exit the rest)
  tc_ev.reserve(2ull * gsz[2]);
  for (u32 n : tierC) {
    const u32 g0 = net_x0[n], m = c->rc_ptr[n + 1] - c->rc_ptr[n];
    std::vector<std::vector<u32>> ends_at(m + 1);
    for (u32 a2 = 0; a2 < m; ++a2) ends_at[tc_end[g0 + a2] - g0].push_back(a2);
    for (u32 t2 = 0; t2 <= m; ++t2) {
      for (auto it = ends_at[t2].rbegin(); it != ends_at[t2].rend(); ++it) tc_ev.push_back((g0 + *it) | 0x80000000u);
      if (t2 == m) break;
      tc_ev.push_back(g0 + t2);
    }
    if (tc_ev.size() != 2 * (size_t)(g0 + m)) fail(STA_ERR_RC, "internal error: Euler tour of net %u", n);
  }
  // concatenate the groups; rebase block tiles and tier-C internal ids
  const u32 nA = (u32)grp[0].user.size(), nB = (u32)grp[1].user.size();
  for (uint2& b : btiles) b.x += nA;
  std::vector<u32> node_user, node_meta, node_tag, node_z;
  node_user.reserve(c->n_rc);
  node_meta.reserve(c->n_rc);
  node_tag.reserve(c->n_rc);
  for (Group& G : grp) {
    node_user.insert(node_user.end(), G.user.begin(), G.user.end());
    node_meta.insert(node_meta.end(), G.meta.begin(), G.meta.end());
    node_tag.insert(node_tag.end(), G.tag.begin(), G.tag.end());
    node_z.insert(node_z.end(), G.z.begin(), G.z.end());
    G = Group{};
  }
  if (node_user.size() != c->n_rc)   // nets without a driver-order entry cannot exist
    fail(STA_ERR_RC, "internal error: %zu of %u RC nodes placed", node_user.size(), c->n_rc);

  c->big_total = (u32)tc_end.size();

  cudaStream_t s = c->stream;
  c->tree_arena.release();
  Arena& g = c->tree_arena;
  sta::Topo& t = c->topo;
  t.net_drv = g.upload(net_drv, s);
  c->node_meta_h = node_meta;
  c->node_tag_h = node_tag;
  c->node_z_h = std::move(node_z);
  c->tc_end_h = std::move(tc_end);
  c->n_rc_ab = nA + nB;
  t.n_wtiles = (u32)wtiles.size();
  t.wtiles = g.upload(wtiles, s);
  t.n_btiles = (u32)btiles.size();
  t.btiles = g.upload(btiles, s);
  t.n_lumped = (u32)lumped_j.size();
  t.lumped_j = g.upload(lumped_j, s);
  t.nC = (u32)tierC.size();
  t.nCn = c->big_total;
  {   // static event records {position | exit << 31, output tag of an enter event (kNone for exits)}
    std::vector<uint2> ev2(tc_ev.size());
    for (size_t e = 0; e < tc_ev.size(); ++e) {
      const u32 pos = tc_ev[e] & 0x7FFFFFFFu;
      ev2[e] = make_uint2(tc_ev[e], (tc_ev[e] >> 31) ? kNone : node_tag[nA + nB + pos]);
    }
    t.tc_ev = g.upload(ev2, s);
  }
  c->node_user = std::move(node_user);
  c->rc_net_j = std::move(net_drv);
  ck(cudaStreamSynchronize(s), "rc upload");
  tm.mark("rc tree: validate + schedule + upload");
}

// constraints + tree dependent arrays (endpoints, seeds, static node caps)
// The corners of ctx in launch batches of <= kMaxBatch, each corner's table
// pool placed in the batch's shared-memory image (global lookups if the image
// exceeds kLutSmemMax).
std::vector<sta::Batch> make_batches(sta_ctx c) {
  std::vector<sta::Batch> out;
  for (u32 k0 = 0; k0 < c->K; k0 += sta::kMaxBatch) {
    sta::Batch b{};
    b.K = std::min<u32>(sta::kMaxBatch, c->K - k0);
    u32 off = 0;
    for (u32 k = 0; k < b.K; ++k) {
      sta::CornerDev d = c->corners[k0 + k].dev;
      d.lut_off4 = off;
      off += d.lut_n4;
      b.c[k] = d;
    }
    b.smem_f4 = 16ull * off <= sta::kLutSmemMax ? off : 0;
    out.push_back(b);
  }
  return out;
}

// shared-memory limit and co-resident grids of the persistent kernels for
// the largest batch image
void size_kernels(sta_ctx c) {
  u32 mx = 0;
  for (const sta::Batch& b : make_batches(c)) mx = std::max(mx, b.smem_f4);
  c->smem_f4 = mx;
  if (16ull * mx + sta::kBwdExtraSmem > 48 * 1024) ck(sta::set_lut_smem_limit(16ull * mx), "smem attribute");
  c->pgrid = c->use_persistent ? sta::persistent_grid(mx, 0) : 0;
  c->pgrid_b = c->use_persistent ? sta::persistent_grid(mx, 1) : 0;
  if (!c->wgrid) c->wgrid = sta::rc_warp_grid();
}

void prepare(sta_ctx c) {
  if (c->prepared) return;
  invalidate_graph(c);
  size_kernels(c);
  const u32 P = c->P;
  if (c->NP >= 0x80000000u) fail(STA_ERR_ARG, "too many pins for the backward records");
  std::vector<u32> pi_idx(P, kNone), po_idx(P, kNone);
  for (u32 k = 0; k < c->pi_pin.size(); ++k) pi_idx[c->pi_pin[k]] = k;
  for (u32 k = 0; k < c->po_pin.size(); ++k) po_idx[c->po_pin[k]] = k;
  std::vector<float> po_ld(P, 0.f);
  for (u32 k = 0; k < c->po_pin.size(); ++k) po_ld[c->po_pin[k]] += c->po_load[k];

  // endpoints in increasing user pin id
  std::vector<u32> pin_ep(c->Pi, kNone);
  std::vector<u32>& ep_int = c->ep_int_h;
  ep_int.clear();
  c->path_arena.release();                 // the path report's device arrays are rebuilt lazily
  c->path_scratch.a.release();
  c->path_scratch = PathScratch{};
  c->fi_p_d = c->fi_slot_d = c->ep_int_d = c->uoi_d = nullptr;
  std::vector<sta::EpRec> ep;
  for (u32 p = 0; p < P; ++p) {
    if (po_idx[p] == kNone && c->chk_of_pin[p] == kNone) continue;
    sta::EpRec r;
    r.po = po_idx[p];
    r.chk_tab = c->chk_of_pin[p] == kNone ? kNone : c->chk_tab[c->chk_of_pin[p]];
    pin_ep[c->int_of_user[p]] = (u32)ep.size();
    ep_int.push_back(c->int_of_user[p]);
    ep.push_back(r);
  }
  c->n_ep = (u32)ep.size();
  // backward fan-out records (layout in sta_internal.h) and PO seeds
  std::vector<float4> po_seed(c->po_pin.size());
  for (u32 k = 0; k < c->po_pin.size(); ++k)   // fp32 arithmetic, as the kernels did it
    po_seed[k] = make_float4(-c->po_out_min[2 * k], -c->po_out_min[2 * k + 1], c->period - c->po_out_max[2 * k],
                             c->period - c->po_out_max[2 * k + 1]);
  auto fo_rec = [&](uint4* r, u32 aux, u32 e, const std::vector<u32>& ptr, const std::vector<u32>& dst,
                    const std::vector<u32>& info, u32 i) {
    const u32 f0 = ptr[i], nfo = ptr[i + 1] - f0;
    r[0] = make_uint4(aux, nfo, f0, e);
    if (e != kNone) {
      r[1] = make_uint4(ep[e].chk_tab, ep[e].po, 0, 0);
    } else {
      r[1] = make_uint4(nfo > 0 ? dst[f0] : kNone, nfo > 0 ? info[f0] : 0, nfo > 1 ? dst[f0 + 1] : kNone,
                        nfo > 1 ? info[f0 + 1] : 0);
    }
  };
  // row f4: case analysis -- patched copies of the term arrays: a disabled
  // cell arc's forward terms read U (always undefined, no net hop), its
  // backward terms carry sense 7 (not live); a sink whose net arc is
  // disabled (a constant sink: its cell fan-out is disabled too) gets no
  // fan-out terms and bit 31 of its CSR start (killed: no arrival, no
  // required-time contribution to its driver)
  {
    sta::Topo& tp = c->topo;
    c->case_arena.release();
    tp.fterm = c->fterm_d0;
    tp.fi_src = c->fi_src_d0;
    tp.fi_hop = c->fi_hop_d0;
    tp.sfo_info = c->sfo_info_d0;
    tp.pfo_info = c->pfo_info_d0;
  }
  std::vector<u32> sfo_info_c, pfo_info_c;
  const std::vector<u32>* sfo_info = &c->sfo_info;
  const std::vector<u32>* pfo_info = &c->pfo_info;
  std::vector<uint8_t> kill;
  if (c->case_on) {
    const std::vector<uint8_t> off = case_analysis(c, kill);
    std::vector<uint8_t> slot_off(c->n_dslots + 1, 0);
    std::vector<uint4> ft(c->fterm_h);
    std::vector<u32> fs(c->fi_src_h), fh(c->fi_hop_h);
    for (u32 a = 0; a < c->A; ++a) {
      if (!off[a] || c->arc_term_h[a] == kNone) continue;
      const u32 nt = c->arc_sense[a] == STA_NON_UNATE ? 2u : 1u;
      for (u32 q = 0; q < nt; ++q) {
        const u32 e = c->arc_term_h[a] + q, sl = c->fi_slot_h[e];
        fs[e] = c->undef_pin;
        fh[e] = kNone;
        slot_off[sl] = 1;
        if (sl < ft.size()) {
          ft[sl].x = c->undef_pin;
          ft[sl].y = kNone;
        }
      }
    }
    sfo_info_c = c->sfo_info;
    pfo_info_c = c->pfo_info;
    for (u32& x : sfo_info_c) if (slot_off[x >> 3]) x |= 7u;    // sense 7: not live
    for (u32& x : pfo_info_c) if (slot_off[x >> 3]) x |= 7u;
    sfo_info = &sfo_info_c;
    pfo_info = &pfo_info_c;
    sta::Topo& tp = c->topo;
    Arena& ca = c->case_arena;
    tp.fterm = ca.upload(ft, c->stream);
    tp.fi_src = ca.upload(fs, c->stream);
    tp.fi_hop = ca.upload(fh, c->stream);
    tp.sfo_info = ca.upload(sfo_info_c, c->stream);
    tp.pfo_info = ca.upload(pfo_info_c, c->stream);
  }
  std::vector<uint4> sinkfo(2 * (size_t)c->NS), pullfo(2 * (size_t)c->NP);
  for (u32 k = 0; k < c->NS; ++k) {
    // driver field bit 31: the driver has its own endpoint or direct cell
    // fan-out (its pullfo record must be read); most drivers have neither
    const u32 v = c->sink_drv[k];
    const bool work = pin_ep[v] != kNone || c->pfo_p[v + 1] != c->pfo_p[v];
    fo_rec(&sinkfo[2 * (size_t)k], v | (work ? 0x80000000u : 0u), pin_ep[c->NP + k], c->sfo_p, c->sfo_dst,
           *sfo_info, k);
    if (!kill.empty() && kill[k]) {           // a constant sink: no arrival, no fan-out
      uint4* r = &sinkfo[2 * (size_t)k];
      r[0].y = 0;
      r[0].z |= 0x80000000u;
      if (r[0].w == kNone) r[1] = make_uint4(kNone, 0, kNone, 0);
    }
  }
  for (u32 i = 0; i < c->NP; ++i) fo_rec(&pullfo[2 * (size_t)i], 0, pin_ep[i], c->pfo_p, c->pfo_dst, *pfo_info, i);
  // stage-0 seeds
  std::vector<u32> seed(c->n0, kNone);
  for (u32 i = 0; i < c->n0; ++i) {
    const u32 p = c->user_of_int[i];
    if (p == kNone) continue;
    if (c->pin_role[p] == STA_PIN_FF_CK) seed[i] = sta::kSeedClock;
    else if (pi_idx[p] != kNone) seed[i] = pi_idx[p];
  }
  // static node caps (pin cap + PO load, internal node order) and lumped net
  // loads (nets in driver order), in fp64 then rounded once
  std::vector<float> scap(c->n_rc, 0.f);
  for (u32 x = 0; x < c->n_rc; ++x) {
    const u32 pin = c->rc_node_pin[c->node_user[x]];
    if (pin != kNone) scap[x] = (float)((double)c->pin_cap[pin] + (double)po_ld[pin]);
  }
  std::vector<float> lumped;
  lumped.reserve(c->rc_net_j.size());
  for (u32 i : c->rc_net_j) {
    const u32 n = c->pin_net[c->user_of_int[i]];
    double sum = 0;
    for (u32 x = c->net_ptr[n]; x < c->net_ptr[n + 1]; ++x) {
      const u32 pin = c->net_pins[x];
      sum += (double)c->pin_cap[pin] + (double)po_ld[pin];
    }
    lumped.push_back((float)sum);
  }

  cudaStream_t s = c->stream;
  c->cons_arena.release();
  Arena& g = c->cons_arena;
  sta::Topo& t = c->topo;
  t.n_ep = c->n_ep;
  t.n_pi = (u32)c->pi_pin.size();
  t.n_po = (u32)c->po_pin.size();
  t.sinkfo = g.upload(sinkfo, s);
  t.pullfo = g.upload(pullfo, s);
  t.po_seed = g.upload(po_seed, s);
  t.ep = g.upload(ep, s);
  t.seed = g.upload(seed, s);
  t.ep_ovr = nullptr;
  // row f4: startpoint tags (the exception sets of the -from lists holding
  // each seeded stage-0 pin), one seed array and one endpoint-override array
  // per tag (X1-X6; the oracle's O13)
  c->exc_arena.release();
  c->exc_seed_d.clear();
  c->exc_ovr_d.clear();
  // multiple clocks: the clock pins' seeds become "virtual PI" entries after
  // the real ones, one per clock: arrival (0, T_c / 2), the clock slew
  std::vector<float> pi_at_v(c->pi_at), pi_slew_v(c->pi_slew);
  const u32 n_clk = (u32)c->clk_period.size();
  if (n_clk) {
    const u32 base = (u32)(c->pi_at.size() / 4);
    for (u32 k = 0; k < n_clk; ++k) {
      const float h = 0.5f * c->clk_period[k];
      const float a4[4] = {0.f, h, 0.f, h};
      for (int q = 0; q < 4; ++q) {
        pi_at_v.push_back(a4[q]);
        pi_slew_v.push_back(c->clock_slew);
      }
    }
    for (u32 i = 0; i < c->n0; ++i)
      if (seed[i] == sta::kSeedClock) seed[i] = base + c->pin_clk[c->user_of_int[i]];
    c->topo.seed = t.seed = g.upload(seed, s);
  }
  c->exc_thr_dst_d.clear();
  c->n_thr = 0;
  t.thr_pull = t.thr_sink = t.thr_dst = nullptr;
  t.thr_sk = nullptr;
  t.n_thr = t.n_thr_sk = t.thr_cur = 0;
  if (!c->exc_kind.empty() || n_clk) {
    const u32 E = (u32)c->exc_kind.size();
    // segment bits (the oracle's O15): exception e has the
    // ordered segments [from (if listed), through_1 .. through_m], one tag
    // bit each from base[e]; a path's bits of e are a prefix of them
    const bool has_thr = !c->exc_thr_ptr.empty() && c->exc_thr_ptr[E] > 0;
    std::vector<u32> base(E), nseg(E), has_from(E);
    u32 total = 0;
    for (u32 e = 0; e < E; ++e) {
      has_from[e] = c->exc_from_ptr[e + 1] > c->exc_from_ptr[e];
      nseg[e] = has_from[e] + (has_thr ? c->exc_thr_ptr[e + 1] - c->exc_thr_ptr[e] : 0);
      base[e] = total;
      total += nseg[e];
    }
    if (total > 32) fail(STA_ERR_ARG, "%u exception segments (-from and -through lists, at most 32)", total);
    // membership of pin p in segment k of exception e (sorted pin lists)
    std::vector<std::vector<u32>> segl(total);
    for (u32 e = 0; e < E; ++e)
      for (u32 k = 0; k < nseg[e]; ++k) {
        std::vector<u32>& L = segl[base[e] + k];
        if (has_from[e] && k == 0) {
          L.assign(c->exc_from.begin() + c->exc_from_ptr[e], c->exc_from.begin() + c->exc_from_ptr[e + 1]);
        } else {
          const u32 sg = c->exc_thr_ptr[e] + k - has_from[e];
          L.assign(c->exc_seg.begin() + c->exc_seg_ptr[sg], c->exc_seg.begin() + c->exc_seg_ptr[sg + 1]);
        }
        std::sort(L.begin(), L.end());
      }
    auto seg_has = [&](u32 e, u32 k, u32 p) {
      const std::vector<u32>& L = segl[base[e] + k];
      return std::binary_search(L.begin(), L.end(), p);
    };
    // one step of the tag automaton at pin p (start: p is the path's startpoint)
    auto adv = [&](u32 bits, u32 p, bool start) {
      for (u32 e = 0; e < E; ++e) {
        u32 k = 0;
        while (k < nseg[e] && ((bits >> (base[e] + k)) & 1u)) ++k;
        if (has_from[e] && k == 0) {
          if (!start || !seg_has(e, 0, p)) continue;
          bits |= 1u << base[e];
          k = 1;
        }
        while (k < nseg[e] && seg_has(e, k, p)) {
          bits |= 1u << (base[e] + k);
          ++k;
        }
      }
      return bits;
    };
    auto full = [&](u32 e, uint64_t tg) {
      const u32 mask = nseg[e] >= 32 ? 0xFFFFFFFFu : ((1u << nseg[e]) - 1u);
      return (((u32)tg >> base[e]) & mask) == mask;
    };
    // a startpoint's tag: its launch clock (bits 32+) and its segment bits
    std::vector<uint64_t> tagp(P, 0);
    for (u32 e = 0; e < E; ++e)
      if (has_from[e])
        for (u32 x = c->exc_from_ptr[e]; x < c->exc_from_ptr[e + 1]; ++x) {
          const u32 p = c->exc_from[x];
          tagp[p] = adv((u32)tagp[p], p, true);
        }
    if (has_thr)   // a startpoint may also begin a -through segment (from-less exceptions)
      for (u32 v : c->exc_seg) tagp[v] = adv((u32)tagp[v], v, true);
    if (n_clk)
      for (u32 p = 0; p < P; ++p) tagp[p] |= (uint64_t)c->pin_clk[p] << 32;
    // (setup, hold) relationship of a launch / capture period pair: the
    // first 1000 launch edges, the next capture edge (the oracle's O14)
    auto rel = [](double TL, double TC, double& rs, double& rh) {
      rs = std::numeric_limits<double>::infinity();
      rh = -rs;
      for (int i = 0; i < 1000; ++i) {
        const double a = i * TL, nxt = (std::floor(a / TC) + 1.0) * TC;
        rs = std::min(rs, nxt - a);
        rh = std::max(rh, nxt - TC - a);
      }
    };
    std::vector<uint64_t> tags;
    for (u32 p = 0; p < P; ++p) {
      const u32 i = c->int_of_user[p];
      if (i >= c->n0 || seed[i] == kNone) continue;
      if (std::find(tags.begin(), tags.end(), tagp[p]) == tags.end()) tags.push_back(tagp[p]);
    }
    if (tags.empty()) tags.push_back(0);
    // -through: the tags reached by advancing at the segments' pins (closure),
    // ordered by set segment bits (a tag only advances to tags after it)
    std::vector<u32> slot_of(has_thr ? P : 0, kNone), thr_pins;
    if (has_thr) {
      for (u32 v : c->exc_seg)
        if (slot_of[v] == kNone) { slot_of[v] = (u32)thr_pins.size(); thr_pins.push_back(v); }
      for (size_t i = 0; i < tags.size() && tags.size() <= 32; ++i)
        for (u32 v : thr_pins) {
          const uint64_t t2 = (tags[i] & ~0xFFFFFFFFull) | adv((u32)tags[i], v, false);
          if (std::find(tags.begin(), tags.end(), t2) == tags.end()) tags.push_back(t2);
        }
      std::stable_sort(tags.begin(), tags.end(), [](uint64_t a, uint64_t b) {
        return __builtin_popcount((u32)a) < __builtin_popcount((u32)b);
      });
    }
    if (tags.size() > 32) fail(STA_ERR_ARG, "%zu timing tags (at most 32)", tags.size());
    if (has_thr) {
      const u32 n_thr = (u32)thr_pins.size();
      std::vector<u32> tp(c->NP, kNone), ts(c->NS, kNone);
      std::vector<uint2> sk;
      for (u32 x = 0; x < n_thr; ++x) {
        const u32 i = c->int_of_user[thr_pins[x]];
        if (i < c->NP) tp[i] = x;
        else { ts[i - c->NP] = x; sk.push_back(make_uint2(i - c->NP, x)); }
      }
      c->n_thr = n_thr;
      t.n_thr = n_thr;
      t.n_thr_sk = (u32)sk.size();
      t.thr_pull = c->exc_arena.upload(tp, s);
      t.thr_sink = c->exc_arena.upload(ts, s);
      t.thr_sk = sk.empty() ? nullptr : c->exc_arena.upload(sk, s);
      for (uint64_t tg : tags) {
        std::vector<u32> dst(n_thr, kNone);
        for (u32 x = 0; x < n_thr; ++x) {
          const uint64_t t2 = (tg & ~0xFFFFFFFFull) | adv((u32)tg, thr_pins[x], false);
          if (t2 != tg) dst[x] = (u32)(std::find(tags.begin(), tags.end(), t2) - tags.begin());
        }
        c->exc_thr_dst_d.push_back(c->exc_arena.upload(dst, s));
      }
    }
    std::vector<std::vector<uint8_t>> in_to(E);
    for (u32 e = 0; e < E; ++e) {
      in_to[e].assign(P, 0);
      for (u32 x = c->exc_to_ptr[e]; x < c->exc_to_ptr[e + 1]; ++x) in_to[e][c->exc_to[x]] = 1;
    }
    for (uint64_t tg : tags) {
      const u32 lclk = (u32)(tg >> 32);
      std::vector<u32> sd(seed);
      for (u32 i = 0; i < c->n0; ++i) {
        const u32 p = c->user_of_int[i];
        if (p != kNone && sd[i] != kNone && tagp[p] != tg) sd[i] = kNone;   // another tag's startpoint
      }
      std::vector<uint4> ov(c->n_ep);
      for (u32 k = 0; k < c->n_ep; ++k) {
        const u32 p = c->user_of_int[ep_int[k]];
        // capture clock (a PO's own, a D pin's register clock) and the
        // relationship to this tag's launch clock; the base seeds assume one
        // clock of period T (setup T, hold 0)
        double Tcap = c->period, sh_l = 0.0, sh_e = 0.0;
        if (n_clk) {
          u32 cc = c->pin_clk[p];
          if (c->chk_of_pin[p] != kNone) cc = c->pin_clk[c->chk_ck[c->chk_of_pin[p]]];
          Tcap = c->clk_period[cc];
          double rs, rh;
          rel(c->clk_period[lclk], Tcap, rs, rh);
          sh_l = rs - (double)c->period;
          sh_e = rh;
        }
        int lf = -1, lm = -1, lc = -1, ef = -1, em = -1, ec = -1;
        for (u32 e = 0; e < E; ++e) {
          if (!full(e, tg)) continue;        // the tag has not matched all of e's segments
          if (c->exc_to_ptr[e + 1] > c->exc_to_ptr[e] && !in_to[e][p]) continue;
          switch (c->exc_kind[e]) {
            case STA_EXC_FALSE_PATH: if (lf < 0) lf = (int)e; if (ef < 0) ef = (int)e; break;
            case STA_EXC_MAX_DELAY: if (lm < 0) lm = (int)e; break;
            case STA_EXC_MIN_DELAY: if (em < 0) em = (int)e; break;
            case STA_EXC_MULTICYCLE: if (lc < 0) lc = (int)e; if (ec < 0) ec = (int)e; break;
          }
        }
        auto bits = [](float f) { u32 u; std::memcpy(&u, &f, 4); return u; };
        uint4 o = make_uint4(0, bits((float)sh_l), 0, bits((float)sh_e));
        if (lf >= 0) o.x = 2;
        else if (lm >= 0) { o.x = 1; o.y = bits(c->exc_value[lm]); }
        else if (lc >= 0) o.y = bits((float)(sh_l + ((double)c->exc_value[lc] - 1.0) * Tcap));
        if (ef >= 0) o.z = 2;
        else if (em >= 0) { o.z = 1; o.w = bits(c->exc_value[em]); }
        else if (ec >= 0) o.w = bits((float)(sh_e + ((double)c->exc_value[ec] - 1.0) * Tcap));
        ov[k] = o;
      }
      c->exc_seed_d.push_back(c->exc_arena.upload(sd, s));
      c->exc_ovr_d.push_back(c->exc_arena.upload(ov, s));
    }
  }
  t.pi_at = reinterpret_cast<const float4*>(g.upload(pi_at_v, s));
  t.pi_slew = reinterpret_cast<const float4*>(g.upload(pi_slew_v, s));
  t.po_out_max = reinterpret_cast<const float2*>(g.upload(c->po_out_max, s));
  t.po_out_min = reinterpret_cast<const float2*>(g.upload(c->po_out_min, s));
  t.period = c->period;
  t.clock_slew = c->clock_slew;
  t.net_lumped = g.upload(lumped, s);
  {   // packed per-node records of the small-net RC kernels (tiers A and B)
    std::vector<uint4> nodes(c->n_rc_ab);
    for (u32 x = 0; x < c->n_rc_ab; ++x) {
      u32 sc;
      std::memcpy(&sc, &scap[x], 4);
      nodes[x] = make_uint4(c->node_meta_h[x], c->node_tag_h[x], c->node_z_h[x], sc);
    }
    t.rc_node = g.upload(nodes, s);
    // tier C: {caller node, tag, subtree end, static cap}
    std::vector<uint4> tcn(c->big_total);
    for (u32 gq = 0; gq < c->big_total; ++gq) {
      const u32 x = c->n_rc_ab + gq;
      u32 sc;
      std::memcpy(&sc, &scap[x], 4);
      tcn[gq] = make_uint4(c->node_user[x], c->node_tag_h[x], c->tc_end_h[gq], sc);
    }
    t.tc_node = g.upload(tcn, s);
  }
  // row f1: the Arnoldi layout (internal nodes: each net contiguous in DFS
  // preorder) -- parents / subtree ends from the caller's tree
  c->arn_arena.release();
  t.net_model = (u32)c->net_model;
  t.arn_q = c->arn_q;
  t.n_arn_nets = 0;
  t.n_arn_big = 0;
  t.n_rc_nodes = c->n_rc;
  if (c->net_model == 1) {
    std::vector<u32> inv(c->n_rc);
    for (u32 x = 0; x < c->n_rc; ++x) inv[c->node_user[x]] = x;
    std::vector<uint4> an(c->n_rc), nets;
    std::vector<u32> sz;
    for (u32 n = 0; n < c->N; ++n) {
      const u32 drv = c->drv_of_net[n];
      if (drv == kNone) continue;
      const u32 b = c->rc_ptr[n], m = c->rc_ptr[n + 1] - b;
      if (!m) {
        nets.push_back(make_uint4(0, 0, drv, 0));
        continue;
      }
      sz.assign(m, 1);
      for (u32 i = m - 1; i >= 1; --i) sz[(u32)c->rc_parent[b + i]] += sz[i];
      for (u32 i = 0; i < m; ++i) {
        const u32 x = inv[b + i];
        const u32 tag = c->node_tag_h[x];
        an[x] = make_uint4(b + i, i ? inv[b + (u32)c->rc_parent[b + i]] : kNone, x + sz[i],
                           (i && !(tag & 0x80000000u)) ? tag : kNone);
      }
      nets.push_back(make_uint4(inv[b], m, drv, 0));
    }
    t.n_arn_nets = (u32)nets.size();
    t.arn_nets = c->arn_arena.upload(nets, s);
    std::vector<u32> big;
    for (u32 j = 0; j < t.n_arn_nets; ++j)
      if (nets[j].y > 1024) big.push_back(j);
    t.n_arn_big = (u32)big.size();
    t.arn_big = c->arn_arena.upload(big, s);
    t.arn_node = c->arn_arena.upload(an, s);
    t.arn_scap = c->arn_arena.upload(scap, s);
  }

  // per-corner state buffers
  for (CornerState& cs : c->corners) {
    cs.state_arena.release();
    Arena& a = cs.state_arena;
    sta::CornerDev& d = cs.dev;
    d.rec = a.alloc<uint4>(4 * (size_t)c->NP);
    d.rat_ll = a.alloc<uint4>(2 * (size_t)c->NP);
    d.at4 = a.alloc<float4>(c->NP);
    d.tdel = a.alloc<float4>(std::max<u32>(c->n_dslots, 1));
    d.epoch = a.alloc<u32>(1);
    ck(cudaMemsetAsync(d.rec, 0, sizeof(uint4) * 4 * (size_t)c->NP, s), "memset");
    ck(cudaMemsetAsync(d.rat_ll, 0, sizeof(uint4) * 2 * (size_t)c->NP, s), "memset");
    d.rat = a.alloc<float4>(c->Pi);
    d.slack = a.alloc<float4>(c->Pi);
    d.elm = a.alloc<float>(c->NS);
    d.load = a.alloc<float>(c->NP);
    d.ep_ws = a.alloc<float2>(c->n_ep);
    d.res = a.alloc<double>(4);
    d.red_part = a.alloc<double>(4 * sta::kRedBlocks);
    d.red_cnt = a.alloc<u32>(2);
    ck(cudaMemsetAsync(d.red_cnt, 0, 2 * sizeof(u32), s), "memset");
    d.heavy_part = a.alloc<float4>(c->n_heavy_parts);
    d.heavy_cnt = a.alloc<u32>(c->n_heavy);
    d.scratch = a.alloc<double>(sta::tierC_scratch(c->big_total));
    ck(cudaMemsetAsync(d.scratch, 0, sizeof(double) * sta::tierC_scratch(c->big_total), s), "memset");
    d.err_flag = a.alloc<u32>(1);
    d.trace = nullptr;
    if (!c->trace_path.empty()) {   // debug: per-chunk / per-unit timestamps
      const size_t n = 4 * ((size_t)c->n_fwu + c->n_bwu);
      d.trace = a.alloc<unsigned long long>(n);
      ck(cudaMemsetAsync(d.trace, 0, n * sizeof(unsigned long long), s), "memset");
    }
    ck(cudaMemsetAsync(d.load, 0, sizeof(float) * std::max<u32>(c->NP, 1), s), "memset");
    d.m_pin = nullptr;
    d.m_ep_ws = nullptr;
    if (!c->exc_kind.empty() || !c->clk_period.empty()) {
      d.m_pin = a.alloc<float4>(4 * (size_t)std::max<u32>(c->Pi, 1));
      d.m_ep_ws = a.alloc<float2>(std::max<u32>(c->n_ep, 1));
    }
    d.thr_hat = d.thr_hsl = d.thr_hrat = nullptr;
    cs.p_rec.assign(1, d.rec);
    cs.p_at4.assign(1, d.at4);
    cs.p_tdel.assign(1, d.tdel);
    if (c->n_thr) {                          // -through handoff, [tags][slots]
      const size_t n = c->exc_thr_dst_d.size() * (size_t)c->n_thr;
      d.thr_hat = a.alloc<float4>(n);
      d.thr_hsl = a.alloc<float4>(n);
      d.thr_hrat = a.alloc<float4>(n);
      for (size_t j = 1; j < c->exc_thr_dst_d.size(); ++j) {   // per-pass forward results
        cs.p_rec.push_back(a.alloc<uint4>(4 * (size_t)c->NP));
        cs.p_at4.push_back(a.alloc<float4>(c->NP));
        cs.p_tdel.push_back(a.alloc<float4>(std::max<u32>(c->n_dslots, 1)));
        ck(cudaMemsetAsync(cs.p_rec.back(), 0, 64ull * c->NP, s), "memset");
      }
    }
    d.arn_lam = nullptr;
    d.arn_res = nullptr;
    d.arn_scr = nullptr;
    if (c->net_model == 1) {
      d.arn_lam = a.alloc<float4>(c->NP);
      d.arn_res = a.alloc<float4>(c->NS);
      d.arn_scr = a.alloc<double>(((size_t)c->arn_q + 4) * std::max<u32>(c->n_rc, 1));
      // drivers without a net: no sink reads them; mark every entry "Elmore" first
      ck(cudaMemsetAsync(d.arn_lam, 0xFF, sizeof(float4) * std::max<u32>(c->NP, 1), s), "memset");
    }
    ck(sta::launch_init_corner(t, d, c->n_heavy, s), "init kernel");
  }
  ck(cudaStreamSynchronize(s), "prepare upload");
  c->prepared = true;
}

// RC of one batch (tier C on the side stream beside the small nets), then the
// nets' reduced-order models under the Arnoldi model
u32 enqueue_rc(sta_ctx c, const sta::Batch& b, const sta::Topo& t) {
  cudaStream_t s = c->stream;
  u32 launches = 0;
  if (t.nC && std::getenv("STA_RC_SERIAL")) {
    ck(sta::launch_rc_tierC(t, b, s), "rc tier-C kernels");
  } else if (t.nC) {                         // tier C concurrently with the small nets
    ck(cudaEventRecord(c->fork_ev, s), "fork");
    ck(cudaStreamWaitEvent(c->side, c->fork_ev, 0), "fork wait");
    ck(sta::launch_rc_tierC(t, b, c->side), "rc tier-C kernels");
    ck(cudaEventRecord(c->join_ev, c->side), "join");
  }
  ck(sta::launch_rc(t, b, c->wgrid, s), "rc kernel");
  if (t.nC && !std::getenv("STA_RC_SERIAL")) ck(cudaStreamWaitEvent(s, c->join_ev, 0), "join wait");
  launches += (t.n_wtiles ? 1 : 0) + (t.n_btiles ? 1 : 0) + (t.n_lumped ? 1 : 0) + (t.nC ? 3 : 0);
  if (t.net_model == 1) {                    // row f1: the nets' reduced-order models
    ck(sta::launch_arn_reduce(t, b, s), "arnoldi kernel");
    launches += t.n_arn_nets ? 1 : 0;
  }
  return launches;
}

// Kernel sequence of one update of one batch of corners (see sta_kernels.cu);
// rc = false: a later exception tag of the same update (row f4), the RC
// results are shared
u32 enqueue_batch(sta_ctx c, const sta::Batch& b, const sta::Topo& t, bool rc, bool fwd = true) {
  cudaStream_t s = c->stream;
  u32 launches = 0;
  prof_mark(c, 0);
  if (rc) launches += enqueue_rc(c, b, t);
  prof_mark(c, 1);
  // (the Arnoldi and -through instantiations exist only as persistent kernels)
  if ((c->use_persistent && c->pgrid && c->pgrid_b) || t.net_model == 1 || t.thr_pull) {
    prof_mark(c, 2);
    if (fwd) ck(sta::launch_fwd_persistent(t, b, c->pgrid, s), "forward persistent kernel");
    else launches -= 1;                      // (-through: the forward ran in the first sweep)
    prof_mark(c, 3);
    prof_mark(c, 4);
    ck(sta::launch_bwd_persistent(t, b, c->pgrid_b, s), "backward persistent kernel");
    prof_mark(c, 5);
    prof_mark(c, 6);
    ck(sta::launch_reduce(t, b, s), "reduce kernel");
    prof_mark(c, 7);
    return launches + 3;
  }
  prof_mark(c, 2);
  for (u32 st = 0; st < c->S; ++st) {
    const u32 u0 = c->fwu_stage_ptr[st], u1 = c->fwu_stage_ptr[st + 1];
    ck(sta::launch_fwd_stage(t, b, u0, u1, s), "forward kernel");
    launches += u1 > u0 ? 1 : 0;
  }
  prof_mark(c, 3);
  prof_mark(c, 4);
  for (u32 st = c->S; st-- > 0;) {
    const u32 u0 = c->bwu_stage_lo[st], u1 = c->bwu_stage_hi[st];
    ck(sta::launch_bwd_stage(t, b, u0, u1, s), "backward kernel");
    launches += u1 > u0 ? 1 : 0;
  }
  prof_mark(c, 5);
  prof_mark(c, 6);
  ck(sta::launch_reduce(t, b, s), "reduce kernel");
  launches += 1;
  prof_mark(c, 7);
  return launches;
}

// One update of every batch; with exceptions (row f4) one forward / backward
// pass per tag (RC in the first only), each folded into the merged arrays,
// then WNS / TNS from the merged per-endpoint worst slacks.  With -through
// segments (the oracle's O15): a forward sweep in tag order hands the
// arrivals of advancing tags on (each pass into its own forward buffers, the
// record epoch advanced after each), then the backward passes run in reverse
// tag order, so that every pass finds the arrivals handed to it and the
// required times it takes over.
u32 enqueue_all(sta_ctx c, const std::vector<sta::Batch>& batches) {
  u32 launches = 0;
  if (c->exc_seed_d.empty()) {
    for (const sta::Batch& b : batches) launches += enqueue_batch(c, b, c->topo, true);
    return launches;
  }
  const size_t T = c->exc_seed_d.size();
  const bool thr = c->n_thr != 0;
  auto pass_topo = [&](size_t j) {
    sta::Topo tj = c->topo;
    tj.seed = c->exc_seed_d[j];
    tj.ep_ovr = c->exc_ovr_d[j];
    if (thr) {
      tj.thr_dst = c->exc_thr_dst_d[j];
      tj.thr_cur = (u32)j;
    }
    return tj;
  };
  // -through: every pass keeps its own forward results (CornerState::p_*)
  auto pass_batch = [&](const sta::Batch& b, size_t bi, size_t j) {
    sta::Batch bj = b;
    if (thr)
      for (u32 k = 0; k < b.K; ++k) {
        const CornerState& cs = c->corners[bi * sta::kMaxBatch + k];
        bj.c[k].rec = cs.p_rec[j];
        bj.c[k].at4 = cs.p_at4[j];
        bj.c[k].tdel = cs.p_tdel[j];
      }
    return bj;
  };
  if (thr) {
    for (const sta::Batch& b : batches) {
      ck(sta::launch_thr_reset(c->topo, b, (u32)T, c->stream), "through reset kernel");
      launches += 1;
    }
    for (size_t j = 0; j < T; ++j) {
      const sta::Topo tj = pass_topo(j);
      for (size_t bi = 0; bi < batches.size(); ++bi) {
        const sta::Batch bj = pass_batch(batches[bi], bi, j);
        if (j == 0) launches += enqueue_rc(c, bj, tj);
        ck(sta::launch_fwd_persistent(tj, bj, c->pgrid, c->stream), "forward persistent kernel");
        ck(sta::launch_thr_capture(tj, bj, c->stream), "through capture kernel");
        ck(sta::launch_bump_epoch(bj, c->stream), "epoch kernel");
        launches += 2 + (tj.n_thr_sk ? 1 : 0);
      }
    }
  }
  for (size_t jj = 0; jj < T; ++jj) {
    const size_t j = thr ? T - 1 - jj : jj;
    const sta::Topo tj = pass_topo(j);
    for (size_t bi = 0; bi < batches.size(); ++bi) {
      const sta::Batch bj = pass_batch(batches[bi], bi, j);
      // (-through: the forward of this pass ran in the first sweep, its hand-
      // over arrivals were complete then: every earlier tag ran before it)
      launches += enqueue_batch(c, bj, tj, !thr && jj == 0, !thr);
      for (u32 k = 0; k < bj.K; ++k) ck(sta::launch_merge_tag(tj, bj.c[k], jj == 0 ? 1 : 0, c->stream), "merge kernel");
      launches += bj.K;
    }
  }
  for (const sta::Batch& b : batches) {
    sta::Batch bm = b;
    for (u32 k = 0; k < b.K; ++k) bm.c[k].ep_ws = bm.c[k].m_ep_ws;
    ck(sta::launch_reduce(c->topo, bm, c->stream), "merged reduce kernel");
    launches += 1;
  }
  return launches;
}

// STA_TRACE=<path>: after an update, write the persistent kernels' per-chunk
// and per-unit {start, ready, end} timestamps of corner 0 and the stage of
// every chunk / unit (debug tooling: scripts/trace_report.py)
void dump_trace(sta_ctx c) {
  const sta::CornerDev& d = c->corners[0].dev;
  if (!d.trace) return;
  ck(cudaStreamSynchronize(c->stream), "sync");
  const size_t nch = c->n_fwu, n = 4 * (nch + c->n_bwu);
  std::vector<unsigned long long> h(n);
  ck(cudaMemcpy(h.data(), d.trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost), "D2H trace");
  FILE* f = std::fopen(c->trace_path.c_str(), "w");
  if (!f) return;
  std::fprintf(f, "kind,index,stage,start,ready,data,end,type\n");
  for (size_t x = 0; x < nch; ++x)
    std::fprintf(f, "fwd,%zu,%u,%llu,%llu,%llu,%llu,0\n", x, c->fwu_stage_h[x], h[4 * x], h[4 * x + 1], h[4 * x + 2],
                 h[4 * x + 3]);
  for (size_t u = 0; u < c->n_bwu; ++u) {
    const unsigned long long* q = &h[4 * (nch + u)];
    std::fprintf(f, "bwd,%zu,%u,%llu,%llu,%llu,%llu,%u\n", u, c->bwu_stage_h[u], q[0], q[1], q[2], q[3], c->bwu_kind_h[u]);
  }
  std::fclose(f);
}

void enqueue_update(sta_ctx c) {
  cudaStream_t s = c->stream;
  const std::vector<sta::Batch> batches = make_batches(c);
  if (!c->trace_path.empty()) {
    u32 launches = 0;
    launches += enqueue_all(c, batches);
    c->launches_per_update = launches;
    dump_trace(c);
    return;
  }
  if (!c->prof && c->use_graph) {
    if (!c->gexec) {
      cudaGraph_t g = nullptr;
      ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "begin capture");
      u32 launches = 0;
      try {
        launches += enqueue_all(c, batches);
      } catch (...) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      ck(cudaStreamEndCapture(s, &g), "end capture");
      cudaError_t e = cudaGraphInstantiate(&c->gexec, g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      ck(e, "graph instantiate");
      c->launches_per_update = launches;
    }
    ck(cudaGraphLaunch(c->gexec, s), "graph launch");
    return;
  }
  u32 launches = 0;
  prof_mark(c, 8);
  if (!c->exc_seed_d.empty()) launches += enqueue_all(c, batches);   // (per-phase times: not split)
  for (const sta::Batch& b : batches) {
    if (!c->exc_seed_d.empty()) break;
    launches += enqueue_batch(c, b, c->topo, true);
    if (c->prof) {
      // accumulate per phase (synchronous read of the event pairs)
      ck(cudaEventSynchronize(c->ev[7]), "event sync");
      for (int ph = 0; ph < 4; ++ph) {
        float ms = 0;
        ck(cudaEventElapsedTime(&ms, c->ev[2 * ph], c->ev[2 * ph + 1]), "elapsed");
        c->profile.ms[ph] += ms;
      }
    }
  }
  if (c->prof) {
    ck(cudaEventRecord(c->ev[9], s), "cudaEventRecord");
    ck(cudaEventSynchronize(c->ev[9]), "event sync");
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, c->ev[8], c->ev[9]), "elapsed");
    c->profile.ms[4] += ms;
    c->profile.launches[4] += launches;
    c->profile.updates += 1;
  }
  c->launches_per_update = launches;
}

// device error flag check after a sync
void check_flags(sta_ctx c) {
  for (size_t k = 0; k < c->corners.size(); ++k) {
    CornerState& cs = c->corners[k];
    if (!cs.dev.err_flag) continue;
    u32 f = 0;
    ck(cudaMemcpyAsync(&f, cs.dev.err_flag, sizeof f, cudaMemcpyDeviceToHost, c->stream), "flag D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
    if (f) {
      ck(cudaMemsetAsync(cs.dev.err_flag, 0, sizeof f, c->stream), "memset");
      fail(STA_ERR_RC, "corner %zu: negative or non-finite RC value in the borrowed arrays", k);
    }
  }
}

template <class F>
sta_status guard(sta_ctx c, F&& f) {
  if (!c) return STA_ERR_ARG;
  if (c->poisoned) {
    return STA_ERR_CUDA;
  }
  try {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != c->device) ck(cudaSetDevice(c->device), "cudaSetDevice");
    f();
    c->err.clear();
    return STA_OK;
  } catch (const StaError& e) {
    c->err = e.msg;
    if (e.st == STA_ERR_CUDA) c->poisoned = true;
    return e.st;
  } catch (const std::bad_alloc&) {
    c->err = "host allocation failed";
    return STA_ERR_OOM;
  }
}

CornerState& corner_of(sta_ctx c, u32 corner) {
  if (corner >= c->K) fail(STA_ERR_ARG, "corner %u out of range (ctx has %u)", corner, c->K);
  return c->corners[corner];
}

void require_updated(sta_ctx c) {
  if (!c->prepared) fail(STA_ERR_ORDER, "no timing update has been run");
}

// copy a device buffer of n elements to the caller (host or device)
template <class T>
void deliver(sta_ctx c, T* dst, const T* dev_src, size_t n, sta_mem mem) {
  if (!n) return;
  if (mem == STA_MEM_DEVICE) {
    ck(cudaMemcpyAsync(dst, dev_src, n * sizeof(T), cudaMemcpyDeviceToDevice, c->stream), "D2D");
  } else if (mem == STA_MEM_HOST) {
    ck(cudaMemcpyAsync(dst, dev_src, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream), "D2H");
    ck(cudaStreamSynchronize(c->stream), "sync");
  } else {
    fail(STA_ERR_ARG, "bad sta_mem %d", (int)mem);
  }
}

// gather a float4 per user pin (what: 0 at, 1 slew, 2 rat, 3 slack) into the
// caller buffer
void deliver_pins(sta_ctx c, float* dst, const sta::CornerDev& d, int what, sta_mem mem) {
  if (!dst || !c->P) return;
  const u32 P = c->P;
  float4* out;
  if (mem == STA_MEM_DEVICE) {
    out = reinterpret_cast<float4*>(dst);
  } else if (mem == STA_MEM_HOST) {
    c->tmp_arena.release();
    out = c->tmp_arena.alloc<float4>(P);
  } else {
    fail(STA_ERR_ARG, "bad sta_mem %d", (int)mem);
  }
  ck(sta::launch_gather_pins(c->topo, d, what, out, c->stream), "gather kernel");
  if (mem != STA_MEM_DEVICE) deliver(c, reinterpret_cast<float4*>(dst), out, P, STA_MEM_HOST);
}

// per-corner {res, cap} device pointer pair, rewritten in stream order by a
// one-thread kernel (no host staging, no host synchronization), so a captured
// update graph stays valid when the borrowed arrays change
void publish_rc_pointers(sta_ctx c, CornerState& cs) {
  if (!cs.dev.rc_vals) cs.dev.rc_vals = cs.ptr_arena.alloc<const float*>(2);
  ck(sta::launch_set_ptrs(cs.dev.rc_vals, cs.rc_res, cs.rc_cap, c->stream), "rc pointer kernel");
}

// ------------------------------------------------------------- row f2: Steiner RC
// Static plan of the construction (once per graph): each net's pins as
// driver then sinks by pin id, the nets by size class, the scratch arrays.
void steiner_plan(sta_ctx c) {
  if (c->steiner_ready) return;
  const u32 N = c->N, NNP = N ? c->net_ptr[N] : 0;
  std::vector<u32> spins(c->net_pins);
  std::vector<u32> warp, smem, big;
  u32 max_smem = 0, max_big = 0;
  const u32 lim = sta::steiner_smem_pins();
  for (u32 n = 0; n < N; ++n) {
    const u32 a = c->net_ptr[n], b = c->net_ptr[n + 1], m = b - a;
    std::sort(spins.begin() + a + 1, spins.begin() + b);
    if (m >= 2 && m <= 32) warp.push_back(n);
    else if (m > 32 && m <= lim) { smem.push_back(n); max_smem = std::max(max_smem, m); }
    else if (m > lim) { big.push_back(n); max_big = std::max(max_big, m); }
  }
  Arena& g = c->steiner_arena;
  cudaStream_t s = c->stream;
  c->st_net_ptr = g.upload(c->net_ptr, s);
  c->st_spins = g.upload(spins, s);
  c->st_warp = g.upload(warp, s);
  c->st_smem = g.upload(smem, s);
  c->st_big = g.upload(big, s);
  c->st_n_warp = (u32)warp.size();
  c->st_n_smem = (u32)smem.size();
  c->st_n_big = (u32)big.size();
  c->st_max_smem = max_smem;
  c->st_max_big = max_big;
  sta::SteinerArgs& a = c->st_args;
  a = sta::SteinerArgs{};
  a.net_ptr = c->st_net_ptr;
  a.spins = c->st_spins;
  a.ord = g.alloc<u32>(NNP);
  a.ppos = g.alloc<u32>(NNP);
  a.nodeix = g.alloc<u32>(NNP);
  a.cnt = g.alloc<u32>(N + 1);
  ck(cudaMemsetAsync(a.cnt, 0, sizeof(u32) * (N + 1), s), "memset");
  a.scratch = big.empty() ? nullptr : g.alloc<float4>(NNP);
  c->st_scan_bytes = sta::steiner_scan_bytes(N);
  c->st_scan = g.alloc<char>(c->st_scan_bytes);
  ck(cudaStreamSynchronize(s), "steiner plan");
  c->steiner_ready = true;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char* sta_status_string(sta_status st) {
  switch (st) {
    case STA_OK: return "STA_OK";
    case STA_ERR_ARG: return "STA_ERR_ARG";
    case STA_ERR_CSR: return "STA_ERR_CSR";
    case STA_ERR_ID: return "STA_ERR_ID";
    case STA_ERR_MULTIDRIVER: return "STA_ERR_MULTIDRIVER";
    case STA_ERR_CYCLE: return "STA_ERR_CYCLE";
    case STA_ERR_LUT: return "STA_ERR_LUT";
    case STA_ERR_RC: return "STA_ERR_RC";
    case STA_ERR_ORDER: return "STA_ERR_ORDER";
    case STA_ERR_CUDA: return "STA_ERR_CUDA";
    case STA_ERR_OOM: return "STA_ERR_OOM";
  }
  return "STA_ERR_UNKNOWN";
}

sta_status sta_create(int cuda_device, uint32_t num_corners, void* cuda_stream, sta_ctx* out) {
  if (!out || num_corners == 0) return STA_ERR_ARG;
  *out = nullptr;
  sta_ctx c = new (std::nothrow) sta_ctx_s;
  if (!c) return STA_ERR_OOM;
  c->device = cuda_device;
  c->K = num_corners;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) {
    delete c;
    return ndev == 0 ? STA_ERR_CUDA : STA_ERR_ARG;
  }
  if (cudaSetDevice(cuda_device) != cudaSuccess) { delete c; return STA_ERR_CUDA; }
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) { delete c; return STA_ERR_CUDA; }
    c->own_stream = true;
  }
  for (auto& e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) { delete c; return STA_ERR_CUDA; }
  int prio_lo = 0, prio_hi = 0;
  if (cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi) != cudaSuccess ||
      // (tier-C RC side stream at the default priority: measured 0.1-0.3 %
      // faster than high priority over the tier-A kernel; STA_SIDE_PRIO_HI)
      cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking,
                                   std::getenv("STA_SIDE_PRIO_HI") ? prio_hi : prio_lo) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->copy_ev, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return STA_ERR_CUDA;
  }
  c->corners.resize(num_corners);
  for (CornerState& cs : c->corners)
    for (auto& e : cs.free_ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) { delete c; return STA_ERR_CUDA; }
  if (const char* g = std::getenv("STA_NO_GRAPH")) c->use_graph = g[0] == '0';
  if (const char* g = std::getenv("STA_STAGE_KERNELS")) c->use_persistent = g[0] == '0';
  if (const char* g = std::getenv("STA_TRACE")) c->trace_path = g;
  *out = c;
  return STA_OK;
}

sta_status sta_destroy(sta_ctx c) {
  if (!c) return STA_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  c->graph_arena.release();
  c->tree_arena.release();
  c->cons_arena.release();
  c->tmp_arena.release();
  c->path_arena.release();
  c->path_scratch.a.release();
  cudaStreamSynchronize(c->copy);
  for (CornerState& cs : c->corners) {
    for (auto& e : cs.free_ev)
      if (e) cudaEventDestroy(e);
    cs.lib_arena.release();
    cs.rc_arena.release();
    cs.state_arena.release();
    cs.ptr_arena.release();
  }
  invalidate_graph(c);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->copy_ev) cudaEventDestroy(c->copy_ev);
  if (c->copy) cudaStreamDestroy(c->copy);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return STA_OK;
}

const char* sta_last_error(sta_ctx c) { return c ? c->err.c_str() : "null ctx"; }

sta_status sta_load_graph(sta_ctx c, const sta_graph_desc* d) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_load_graph");
    PhaseTimer tm;
    if (!d) fail(STA_ERR_ARG, "desc is NULL");
    c->has_graph = c->has_tree = c->has_cons = c->prepared = false;
    for (CornerState& cs : c->corners) { cs.lib = false; cs.rcv = false; }
    c->graph_arena.release();
    c->tree_arena.release();
    c->cons_arena.release();
    c->path_arena.release();
    c->path_scratch.a.release();
    c->path_scratch = PathScratch{};
    c->fi_p_d = c->fi_slot_d = c->ep_int_d = c->uoi_d = nullptr;
    c->steiner_arena.release();
    c->steiner_ready = false;
    c->exc_kind.clear();
    c->exc_value.clear();
    c->exc_from_ptr.clear();
    c->exc_from.clear();
    c->exc_to_ptr.clear();
    c->exc_to.clear();
    c->clk_period.clear();
    c->pin_clk.clear();
    c->P = d->num_pins; c->N = d->num_nets; c->A = d->num_arcs; c->C = d->num_checks; c->T = d->num_tables;
    c->pin_cap = fetch(d->pin_cap, c->P, d->mem, "pin_cap", c->stream);
    c->pin_role = fetch(d->pin_role, c->P, d->mem, "pin_role", c->stream);
    c->net_ptr = fetch(d->net_ptr, c->N ? c->N + 1 : 0, d->mem, "net_ptr", c->stream);
    const u32 nnp = c->N ? c->net_ptr[c->N] : 0;
    c->net_pins = fetch(d->net_pins, nnp, d->mem, "net_pins", c->stream);
    c->arc_from = fetch(d->arc_from, c->A, d->mem, "arc_from", c->stream);
    c->arc_to = fetch(d->arc_to, c->A, d->mem, "arc_to", c->stream);
    c->arc_sense = fetch(d->arc_sense, c->A, d->mem, "arc_sense", c->stream);
    c->arc_tab = fetch(d->arc_tab, c->A, d->mem, "arc_tab", c->stream);
    c->chk_d = fetch(d->chk_d, c->C, d->mem, "chk_d", c->stream);
    c->chk_ck = fetch(d->chk_ck, c->C, d->mem, "chk_ck", c->stream);
    c->chk_tab = fetch(d->chk_tab, c->C, d->mem, "chk_tab", c->stream);
    tm.mark("load: fetch");
    validate_graph(c);
    tm.mark("load: validate");
    build_plan(c);
    c->has_graph = true;
  });
}

sta_status sta_set_library(sta_ctx c, uint32_t corner, sta_mem mem, uint32_t num_tables, const uint8_t* n1,
                           const uint8_t* n2, const uint32_t* off, const float* data, uint32_t data_len) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_library");
    CornerState& cs = corner_of(c, corner);
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_set_library before sta_load_graph");
    if (num_tables != c->T) fail(STA_ERR_ARG, "library has %u tables, graph expects %u", num_tables, c->T);
    auto h1 = fetch(n1, num_tables, mem, "n1", c->stream);
    auto h2 = fetch(n2, num_tables, mem, "n2", c->stream);
    auto ho = fetch(off, num_tables, mem, "off", c->stream);
    auto hd = fetch(data, data_len, mem, "data", c->stream);
    // device pool (sta_internal.h): table blocks of kTabStride floats, then
    // deduplicated 16-byte aligned axis templates of kTmplStride floats
    const size_t tmpl0 = ((size_t)num_tables * sta::kTabStride + 3) / 4 * 4;
    std::vector<float> rec(tmpl0, 0.f);
    std::vector<std::vector<float>> tmpls;
    const float inf = std::numeric_limits<float>::infinity();
    for (u32 t = 0; t < num_tables; ++t) {
      const u32 a = h1[t], b = h2[t];
      if (a < 1 || a > 8 || b < 1 || b > 8) fail(STA_ERR_LUT, "table %u: size %ux%u outside 1..8", t, a, b);
      if ((uint64_t)ho[t] + a + b + (uint64_t)a * b > data_len) fail(STA_ERR_LUT, "table %u: data out of range", t);
      const float* x = hd.data() + ho[t];
      for (u32 k = 0; k < a + b + a * b; ++k)
        if (!std::isfinite(x[k])) fail(STA_ERR_LUT, "table %u: non-finite entry %u", t, k);
      for (u32 k = 1; k < a; ++k)
        if (!(x[k] > x[k - 1])) fail(STA_ERR_LUT, "table %u: index_1 not strictly ascending", t);
      for (u32 k = 1; k < b; ++k)
        if (!(x[a + k] > x[a + k - 1])) fail(STA_ERR_LUT, "table %u: index_2 not strictly ascending", t);
      std::vector<float> tm(sta::kTmplStride);
      auto axis = [&](const float* ax, u32 n, float* sx, float* xx, float* rx) {
        for (u32 k = 0; k < 8; ++k) {
          sx[k] = (k >= 1 && k + 2 <= n) ? ax[k] : inf;
          xx[k] = ax[std::min(k, n - 1)];
          if (k + 1 < n) {
            volatile float w = ax[k + 1] - ax[k];     // fp32 width, IEEE
            rx[k] = 1.0f / w;
          } else {
            rx[k] = 0.f;
          }
        }
      };
      axis(x, a, tm.data() + 0, tm.data() + 8, tm.data() + 16);
      axis(x + a, b, tm.data() + 24, tm.data() + 32, tm.data() + 40);
      size_t id = 0;
      while (id < tmpls.size() && std::memcmp(tmpls[id].data(), tm.data(), tm.size() * sizeof(float))) ++id;
      if (id == tmpls.size()) tmpls.push_back(tm);
      float* r = rec.data() + (size_t)t * sta::kTabStride;
      const int32_t toff = (int32_t)(tmpl0 + id * sta::kTmplStride);
      std::memcpy(r, &toff, sizeof toff);
      const float* v = x + a + b;
      for (u32 i = 0; i < 8; ++i)
        for (u32 j = 0; j < 8; ++j) r[1 + i * 8 + j] = v[std::min(i, a - 1) * b + std::min(j, b - 1)];
    }
    for (const auto& tm : tmpls) rec.insert(rec.end(), tm.begin(), tm.end());
    invalidate_graph(c);
    ck(cudaStreamSynchronize(c->stream), "sync");
    cs.lib_arena.release();
    while (rec.size() % 4) rec.push_back(0.f);
    cs.dev.lut = cs.lib_arena.upload(rec, c->stream);
    cs.lut_bytes = rec.size() * sizeof(float);
    cs.dev.lut_n4 = (u32)(rec.size() / 4);   // each corner stages its own pool size
    size_kernels(c);
    ck(cudaStreamSynchronize(c->stream), "library upload");
    cs.lib = true;
  });
}


sta_status sta_set_exceptions(sta_ctx c, const sta_exceptions* ex) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_exceptions");
    if (!ex) fail(STA_ERR_ARG, "exceptions NULL");
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_set_exceptions before sta_load_graph");
    const u32 E = ex->num;
    if (E > 32) fail(STA_ERR_ARG, "%u exceptions (at most 32)", E);
    std::vector<uint8_t> kind;
    std::vector<float> value;
    std::vector<u32> fp, fr, tp, to, th, sp, sg;
    if (E) {
      kind = fetch(ex->kind, E, ex->mem, "kind", c->stream);
      value = fetch(ex->value, E, ex->mem, "value", c->stream);
      fp = fetch(ex->from_ptr, E + 1, ex->mem, "from_ptr", c->stream);
      tp = fetch(ex->to_ptr, E + 1, ex->mem, "to_ptr", c->stream);
      if (fp[0] != 0 || tp[0] != 0) fail(STA_ERR_CSR, "from_ptr / to_ptr must start at 0");
      for (u32 e = 0; e < E; ++e)
        if (fp[e + 1] < fp[e] || tp[e + 1] < tp[e]) fail(STA_ERR_CSR, "exception %u: offsets not monotone", e);
      fr = fetch(ex->from_pins, fp[E], ex->mem, "from_pins", c->stream);
      to = fetch(ex->to_pins, tp[E], ex->mem, "to_pins", c->stream);
      for (u32 p : fr) if (p >= c->P) fail(STA_ERR_ID, "exception -from pin %u out of range", p);
      for (u32 p : to) if (p >= c->P) fail(STA_ERR_ID, "exception -to pin %u out of range", p);
      if (ex->thr_ptr) {                     // ordered -through segments
        th = fetch(ex->thr_ptr, E + 1, ex->mem, "thr_ptr", c->stream);
        if (th[0] != 0) fail(STA_ERR_CSR, "thr_ptr must start at 0");
        for (u32 e = 0; e < E; ++e)
          if (th[e + 1] < th[e]) fail(STA_ERR_CSR, "exception %u: -through offsets not monotone", e);
        if (th[E]) {
          sp = fetch(ex->seg_ptr, th[E] + 1, ex->mem, "seg_ptr", c->stream);
          if (sp[0] != 0) fail(STA_ERR_CSR, "seg_ptr must start at 0");
          for (u32 g = 0; g < th[E]; ++g)
            if (sp[g + 1] <= sp[g]) fail(STA_ERR_CSR, "-through segment %u: empty or offsets not monotone", g);
          sg = fetch(ex->seg_pins, sp[th[E]], ex->mem, "seg_pins", c->stream);
          for (u32 p : sg) if (p >= c->P) fail(STA_ERR_ID, "exception -through pin %u out of range", p);
        } else {
          th.clear();
        }
      }
      for (u32 e = 0; e < E; ++e) {
        if (kind[e] > STA_EXC_MIN_DELAY) fail(STA_ERR_ARG, "exception %u: kind %u", e, kind[e]);
        if (!std::isfinite(value[e])) fail(STA_ERR_ARG, "exception %u: non-finite value", e);
        if (kind[e] == STA_EXC_MULTICYCLE && !(value[e] >= 1.f && value[e] == std::floor(value[e])))
          fail(STA_ERR_ARG, "exception %u: multicycle needs an integer N >= 1", e);
      }
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->exc_kind = std::move(kind);
    c->exc_value = std::move(value);
    c->exc_from_ptr = std::move(fp);
    c->exc_from = std::move(fr);
    c->exc_to_ptr = std::move(tp);
    c->exc_to = std::move(to);
    c->exc_thr_ptr = std::move(th);
    c->exc_seg_ptr = std::move(sp);
    c->exc_seg = std::move(sg);
    c->prepared = false;                     // tags, seeds, overrides and merged arrays next update
    invalidate_graph(c);
  });
}

sta_status sta_set_case_analysis(sta_ctx c, const sta_case_analysis* ca) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_case_analysis");
    if (!ca) fail(STA_ERR_ARG, "case analysis NULL");
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_set_case_analysis before sta_load_graph");
    std::vector<u32> fp, fptr, fin, cp;
    std::vector<uint64_t> tt, when;
    std::vector<uint8_t> cv;
    const u32 F = ca->num_fn;
    if (F) {
      fp = fetch(ca->fn_pin, F, ca->mem, "fn_pin", c->stream);
      fptr = fetch(ca->fn_in_ptr, F + 1, ca->mem, "fn_in_ptr", c->stream);
      if (fptr[0] != 0) fail(STA_ERR_CSR, "fn_in_ptr must start at 0");
      for (u32 f = 0; f < F; ++f) {
        if (fptr[f + 1] < fptr[f]) fail(STA_ERR_CSR, "function %u: offsets not monotone", f);
        if (fptr[f + 1] - fptr[f] > 6) fail(STA_ERR_ARG, "function %u: %u inputs (at most 6)", f, fptr[f + 1] - fptr[f]);
      }
      fin = fetch(ca->fn_in, fptr[F], ca->mem, "fn_in", c->stream);
      tt = fetch(ca->fn_tt, F, ca->mem, "fn_tt", c->stream);
      std::vector<uint8_t> has(c->P, 0);
      for (u32 p : fp) {
        if (p >= c->P) fail(STA_ERR_ID, "function pin %u out of range", p);
        if (has[p]) fail(STA_ERR_ARG, "pin %u: two logic functions", p);
        has[p] = 1;
      }
      for (u32 p : fin) if (p >= c->P) fail(STA_ERR_ID, "function input pin %u out of range", p);
    } else {
      fptr.assign(1, 0);
    }
    if (ca->arc_when) when = fetch(ca->arc_when, c->A, ca->mem, "arc_when", c->stream);
    if (ca->num_case) {
      cp = fetch(ca->case_pin, ca->num_case, ca->mem, "case_pin", c->stream);
      cv = fetch(ca->case_val, ca->num_case, ca->mem, "case_val", c->stream);
      for (u32 p : cp) if (p >= c->P) fail(STA_ERR_ID, "case pin %u out of range", p);
      for (uint8_t v : cv) if (v > 1) fail(STA_ERR_ARG, "case value %u (0 or 1)", v);
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->fn_pin = std::move(fp);
    c->fn_in_ptr = std::move(fptr);
    c->fn_in = std::move(fin);
    c->fn_tt = std::move(tt);
    c->arc_when = std::move(when);
    c->case_pin = std::move(cp);
    c->case_val = std::move(cv);
    c->case_on = !c->case_pin.empty() || !c->arc_when.empty();
    c->prepared = false;
    invalidate_graph(c);
  });
}

sta_status sta_set_clocks(sta_ctx c, const sta_clocks* k) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_clocks");
    if (!k) fail(STA_ERR_ARG, "clocks NULL");
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_set_clocks before sta_load_graph");
    std::vector<float> per;
    std::vector<u32> pc;
    if (k->num_clocks) {
      if (k->num_clocks > 16) fail(STA_ERR_ARG, "%u clocks (at most 16)", k->num_clocks);
      per = fetch(k->period_ps, k->num_clocks, k->mem, "period_ps", c->stream);
      for (float v : per)
        if (!(v > 0.f) || !std::isfinite(v)) fail(STA_ERR_ARG, "clock periods must be finite and > 0");
      pc = fetch(k->pin_clk, c->P, k->mem, "pin_clk", c->stream);
      for (u32 p = 0; p < c->P; ++p)
        if (pc[p] >= k->num_clocks) fail(STA_ERR_ID, "pin %u: clock %u out of range", p, pc[p]);
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
    c->clk_period = std::move(per);
    c->pin_clk = std::move(pc);
    c->prepared = false;
    invalidate_graph(c);
  });
}

sta_status sta_set_net_model(sta_ctx c, sta_net_model model, uint32_t q) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_net_model");
    if (model != STA_NET_ELMORE && model != STA_NET_ARNOLDI) fail(STA_ERR_ARG, "net model %d", (int)model);
    if (model == STA_NET_ARNOLDI && (q < 1 || q > 4)) fail(STA_ERR_ARG, "Arnoldi order %u outside 1..4", q);
    if (c->net_model != (int)model || (model == STA_NET_ARNOLDI && c->arn_q != q)) {
      ck(cudaStreamSynchronize(c->stream), "sync");
      c->net_model = (int)model;
      if (model == STA_NET_ARNOLDI) c->arn_q = q;
      c->prepared = false;                   // layout / scratch / kernels of the next update
      invalidate_graph(c);
    }
  });
}

sta_status sta_build_steiner(sta_ctx c, sta_mem mem, const float* pin_x, const float* pin_y,
                             const sta_steiner_units* u, uint32_t node_capacity, uint32_t* rc_ptr,
                             int32_t* parent, uint32_t* node_pin, float* res, float* cap, uint32_t* num_nodes) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_build_steiner");
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_build_steiner before sta_load_graph");
    if (mem != STA_MEM_HOST && mem != STA_MEM_DEVICE) fail(STA_ERR_ARG, "bad sta_mem %d", (int)mem);
    if (!u) fail(STA_ERR_ARG, "units NULL");
    for (float v : {u->res_x, u->res_y, u->cap_x, u->cap_y})
      if (!(v >= 0.f) || !std::isfinite(v)) fail(STA_ERR_ARG, "Steiner units must be finite and >= 0");
    const u32 N = c->N, P = c->P, NNP = N ? c->net_ptr[N] : 0;
    const uint64_t need = 2ull * NNP - N;
    if (node_capacity < need) fail(STA_ERR_ARG, "node_capacity %u < %llu (2 * pins on nets - nets)",
                                   node_capacity, (unsigned long long)need);
    if (!rc_ptr || !parent || !node_pin || !res || !cap) fail(STA_ERR_ARG, "output arrays NULL");
    if (P && (!pin_x || !pin_y)) fail(STA_ERR_ARG, "positions NULL");
    steiner_plan(c);
    cudaStream_t s = c->stream;
    sta::SteinerArgs a = c->st_args;
    a.rx = u->res_x; a.ry = u->res_y; a.cx = u->cap_x; a.cy = u->cap_y;
    Arena tmp;
    struct Free { Arena& t; cudaStream_t s; ~Free() { cudaStreamSynchronize(s); t.release(); } } fr{tmp, s};
    if (mem == STA_MEM_HOST) {
      std::vector<float> hx(pin_x, pin_x + P), hy(pin_y, pin_y + P);
      for (u32 p = 0; p < P; ++p)
        if (!std::isfinite(hx[p]) || !std::isfinite(hy[p])) fail(STA_ERR_ARG, "pin %u: non-finite position", p);
      a.x = tmp.upload(hx, s);
      a.y = tmp.upload(hy, s);
      a.rc_ptr = tmp.alloc<u32>(N + 1);
      a.parent = tmp.alloc<int32_t>(need);
      a.node_pin = tmp.alloc<u32>(need);
      a.res = tmp.alloc<float>(need);
      a.cap = tmp.alloc<float>(need);
    } else {
      a.x = pin_x; a.y = pin_y;
      a.rc_ptr = rc_ptr; a.parent = parent; a.node_pin = node_pin; a.res = res; a.cap = cap;
    }
    ck(sta::run_steiner(a, N, c->st_warp, c->st_n_warp, c->st_smem, c->st_n_smem, c->st_big, c->st_n_big,
                        c->st_max_smem, c->st_max_big, c->st_scan, c->st_scan_bytes, s), "steiner kernels");
    u32 nn = 0;
    ck(cudaMemcpyAsync(&nn, a.rc_ptr + N, sizeof(u32), cudaMemcpyDeviceToHost, s), "D2H");
    ck(cudaStreamSynchronize(s), "steiner");
    if (num_nodes) *num_nodes = nn;
    if (mem == STA_MEM_HOST) {
      ck(cudaMemcpyAsync(rc_ptr, a.rc_ptr, sizeof(u32) * (N + 1), cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaMemcpyAsync(parent, a.parent, sizeof(int32_t) * nn, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaMemcpyAsync(node_pin, a.node_pin, sizeof(u32) * nn, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaMemcpyAsync(res, a.res, sizeof(float) * nn, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaMemcpyAsync(cap, a.cap, sizeof(float) * nn, cudaMemcpyDeviceToHost, s), "D2H");
      ck(cudaStreamSynchronize(s), "D2H");
    }
  });
}

sta_status sta_set_rc_tree(sta_ctx c, sta_mem mem, const uint32_t* rc_ptr, uint32_t num_nodes,
                           const int32_t* parent, const uint32_t* node_pin) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_rc_tree");
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_set_rc_tree before sta_load_graph");
    c->has_tree = false;
    c->prepared = false;
    for (CornerState& cs : c->corners) cs.rcv = false;
    c->n_rc = num_nodes;
    c->rc_ptr = fetch(rc_ptr, c->N + 1, mem, "rc_ptr", c->stream);
    c->rc_parent = fetch(parent, num_nodes, mem, "parent", c->stream);
    c->rc_node_pin = fetch(node_pin, num_nodes, mem, "node_pin", c->stream);
    build_rc(c);
    c->has_tree = true;
  });
}

sta_status sta_set_rc_values(sta_ctx c, uint32_t corner, sta_mem mem, const float* res, const float* cap) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_rc_values");
    CornerState& cs = corner_of(c, corner);
    if (!c->has_tree) fail(STA_ERR_ORDER, "sta_set_rc_values before sta_set_rc_tree");
    if (c->n_rc && (!res || !cap)) fail(STA_ERR_ARG, "res/cap NULL");
    if (mem == STA_MEM_DEVICE) {
      if (!cs.rc_arena.ptrs.empty()) {         // owned buffers of an earlier HOST call may be in use
        ck(cudaStreamSynchronize(c->stream), "sync");
        cs.rc_arena.release();
        cs.hcur = -1;
        cs.free_rec[0] = cs.free_rec[1] = false;
      }
      cs.rc_res = res;
      cs.rc_cap = cap;
      publish_rc_pointers(c, cs);
    } else if (mem == STA_MEM_HOST) {
      // copied into owned device buffers (page-locked caller buffers: DMA at
      // link speed) on the copy stream, into the buffer the updates already
      // enqueued do not read, so the copy runs beside an update still in
      // flight (an optimization loop's next values during this update); the
      // values are validated on the device by the RC kernels (STA_ERR_RC at
      // the next synchronizing call)
      if (cs.rc_arena.ptrs.empty() || cs.rc_arena.bytes < 4ull * c->n_rc * sizeof(float)) {
        ck(cudaStreamSynchronize(c->stream), "sync");
        cs.rc_arena.release();
        for (auto& b : cs.hbuf)
          for (auto& x : b) x = cs.rc_arena.alloc<float>(c->n_rc);
        cs.hcur = -1;
        cs.free_rec[0] = cs.free_rec[1] = false;
      }
      const int b = cs.hcur == 0 ? 1 : 0;
      if (cs.free_rec[b]) ck(cudaStreamWaitEvent(c->copy, cs.free_ev[b], 0), "copy wait");
      if (c->n_rc) {
        ck(cudaMemcpyAsync(cs.hbuf[b][0], res, sizeof(float) * c->n_rc, cudaMemcpyHostToDevice, c->copy), "H2D");
        ck(cudaMemcpyAsync(cs.hbuf[b][1], cap, sizeof(float) * c->n_rc, cudaMemcpyHostToDevice, c->copy), "H2D");
      }
      ck(cudaEventRecord(c->copy_ev, c->copy), "copy event");
      ck(cudaStreamWaitEvent(c->stream, c->copy_ev, 0), "copy join");
      cs.rc_res = cs.hbuf[b][0];
      cs.rc_cap = cs.hbuf[b][1];
      publish_rc_pointers(c, cs);
      if (cs.hcur >= 0) {                    // the old buffer is free once the work before this point is done
        ck(cudaEventRecord(cs.free_ev[cs.hcur], c->stream), "free event");
        cs.free_rec[cs.hcur] = true;
      }
      cs.hcur = b;
      ck(cudaStreamSynchronize(c->copy), "sync");   // host buffers read before return
    } else {
      fail(STA_ERR_ARG, "bad sta_mem %d", (int)mem);
    }
    cs.rcv = true;
  });
}

sta_status sta_set_constraints(sta_ctx c, const sta_constraints* k) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_set_constraints");
    if (!k) fail(STA_ERR_ARG, "constraints NULL");
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_set_constraints before sta_load_graph");
    if (!(k->period_ps > 0.f) || !std::isfinite(k->period_ps)) fail(STA_ERR_ARG, "period must be > 0");
    if (!(k->clock_slew_ps >= 0.f) || !std::isfinite(k->clock_slew_ps)) fail(STA_ERR_ARG, "clock slew must be >= 0");
    auto pi_pin = fetch(k->pi_pin, k->n_pi, k->mem, "pi_pin", c->stream);
    auto pi_at = fetch(k->pi_at, 4ull * k->n_pi, k->mem, "pi_at", c->stream);
    auto pi_slew = fetch(k->pi_slew, 4ull * k->n_pi, k->mem, "pi_slew", c->stream);
    auto po_pin = fetch(k->po_pin, k->n_po, k->mem, "po_pin", c->stream);
    auto po_max = fetch(k->po_out_max, 2ull * k->n_po, k->mem, "po_out_max", c->stream);
    auto po_min = fetch(k->po_out_min, 2ull * k->n_po, k->mem, "po_out_min", c->stream);
    auto po_ld = fetch(k->po_load_ff, k->n_po, k->mem, "po_load_ff", c->stream);
    std::vector<uint8_t> seen(c->P, 0);
    for (u32 i = 0; i < k->n_pi; ++i) {
      const u32 p = pi_pin[i];
      if (p >= c->P) fail(STA_ERR_ID, "pi %u: pin id %u out of range", i, p);
      if (c->pin_role[p] != STA_PIN_PI) fail(STA_ERR_ARG, "pi %u: pin %u does not have role PI", i, p);
      if (seen[p]++) fail(STA_ERR_ARG, "pi %u: pin %u listed twice", i, p);
      for (int q = 0; q < 4; ++q)
        if (!std::isfinite(pi_at[4 * i + q]) || !std::isfinite(pi_slew[4 * i + q]) || pi_slew[4 * i + q] < 0)
          fail(STA_ERR_ARG, "pi %u: non-finite arrival or bad slew", i);
    }
    std::fill(seen.begin(), seen.end(), 0);
    for (u32 i = 0; i < k->n_po; ++i) {
      const u32 p = po_pin[i];
      if (p >= c->P) fail(STA_ERR_ID, "po %u: pin id %u out of range", i, p);
      if (c->pin_role[p] != STA_PIN_PO) fail(STA_ERR_ARG, "po %u: pin %u does not have role PO", i, p);
      if (seen[p]++) fail(STA_ERR_ARG, "po %u: pin %u listed twice", i, p);
      if (!std::isfinite(po_max[2 * i]) || !std::isfinite(po_max[2 * i + 1]) || !std::isfinite(po_min[2 * i]) ||
          !std::isfinite(po_min[2 * i + 1]) || !(po_ld[i] >= 0.f) || !std::isfinite(po_ld[i]))
        fail(STA_ERR_ARG, "po %u: non-finite output delay or bad load", i);
    }
    c->period = k->period_ps;
    c->clock_slew = k->clock_slew_ps;
    c->pi_pin = std::move(pi_pin);
    c->pi_at = std::move(pi_at);
    c->pi_slew = std::move(pi_slew);
    c->po_pin = std::move(po_pin);
    c->po_out_max = std::move(po_max);
    c->po_out_min = std::move(po_min);
    c->po_load = std::move(po_ld);
    c->has_cons = true;
    c->prepared = false;
  });
}

sta_status sta_update_timing(sta_ctx c) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_update_timing");
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_update_timing before sta_load_graph");
    if (!c->has_tree) fail(STA_ERR_ORDER, "sta_update_timing before sta_set_rc_tree");
    if (!c->has_cons) fail(STA_ERR_ORDER, "sta_update_timing before sta_set_constraints");
    for (u32 k = 0; k < c->K; ++k) {
      if (!c->corners[k].lib) fail(STA_ERR_ORDER, "corner %u: no library", k);
      if (!c->corners[k].rcv) fail(STA_ERR_ORDER, "corner %u: no RC values", k);
    }
    prepare(c);
    enqueue_update(c);
  });
}

sta_status sta_synchronize(sta_ctx c) {
  return guard(c, [&] {
    ck(cudaStreamSynchronize(c->stream), "sync");
    check_flags(c);
  });
}

sta_status sta_report_slack(sta_ctx c, uint32_t corner, double* res4, float* pin_slack, sta_mem mem) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_report_slack");
    CornerState& cs = corner_of(c, corner);
    require_updated(c);
    if (res4) {
      deliver(c, res4, cs.dev.res, 4, mem);
      if (mem == STA_MEM_HOST) check_flags(c);
    }
    deliver_pins(c, pin_slack, cs.dev, 3, mem);
  });
}

sta_status sta_get_timing(sta_ctx c, uint32_t corner, float* at, float* slew, float* rat, sta_mem mem) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_get_timing");
    CornerState& cs = corner_of(c, corner);
    require_updated(c);
    deliver_pins(c, at, cs.dev, 0, mem);
    deliver_pins(c, slew, cs.dev, 1, mem);
    deliver_pins(c, rat, cs.dev, 2, mem);
  });
}

sta_status sta_get_rc(sta_ctx c, uint32_t corner, float* net_load, float* pin_elm, sta_mem mem) {
  return guard(c, [&] {
    CornerState& cs = corner_of(c, corner);
    require_updated(c);
    float* nl = net_load;
    float* pe = pin_elm;
    if (mem == STA_MEM_HOST) {
      c->tmp_arena.release();
      nl = net_load ? c->tmp_arena.alloc<float>(c->N) : nullptr;
      pe = pin_elm ? c->tmp_arena.alloc<float>(c->P) : nullptr;
    } else if (mem != STA_MEM_DEVICE) {
      fail(STA_ERR_ARG, "bad sta_mem %d", (int)mem);
    }
    ck(sta::launch_gather_rc(c->topo, cs.dev, nl, pe, c->stream), "gather rc");
    if (mem == STA_MEM_HOST) {
      if (net_load) deliver(c, net_load, nl, c->N, STA_MEM_HOST);
      if (pin_elm) deliver(c, pin_elm, pe, c->P, STA_MEM_HOST);
    }
    ck(cudaStreamSynchronize(c->stream), "sync");
  });
}

sta_status sta_get_levels(sta_ctx c, uint32_t* level, uint32_t* perm, uint32_t* num_levels, sta_mem mem) {
  return guard(c, [&] {
    if (!c->has_graph) fail(STA_ERR_ORDER, "sta_get_levels before sta_load_graph");
    if (num_levels) *num_levels = c->num_levels;
    auto put = [&](uint32_t* dst, const std::vector<u32>& v) {
      if (!dst || v.empty()) return;
      if (mem == STA_MEM_HOST) std::memcpy(dst, v.data(), v.size() * sizeof(u32));
      else if (mem == STA_MEM_DEVICE)
        ck(cudaMemcpyAsync(dst, v.data(), v.size() * sizeof(u32), cudaMemcpyHostToDevice, c->stream), "H2D");
      else fail(STA_ERR_ARG, "bad sta_mem %d", (int)mem);
    };
    put(level, c->level);
    put(perm, c->perm);
  });
}

sta_status sta_report_paths(sta_ctx c, uint32_t corner, const sta_path_query* q, sta_path_set* out, sta_mem mem) {
  return guard(c, [&] {
    Nvtx nvtx_range("sta_report_paths");
    CornerState& cs = corner_of(c, corner);
    require_updated(c);
    if (!q || !out) fail(STA_ERR_ARG, "query / output NULL");
    if (q->mode > 1) fail(STA_ERR_ARG, "mode %u (0 setup, 1 hold)", q->mode);
    if (q->k == 0 || q->nworst == 0) fail(STA_ERR_ARG, "k and nworst must be >= 1");
    if (c->net_model != 0) fail(STA_ERR_ORDER, "the path report needs the Elmore net model");
    if (!c->exc_kind.empty() || !c->clk_period.empty())
      fail(STA_ERR_ORDER, "the path report needs one clock and no timing exceptions");
    if (mem != STA_MEM_HOST && mem != STA_MEM_DEVICE) fail(STA_ERR_ARG, "bad sta_mem %d", (int)mem);
    const u32 m = std::min(q->k, q->nworst);
    if (m > 255) fail(STA_ERR_ARG, "min(k, nworst) = %u exceeds 255", m);
    cudaStream_t s = c->stream;
    if (!c->fi_p_d) {                        // lazily: the report's static arrays
      Arena& g = c->path_arena;
      c->fi_p_d = g.upload(c->fi_p_h, s);
      c->fi_slot_d = g.upload(c->fi_slot_h, s);
      c->ep_int_d = g.upload(c->ep_int_h, s);
      c->uoi_d = g.upload(c->user_of_int, s);
    }
    // scratch kept by the ctx and grown on demand (a cudaMalloc / cudaFree
    // of the ~2 NP m lists per call cost more than the report on C3)
    PathScratch& ps = c->path_scratch;
    const bool dev = mem == STA_MEM_DEVICE;
    const u32 cp = out->cap_paths, cq = out->cap_pins;
    if (m > ps.m || (!dev && (cp > ps.cp || cq > ps.cq)) || !ps.lists) {
      ck(cudaStreamSynchronize(s), "sync");
      ps.a.release();
      ps.m = std::max(m, ps.m);
      ps.cp = std::max(dev ? 0u : cp, ps.cp);
      ps.cq = std::max(dev ? 0u : cq, ps.cq);
      const size_t nc = (size_t)c->n_ep * ps.m;
      ps.lists = ps.a.alloc<sta::PathEnt>(2ull * c->NP * ps.m);
      ps.cnt = ps.a.alloc<uint8_t>(2ull * c->NP);
      ps.key = ps.a.alloc<unsigned long long>(nc);
      ps.ref = ps.a.alloc<u32>(nc);
      ps.sub = ps.a.alloc<u32>(nc);
      ps.sl = ps.a.alloc<float>(nc);
      ps.pptr = ps.a.alloc<u32>((size_t)ps.cp + 1);
      ps.ppin = ps.a.alloc<u32>(ps.cq);
      ps.prf = ps.a.alloc<uint8_t>(ps.cq);
      ps.pat = ps.a.alloc<float>(ps.cq);
      ps.psl = ps.a.alloc<float>(ps.cp);
      ps.pep = ps.a.alloc<u32>(ps.cp);
    }
    try {
      sta::PathArgs pa{};
      pa.mode = q->mode;
      pa.m = m;
      pa.lists = ps.lists;
      pa.cnt = ps.cnt;
      pa.fi_p = c->fi_p_d;
      pa.fi_slot = c->fi_slot_d;
      pa.uoi = c->uoi_d;
      pa.ep_int = c->ep_int_d;
      pa.cand_key = ps.key;
      pa.cand_ref = ps.ref;
      pa.cand_sub = ps.sub;
      pa.cand_slack = ps.sl;
      pa.path_ptr = dev ? out->path_ptr : ps.pptr;
      pa.path_pin = dev ? out->path_pin : ps.ppin;
      pa.path_rf = dev ? out->path_rf : ps.prf;
      pa.path_at = dev ? out->path_at : ps.pat;
      pa.path_slack = dev ? out->path_slack : ps.psl;
      pa.path_ep = dev ? out->path_ep : ps.pep;
      if (!pa.path_ptr || !pa.path_pin || !pa.path_rf || !pa.path_at || !pa.path_slack || !pa.path_ep)
        fail(STA_ERR_ARG, "output arrays NULL");
      u32 np = 0, npin = 0;
      bool fits = true;
      const u32 kk = std::min(q->k, cp);
      ck(sta::run_path_report(c->topo, cs.dev, pa, c->pull_stage_ptr.data(), c->S, kk, q->slack_lt, cq, &np,
                              &npin, &fits, s), "path report kernels");
      out->n_paths = np;
      out->n_pins = npin;
      if (q->k > cp && np == cp) fail(STA_ERR_ARG, "cap_paths %u < k %u", cp, q->k);
      if (!fits) fail(STA_ERR_ARG, "cap_pins %u < %u pins of the %u paths", cq, npin, np);
      if (!dev && np) {
        ck(cudaMemcpyAsync(out->path_ptr, pa.path_ptr, 4ull * (np + 1), cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(out->path_pin, pa.path_pin, 4ull * npin, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(out->path_rf, pa.path_rf, npin, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(out->path_at, pa.path_at, 4ull * npin, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(out->path_slack, pa.path_slack, 4ull * np, cudaMemcpyDeviceToHost, s), "D2H");
        ck(cudaMemcpyAsync(out->path_ep, pa.path_ep, 4ull * np, cudaMemcpyDeviceToHost, s), "D2H");
      }
      ck(cudaStreamSynchronize(s), "sync");
    } catch (...) {
      cudaStreamSynchronize(s);
      throw;
    }
  });
}

sta_status sta_get_info(sta_ctx c, sta_info* o) {
  return guard(c, [&] {
    if (!o) fail(STA_ERR_ARG, "out NULL");
    std::memset(o, 0, sizeof *o);
    o->num_pins = c->P;
    o->num_nets = c->N;
    o->num_net_arcs = c->N ? c->net_ptr[c->N] - c->N : 0;
    o->num_cell_arcs = c->A;
    o->num_checks = c->C;
    o->num_endpoints = c->n_ep;
    o->num_levels = c->num_levels;
    o->num_stages = c->S;
    o->num_pull_pins = c->NP;
    o->num_sink_pins = c->NS;
    o->num_heavy_drivers = c->n_heavy;
    o->kernels_per_update = c->launches_per_update;
    o->lut_smem_bytes = 16u * c->smem_f4;
    uint64_t b = c->graph_arena.bytes + c->tree_arena.bytes + c->cons_arena.bytes;
    for (auto& cs : c->corners) b += cs.lib_arena.bytes + cs.rc_arena.bytes + cs.state_arena.bytes;
    o->device_bytes = b;
  });
}

sta_status sta_profile_enable(sta_ctx c, int enable) {
  return guard(c, [&] {
    c->prof = enable != 0;
    if (c->prof) std::memset(&c->profile, 0, sizeof c->profile);
  });
}

sta_status sta_profile_read(sta_ctx c, sta_profile* out) {
  return guard(c, [&] {
    if (!out) fail(STA_ERR_ARG, "out NULL");
    ck(cudaStreamSynchronize(c->stream), "sync");
    *out = c->profile;
  });
}

}  // extern "C"
