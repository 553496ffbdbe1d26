// sta_internal.h -- device data layout shared by the host engine (sta_api.cpp)
// and the sm_100a kernels (sta_kernels.cu).  See DESIGN.md §5 for the layout.
//
// Internal pin numbering (built once by sta_load_graph):
//   * "pull pins" -- pins without a net arc into them (cell outputs, sources):
//     internal ids [0, NP), sorted by (gate stage, user id).  A pull pin is
//     evaluated by pulling over its cell-arc fan-in.
//   * "sinks" -- net sinks (exactly one fan-in: the net arc): internal ids
//     [NP, P), grouped by driver in driver order, in net order.  A sink is a
//     pure function of its driver (AT + Elmore, PERI slew), so it needs no
//     step of its own: the forward kernel of the stage after its driver's
//     materializes it, and consumers recompute it inline (pull-through).
//   Gate stage: 0 for pins without fan-in, else 1 + max over cell fan-in
//   (u -> v) of stage(driver(u)) (stage(u) if u is itself a pull pin).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sta {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kSeedClock = 0xFFFFFFFEu;   // stage-0 seed: ideal clock pin
constexpr int kSmallNet = 48;                  // RC nodes handled by one thread
constexpr int kHeavyFanout = 32;               // backward: sinks above -> block per driver

// fan-in / fan-out arc info word: sense (3 bits) | first table id << 3
__host__ __device__ inline uint32_t pack_info(uint32_t sense, uint32_t tab) { return sense | (tab << 3); }

// table descriptor: data offset (26 bits) | (n1-1) << 26 | (n2-1) << 29
__host__ __device__ inline uint32_t pack_tdesc(uint32_t off, uint32_t n1, uint32_t n2) {
  return off | ((n1 - 1u) << 26) | ((n2 - 1u) << 29);
}

struct EpRec {          // one timing endpoint
  uint32_t po;          // index into the PO constraint arrays or kNone
  uint32_t chk_tab;     // first of (setup_r, setup_f, hold_r, hold_f) or kNone
};

// Topology shared by all corners (device pointers).
struct Topo {
  uint32_t P, NP, NS, S, N, n_ep, n_pi, n_po;
  // forward
  const uint32_t* fi_ptr;    // [NP+1]
  const uint32_t* fi_src;    // record to read (driver of u, or u if u is a pull pin)
  const uint32_t* fi_hop;    // sink index of u (net hop to apply) or kNone
  const uint32_t* fi_info;
  const uint32_t* sink_ptr;  // [NP+1] sinks of each pull pin (sink index space)
  const uint32_t* sink_drv;  // [NS]
  const uint32_t* seed;      // [pins of stage 0]: PI index, kSeedClock or kNone
  // backward
  const uint32_t* sfo_ptr;   // [NS+1] cell fan-out of each sink
  const uint32_t* sfo_dst;   // pull pin
  const uint32_t* sfo_info;
  const uint32_t* pfo_ptr;   // [NP+1] cell fan-out of each pull pin
  const uint32_t* pfo_dst;
  const uint32_t* pfo_info;
  const uint32_t* pin_ep;    // [P] internal id -> endpoint index or kNone
  const EpRec* ep;           // [n_ep]
  const uint32_t* heavy;     // heavy drivers, grouped by stage
  // constraints
  const float4* pi_at;       // [n_pi]
  const float4* pi_slew;
  const float2* po_out_max;  // [n_po]
  const float2* po_out_min;
  float period, clock_slew;
  // RC (nets in driver order j = 0..N-1)
  const uint32_t* net_drv;   // [N] internal pull id of the driver
  const uint32_t* net_rc;    // [N+1] user RC node offsets in driver order (begin)
  const uint32_t* net_rcn;   // [N] node count
  const float* net_lumped;   // [N] lumped load (nets without RC nodes)
  const int32_t* rc_parent;  // [n_rc] user node order, local parent
  const uint32_t* rc_sink;   // [n_rc] sink index of the node's pin or kNone
  const float* rc_scap;      // [n_rc] pin cap + PO load at the node
  // big-net schedule (block per net)
  uint32_t n_big;
  const uint32_t* big_net;     // [n_big] net index j (driver order)
  const uint32_t* big_scr;     // [n_big+1] prefix of node counts: scratch offset of net b
  const uint32_t* big_hptr_off;// [n_big+1] range of net b in big_hptr
  const uint32_t* big_hptr;    // height-level boundaries, absolute into big_hnode
  const uint32_t* big_hnode;   // local node ids grouped by height (leaves first)
  const uint32_t* big_dptr_off;// [n_big+1] range of net b in big_dptr
  const uint32_t* big_dptr;    // depth-level boundaries, absolute into big_dnode
  const uint32_t* big_dnode;   // local node ids grouped by depth (depth >= 1)
  const uint32_t* big_cptr;    // children CSR: net b node i at big_scr[b] + b + i, absolute
  const uint32_t* big_child;   // child local ids, decreasing within a parent
  // outputs to user order
  const uint32_t* int_of_user; // [P]
};

// Per-corner device state.
struct CornerDev {
  float4* rec;        // [2P]: at, slew per pin (internal order)
  float4* rat;        // [P]
  float4* slack;      // [P]
  float* elm;         // [NS] Elmore delay of each sink's net arc
  float* load;        // [NP] NLDM load seen by each pull pin (0 if no net)
  float2* ep_ws;      // [n_ep] worst setup / hold slack per endpoint
  double* res;        // [4]
  const float* lut;   // table pool
  const uint32_t* tdesc;
  const float* rc_res;  // [n_rc] user node order (owned or borrowed)
  const float* rc_cap;
  double* scratch;    // big-net scratch: cd then elm
  uint32_t* err_flag; // nonzero: bad RC value seen
};

// ---- launchers (sta_kernels.cu); all enqueue on `s`, return cudaGetLastError()
struct StagePlan {
  // host-side per-stage ranges
  const uint32_t* pull_stage_ptr;  // [S+1] (host)
  const uint32_t* sink_stage_ptr;  // [S+1] sink ranges of the drivers of each stage (host)
  const uint32_t* heavy_stage_ptr; // [S+1] (host)
};

cudaError_t launch_rc(const Topo& t, const CornerDev& c, uint32_t n_small_blocks, cudaStream_t s);
cudaError_t launch_seed(const Topo& t, const CornerDev& c, uint32_t n0, cudaStream_t s);
cudaError_t launch_fwd_stage(const Topo& t, const CornerDev& c, uint32_t sinkA0, uint32_t nA,
                             uint32_t pullB0, uint32_t nB, cudaStream_t s);
cudaError_t launch_bwd_stage(const Topo& t, const CornerDev& c, uint32_t pull0, uint32_t nPull,
                             uint32_t heavy0, uint32_t nHeavy, cudaStream_t s);
cudaError_t launch_reduce(const Topo& t, const CornerDev& c, cudaStream_t s);
cudaError_t launch_gather4(const float4* src, const uint32_t* idx, float4* dst, uint32_t n,
                           uint32_t stride_f4, cudaStream_t s);
cudaError_t launch_gather_rc(const Topo& t, const CornerDev& c, float* net_load, float* pin_elm,
                             const uint32_t* net_of_j, const uint32_t* user_of_int, cudaStream_t s);
cudaError_t launch_check_rc_values(const CornerDev& c, uint32_t n_rc, cudaStream_t s);

}  // namespace sta
