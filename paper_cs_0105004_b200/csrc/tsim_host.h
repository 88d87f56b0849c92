// tsim_host.h -- host-side state of one libtsim handle (struct ts_sim) and
// the helpers shared by the host translation units (tsim_api.cu: load,
// layout, init, step; tsim_readers.cu: state read-back, partition).
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <sys/mman.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <chrono>
#include <utility>
#include <memory>
#include <unordered_set>
#include <vector>

#include "../../include/tsim.h"
#include "tsim_internal.h"

namespace tsim {
cudaError_t set_smem_attrs(int bytes);
cudaError_t set_rows_smem(int bytes);
int occupancy_blocks(int threads, int smem);
int occupancy_rows(int threads, int smem);
}  // namespace tsim

using namespace tsim;

extern std::string g_create_err;

struct DevBuf {
  void *p = nullptr;
  size_t bytes = 0;
};

// vector allocator that leaves elements uninitialised (the multi-GB route
// arrays are filled in parallel right after allocation)
template <typename T>
struct UninitAlloc : std::allocator<T> {
  template <typename U>
  struct rebind {
    using other = UninitAlloc<U>;
  };
  UninitAlloc() = default;
  template <typename U>
  UninitAlloc(const UninitAlloc<U> &) {}
  // GB-sized arrays on transparent huge pages: first touch and release
  // (page faults / unmapping of 4 KB pages) dominate their cost otherwise
  // (measured: on for the GB-sized route slots, off below 1 GB where
  // concurrent 2 MB first-touch faults were slower than 4 KB ones)
  static constexpr size_t kHuge = (size_t)64 << 20, kHugeAlign = (size_t)2 << 20, kHugeMin = (size_t)1 << 30;
  T *allocate(size_t n) {
    const size_t b = n * sizeof(T);
    if (b < kHuge) return std::allocator<T>::allocate(n);
    const size_t r = (b + kHugeAlign - 1) & ~(kHugeAlign - 1);
    void *p = aligned_alloc(kHugeAlign, r);
    if (!p) throw std::bad_alloc();
    static const size_t thp = getenv("TSIM_THP_MIN") ? (size_t)atoll(getenv("TSIM_THP_MIN")) : kHugeMin;
    if (b >= thp) madvise(p, r, MADV_HUGEPAGE);
    return static_cast<T *>(p);
  }
  void deallocate(T *p, size_t n) {
    if (n * sizeof(T) < kHuge)
      std::allocator<T>::deallocate(p, n);
    else
      free(p);
  }
  template <typename U>
  void construct(U *p) noexcept {
    ::new (static_cast<void *>(p)) U;
  }
  template <typename U, typename... A>
  void construct(U *p, A &&...a) {
    ::new (static_cast<void *>(p)) U(std::forward<A>(a)...);
  }
};

struct ts_sim {
  ts_config cfg{};
  std::string err;
  int dev = 0;
  cudaStream_t stream = nullptr;
  // second stream: the general-tile move kernel runs beside the row kernel
  // (disjoint tiles, both after the node kernel); fork / join by events
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_lc = nullptr;  // native multi-rank step: exchange #1 may start (side stream)
  size_t dev_bytes = 0;
  std::vector<void *> allocs;
  // network (host)
  bool have_net = false, have_veh = false, inited = false;
  int32_t nn = 0, nl = 0, periodic = -1;
  std::vector<int64_t> nx, ny, len;
  std::vector<int32_t> from, to, lanes, vmax, cls, ncell, lgid;
  std::vector<int32_t> in_off, in_list, out_off, out_list, out_pos;
  std::vector<uint32_t> tt;
  int64_t nlanes = 0, lane_cells = 0;
  // vehicles (host)
  int32_t nv = 0;
  std::vector<int64_t, UninitAlloc<int64_t>> roff;
  // plans as out-slot sequences (R7): rslot[roff[f] + j] = slot of route link
  // j at its from-node (0xFF for j = 0); the link ids are not kept (a link
  // at cursor c is the walk from first_link along the slots, link_at)
  std::vector<uint8_t, UninitAlloc<uint8_t>> rslot;
  std::vector<int32_t, UninitAlloc<int32_t>> dep, entry;
  std::vector<int32_t, UninitAlloc<int32_t>> pl_vid, pl_lane, pl_cell, pl_v, pl_cur;
  std::vector<uint8_t> placed;
  std::vector<int32_t> arr0;     // arrival time of vehicles restored as arrived (-1 otherwise)
  std::vector<int32_t> text_link_id;  // link ids of a network file (ts_load_network_text)
  std::vector<int32_t, UninitAlloc<int32_t>> first_link, entry_h;  // route[0] and entry cell (kept after init)
  // domain decomposition (§4; ts_set_domain): owned cells per link
  int32_t dom_k = 1, dom_me = 0;
  std::vector<int32_t> dom_of_node;
  std::vector<int32_t> own_lo, own_hi;
  std::vector<int32_t> mirror;  // per link: first mirror strip slot of the remote half, or -1
  struct Nbr {
    int32_t dom;
    std::vector<int32_t> send_slot, recv_slot;  // strip slots, (link, lane) order
    int64_t off;                                // first Strip of this neighbour in d_send/d_recv
  };
  std::vector<Nbr> nbrs;
  int64_t n_xs = 0;  // strips per exchange (sum over neighbours)
  Strip *d_send = nullptr, *d_recv = nullptr;
  int32_t *d_send_slot = nullptr, *d_recv_slot = nullptr;
  ncclComm_t comm = nullptr;  // native exchange transport (ts_nccl_init)
  std::vector<int32_t> my_nodes;
  int32_t *d_node_ids = nullptr;
  std::vector<uint32_t> node_sig;  // per node: phase-0 signal word (R23), 0 = none
  uint32_t *d_node_sig = nullptr, *d_lane_sig = nullptr;
  bool rows_s1 = false, gen_s1 = false;  // row / general state holds S1(t) (lane change applied)
  int64_t n_pending0 = 0;
  int32_t folded_t = 0;  // stats folded into the host counters up to this time
  // layout
  std::vector<TileDesc> tiles;
  std::vector<int32_t> link_tile0, link_ntiles;
  int64_t total_cells = 0;
  int32_t nstrips = 0;
  std::vector<int32_t> halo_up, halo_dn;
  WarpLayout lay{};
  int threads = 256, blocks = 1, smem = 0;
  bool gfused = false, rfused = false, node_warp = false;
  // the periodic link as a chain of row-tile segments joined by pass-through
  // virtual nodes (row kernel instead of the warp-per-tile kernels)
  bool ring_rows = false;
  std::vector<NodeOut> ring_nodeout;
  int32_t *d_ring_next = nullptr, *d_ring_prev = nullptr, *d_row_a = nullptr;
  // general tiles (halo / long / periodic links): byte codes at device
  // offsets of their own; uploaded as d_tiles
  std::vector<TileDesc> gtiles;
  std::vector<int32_t> tile_g;  // tile -> index in gtiles, or -1
  int64_t gcells = 0;
  // row tiles (whole links of <= kRowMaxCells cells): k_rows
  std::vector<int32_t> tile_row;  // tile -> global row slot of its lane 0, or -1
  std::vector<RowDesc> rows;      // ngroups * 32 slots
  int32_t ngroups = 0;
  int64_t rvid_entries = 0;
  uint32_t *d_planes[2] = {nullptr, nullptr};
  int32_t *d_rvid[2] = {nullptr, nullptr};
  int32_t *d_gcnt[2] = {nullptr, nullptr};  // vehicles per group
  unsigned long long *d_gctr = nullptr;      // k_rows work counter
  unsigned long long gctr_base = 0;
  int32_t *d_inj_scratch = nullptr;
  RowDesc *d_rows = nullptr;
  int rows_threads = 128, rows_blocks = 1, rows_cap = 0, rows_smem = 0;
  // programmatic dependent launch of the node and move kernels (TSIM_NO_PDL
  // turns it off for comparisons)
  bool pdl = true;
  std::vector<int32_t> gvoff;                // first vid-block entry of each group
  int32_t *d_gvoff = nullptr;
  NodeLane *d_nlanes = nullptr;
  int32_t nchunks = 0;
  std::vector<int32_t> nli;   // node-lane index of every global lane id
  int64_t n_nli = 0;          // size of the node-lane indexed arrays
  int32_t *d_nli = nullptr;
  std::vector<int32_t> nlo;   // node-out-lane index of every global lane id
  int64_t n_nlo = 0;          // size of the node-out-lane indexed arrays
  int32_t *d_nlo = nullptr;
  uint64_t p32 = 0;
  // device
  TileDesc *d_tiles = nullptr;
  uint8_t *d_code[2] = {nullptr, nullptr};
  int32_t *d_vid[2] = {nullptr, nullptr};
  Strip *d_strip[2] = {nullptr, nullptr};
  int32_t *d_halo_up = nullptr, *d_halo_dn = nullptr;
  uint8_t *d_vmax = nullptr;
  uint32_t *d_tt = nullptr;
  int32_t *d_out_pos = nullptr;
  int64_t *d_roff = nullptr;   // route offsets (device read-back of cursors; allocated on demand)
  int32_t *d_rd = nullptr;     // read-back scratch (ts_read_vehicles on the device)
  // pinned double buffer of the read-back (device -> pinned by DMA, pinned ->
  // caller's arrays by the host cores), allocated at the first large read
  uint8_t *pin_rd[2] = {nullptr, nullptr};  // (the route upload's staging, kept after init)
  size_t pin_rd_bytes = 0;
  cudaEvent_t ev_rd[2] = {nullptr, nullptr};
  uint8_t *d_rslot = nullptr;
  NodeOut *d_nodeout = nullptr;
  VehPos *d_vpos = nullptr;
  int32_t *d_dep = nullptr, *d_entry = nullptr;
  int32_t *d_inj = nullptr, *d_arr = nullptr;
  int32_t *d_pend_off = nullptr, *d_pend_list = nullptr, *d_pend_head = nullptr;
  uint64_t *d_tail = nullptr, *d_entr = nullptr;
  uint8_t *d_head = nullptr, *d_ext = nullptr;
  unsigned long long *d_stats = nullptr, *d_work = nullptr, *d_hash = nullptr;
  unsigned long long *d_node_work = nullptr;  // per node (TS_FLAG_LINK_WORK)
  int32_t *d_nl_node = nullptr;               // node id per node-lane index
  int32_t *d_nl_row = nullptr;                // row slot per node-lane index (or -1)
  int32_t *d_lane_row = nullptr;              // row slot per global lane id (or -1)
  uint8_t *d_ext_row = nullptr;               // node grants by row slot
  uint64_t *d_entr_row = nullptr;             // entrant records by row slot
  std::vector<int32_t> lane_row0;             // per link: row slot of its lane 0 (or -1)
  int32_t *d_in_off = nullptr, *d_in_list = nullptr, *d_out_off = nullptr, *d_out_list = nullptr;
  int32_t *d_ncell = nullptr, *d_lanes = nullptr, *d_lgid = nullptr, *d_cls = nullptr;
  int gcur = 0, rcur = 0;  // current buffer of the general / row state
  int32_t t = 0;
  int64_t veh_updates = 0, arrived = 0, injected = 0, n_placed = 0, n_arrived0 = 0;
  // timing
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // CUDA-graph replay of kGraphSteps steps (TS_FLAG_GRAPH): the kernels read
  // the step time from the device clock d_clock; while capturing, step and
  // node parameters carry t - graph_t0 and tdev = d_clock
  int32_t *d_clock = nullptr;
  // one graph per parity of the double buffers (rcur, gcur) at its start
  cudaGraphExec_t graph_exec[4] = {nullptr, nullptr, nullptr, nullptr};
  unsigned long long graph_gctr_end[4] = {0, 0, 0, 0};
  bool graph_off = false, capturing = false;
  int32_t graph_t0 = 0;
  std::vector<cudaEvent_t> mv_ev;
  double last_total_ms = 0, last_move_ms = 0, last_xchg_ms = 0;
  int64_t last_xchg_n = 0;  // exchanges timed in the last native ts_step call
  // device time of all step work since the last ts_busy_time (the measured
  // per-domain step time of the rebalancing feedback)
  double busy_ms = 0;
  std::vector<cudaEvent_t> ph_ev;  // event pairs around ts_step_phase calls
  size_t ph_used = 0;
  int64_t last_move_launches = 0;
  bool timing = true;
  // ts_step_async / ts_sync: the steps enqueued and not yet finished
  int32_t async_from = 0, async_n = 0;
  double async_ms = 0, async_move_ms = 0;  // timing of the leading blocks of a long async run
  int64_t async_move_launches = 0;
  // ts_local_step on one device: strips delivered by one direct kernel per
  // exchange (no pack / copy / unpack of this handle while set)
  bool direct = false;
  bool no_xoverlap = false;  // TSIM_NO_XOVERLAP: exchange #1 in stream order (A/B, tests)
  // ts_exchange_local: reusable ordering events (after the pack, after the copies)
  cudaEvent_t ev_packed = nullptr, ev_copied = nullptr;
};

// shared by the step (tsim_api.cu) and the readers (tsim_readers.cu);
// fail(): the error message of the handle (or of ts_create) and the code
// (library-internal: not exported from libtsim.so)
#define TS_INTERNAL __attribute__((visibility("hidden")))
extern "C" {
TS_INTERNAL StepParams step_params(ts_sim *h, int t, int mode);
TS_INTERNAL RowsParams rows_params(ts_sim *h);
TS_INTERNAL int fold_stats(ts_sim *h);
TS_INTERNAL int fail(ts_sim *h, int code, const char *fmt, ...);
}


#define CK(h, call)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return fail((h), TS_EINTERNAL, "%s failed: %s (%s:%d)", #call,                    \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                          \
  } while (0)

template <class T>
static int dalloc(ts_sim *h, T **p, size_t n, int fill = -1) {
  size_t bytes = std::max<size_t>(n, 1) * sizeof(T);
  cudaError_t e = cudaMalloc((void **)p, bytes);
  if (e != cudaSuccess)
    return fail(h, TS_EINTERNAL, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
  h->allocs.push_back(*p);
  h->dev_bytes += bytes;
  if (fill >= 0) {
    e = cudaMemsetAsync(*p, fill, bytes, h->stream);
    if (e != cudaSuccess) return fail(h, TS_EINTERNAL, "memset: %s", cudaGetErrorString(e));
  }
  return TS_OK;
}

template <class T, class A>
static int upload(ts_sim *h, T **p, const std::vector<T, A> &v) {
  int rc = dalloc(h, p, v.size());
  if (rc) return rc;
  if (!v.empty())
    CK(h, cudaMemcpyAsync(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, h->stream));
  return TS_OK;
}

// TSIM_TRACE=1: wall-clock phases of ts_init on stderr (host-side tuning)
struct InitTrace {
  const char *what = "init";
  bool on = getenv("TSIM_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  InitTrace() = default;
  explicit InitTrace(const char *w) : what(w) {}
  void operator()(const char *phase) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    fprintf(stderr, "[tsim %s] %-28s %8.3f s\n", what, phase, std::chrono::duration<double>(n - t).count());
    t = n;
  }
};

// parallel loop over [0, n) in contiguous chunks on the host cores (load
// and init handle billions of route entries at the largest configs).  The
// chunks (16 per thread) are handed out dynamically: a thread delayed by
// the library's own copy threads or another process does not hold up the
// loop.  f(lo, hi, t) is called once per chunk, chunks of one thread t in
// increasing order.
template <typename F>
static void parallel_for(int64_t n, F f) {
  // host threads: min(cores, 32) (TSIM_THREADS overrides, at most 64: the
  // per-thread result arrays of the callers hold 64 entries)
  static const int nt = []() {
    const char *e = getenv("TSIM_THREADS");
    const int cap = e ? std::max(1, std::min(64, atoi(e))) : 32;
    return (int)std::max(1u, std::min((unsigned)cap, std::thread::hardware_concurrency()));
  }();
  if (n < (int64_t)1 << 16 || nt == 1) {
    f((int64_t)0, n, 0);
    return;
  }
  if (getenv("TSIM_STATIC_CHUNKS")) {  // one contiguous range per thread (A/B timing)
    std::vector<std::thread> th;
    for (int i = 0; i < nt; i++)
      th.emplace_back([=, &f]() { f(n * i / nt, n * (i + 1) / nt, i); });
    for (auto &t : th) t.join();
    return;
  }
  const int64_t chunks = std::min<int64_t>(n, (int64_t)nt * 16);
  std::atomic<int64_t> next{0};
  std::vector<std::thread> th;
  for (int i = 0; i < nt; i++)
    th.emplace_back([=, &f, &next]() {
      for (int64_t c; (c = next.fetch_add(1, std::memory_order_relaxed)) < chunks;)
        f(n * c / chunks, n * (c + 1) / chunks, i);
    });
  for (auto &t : th) t.join();
}

// a host staging array of n copies of v, first-touched by the host cores
// in parallel (value-initialising GB-sized vectors serially dominates init)
template <typename T>
using HostVec = std::vector<T, UninitAlloc<T>>;
template <typename T>
static HostVec<T> filled(size_t n, T v) {
  HostVec<T> a(n);
  parallel_for((int64_t)n, [&](int64_t lo, int64_t hi, int) { std::fill(a.data() + lo, a.data() + hi, v); });
  return a;
}

// the link at cursor c of vehicle f: the walk along its out-slots
static inline int link_at(const ts_sim *h, int f, int c) {
  const int64_t a = h->roff[f];
  int k = h->first_link[f];
  for (int j = 1; j <= c; j++) k = h->out_list[h->out_off[h->to[k]] + h->rslot[a + j]];
  return k;
}
