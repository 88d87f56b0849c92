// tsim_api.cu -- host side of libtsim: input validation, network tables,
// tiling and device layout, initial state, kernel orchestration, the
// exchange transport (state read-back: tsim_readers.cu; handle state and
// shared helpers: tsim_host.h).  C-ABI declared in include/tsim.h.
#include "tsim_host.h"

std::string g_create_err;

int fail(ts_sim *h, int code, const char *fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  else g_create_err = buf;
  return code;
}

// ---------------------------------------------------------------- NCCL
// The strip exchanges of domain mode (H2/H7) can run inside the library over
// NCCL point-to-point (NVLink between the GPUs of one node), so ts_step(n)
// runs whole steps with neighbours and no host round trip per exchange.
// libnccl is opened at run time (the one torch already loaded, else the
// system's): single-GPU use needs no NCCL.
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char *(*errorString)(ncclResult_t) = nullptr;
};

static NcclApi &nccl() {
  static NcclApi a;
  if (a.tried) return a;
  a.tried = true;
  // TSIM_NCCL_LIB: another library with the same entry points (the tests'
  // in-process stand-in, tests/fake_nccl.cpp: several ranks on one GPU)
  const char *alt = getenv("TSIM_NCCL_LIB");
  void *lib = alt ? dlopen(alt, RTLD_NOW | RTLD_LOCAL) : nullptr;
  if (!lib && !alt) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!lib && !alt) lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!lib && !alt) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!lib) return a;
  a.getUniqueId = (decltype(a.getUniqueId))dlsym(lib, "ncclGetUniqueId");
  a.commInitRank = (decltype(a.commInitRank))dlsym(lib, "ncclCommInitRank");
  a.commDestroy = (decltype(a.commDestroy))dlsym(lib, "ncclCommDestroy");
  a.groupStart = (decltype(a.groupStart))dlsym(lib, "ncclGroupStart");
  a.groupEnd = (decltype(a.groupEnd))dlsym(lib, "ncclGroupEnd");
  a.send = (decltype(a.send))dlsym(lib, "ncclSend");
  a.recv = (decltype(a.recv))dlsym(lib, "ncclRecv");
  a.errorString = (decltype(a.errorString))dlsym(lib, "ncclGetErrorString");
  a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.groupStart && a.groupEnd &&
         a.send && a.recv && a.errorString;
  return a;
}

#define NCK(h, x)                                                                       \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess)                                                               \
      return fail(h, TS_EINTERNAL, "%s failed: %s", #x, nccl().errorString(r_));         \
  } while (0)

// one exchange: the packed strips to and from every neighbour domain, one
// message each way per neighbour, on the handle's stream
static int nccl_exchange(ts_sim *h, cudaStream_t st = nullptr) {
  if (h->nbrs.empty()) return TS_OK;
  if (!st) st = h->stream;
  NcclApi &a = nccl();
  NCK(h, a.groupStart());
  for (const ts_sim::Nbr &nb : h->nbrs) {
    // send and receive segments have the same size by construction (one
    // strip per lane of every shared split link, both sides in link order;
    // checked in build_tiles)
    NCK(h, a.send(h->d_send + nb.off, nb.send_slot.size() * sizeof(Strip), ncclUint8, nb.dom,
                  h->comm, st));
    NCK(h, a.recv(h->d_recv + nb.off, nb.recv_slot.size() * sizeof(Strip), ncclUint8, nb.dom,
                  h->comm, st));
  }
  NCK(h, a.groupEnd());
  return TS_OK;
}

extern "C" {

int ts_nccl_unique_id(void *id128) {
  if (!id128) return TS_EINVAL;
  NcclApi &a = nccl();
  if (!a.ok) return TS_EINTERNAL;
  ncclUniqueId id;
  if (a.getUniqueId(&id) != ncclSuccess) return TS_EINTERNAL;
  memcpy(id128, &id, sizeof(id));
  return TS_OK;
}

int ts_nccl_init(ts_sim *h, const void *id128, int32_t nranks, int32_t rank) {
  if (!h || !id128) return TS_EINVAL;
  if (!h->inited) return fail(h, TS_EINVAL, "call ts_init first");
  if (h->comm) return fail(h, TS_EINVAL, "communicator already set");
  if (nranks != h->dom_k || rank != h->dom_me)
    return fail(h, TS_EINVAL, "ranks must be the domains: nranks %d != k %d or rank %d != domain %d",
                nranks, h->dom_k, rank, h->dom_me);
  NcclApi &a = nccl();
  if (!a.ok) return fail(h, TS_EINTERNAL, "libnccl.so.2 not found");
  CK(h, cudaSetDevice(h->dev));
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  NCK(h, a.commInitRank(&h->comm, nranks, id, rank));
  return TS_OK;
}

int ts_exchange(ts_sim *h) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "call ts_init first");
  if (!h->comm) return fail(h, TS_EINVAL, "no communicator (ts_nccl_init)");
  CK(h, cudaSetDevice(h->dev));
  return nccl_exchange(h);
}

int ts_create(const ts_config *cfg, ts_sim **out) {
  if (!out) return fail(nullptr, TS_EINVAL, "out is NULL");
  *out = nullptr;
  if (!cfg) return fail(nullptr, TS_EINVAL, "cfg is NULL");
  if (!(cfg->p_slow >= 0.0 && cfg->p_slow <= 1.0)) return fail(nullptr, TS_EINVAL, "p_slow not in [0,1]");
  if (cfg->gap_accept_G < 0 || cfg->gap_accept_G > kGmax)
    return fail(nullptr, TS_EINVAL, "gap_accept_G must be in [0, 5]");
  if (cfg->desperation_D < 1 || cfg->desperation_D > 4096)
    return fail(nullptr, TS_EINVAL, "desperation_D must be in [1, 4096]");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(nullptr, TS_EINTERNAL, "no CUDA device: %s", cudaGetErrorString(e));
  if (cfg->device < 0 || cfg->device >= ndev) return fail(nullptr, TS_EINVAL, "bad device ordinal");
  ts_sim *h = new ts_sim();
  h->cfg = *cfg;
  h->dev = cfg->device;
  e = cudaSetDevice(h->dev);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev0);
  if (e == cudaSuccess) e = cudaEventCreate(&h->ev1);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_lc, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_packed, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_copied, cudaEventDisableTiming);
  if (e != cudaSuccess) {
    delete h;
    return fail(nullptr, TS_EINTERNAL, "CUDA init failed: %s", cudaGetErrorString(e));
  }
  // floor(p * 2^32), exact for the power-of-two scaling (R3)
  h->p32 = (uint64_t)(cfg->p_slow * 4294967296.0);
  *out = h;
  return TS_OK;
}

static void drop_local_graphs(const ts_sim *h);

static void drop_direct_plans(const ts_sim *h);

void ts_destroy(ts_sim *h) {
  if (!h) return;
  drop_local_graphs(h);
  drop_direct_plans(h);
  cudaSetDevice(h->dev);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void *p : h->allocs) cudaFree(p);
  for (auto e : h->mv_ev) cudaEventDestroy(e);
  for (auto e : h->ph_ev) cudaEventDestroy(e);
  if (h->comm) nccl().commDestroy(h->comm);
  for (auto g : h->graph_exec)
    if (g) cudaGraphExecDestroy(g);
  if (h->ev0) cudaEventDestroy(h->ev0);
  if (h->ev1) cudaEventDestroy(h->ev1);
  if (h->stream) cudaStreamDestroy(h->stream);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ev_lc) cudaEventDestroy(h->ev_lc);
  if (h->ev_packed) cudaEventDestroy(h->ev_packed);
  if (h->ev_copied) cudaEventDestroy(h->ev_copied);
  for (int i = 0; i < 2; i++) {
    if (h->pin_rd[i]) cudaFreeHost(h->pin_rd[i]);
    if (h->ev_rd[i]) cudaEventDestroy(h->ev_rd[i]);
  }
  delete h;
}

const char *ts_last_error(const ts_sim *h) { return h ? h->err.c_str() : g_create_err.c_str(); }

// ------------------------------------------------------------------ network
// reading R7: turn type from integer direction vectors; 0 T, 1 L, 2 R
static int turn_type(const ts_sim *h, int k, int k2) {
  const int64_t ax = h->nx[h->to[k]] - h->nx[h->from[k]], ay = h->ny[h->to[k]] - h->ny[h->from[k]];
  const int64_t bx = h->nx[h->to[k2]] - h->nx[h->from[k2]],
                by = h->ny[h->to[k2]] - h->ny[h->from[k2]];
  const int64_t cross = ax * by - ay * bx, dot = ax * bx + ay * by;
  if (dot > 0 && (cross < 0 ? -cross : cross) <= dot) return 0;
  if (cross < 0) return 2;
  return 1;  // left, or U-turn
}

int ts_load_network(ts_sim *h, int32_t n_nodes, const int64_t *node_x_mm, const int64_t *node_y_mm,
                    int32_t n_links, const int32_t *from, const int32_t *to,
                    const int64_t *length_mm, const int32_t *lanes, const int32_t *vmax,
                    const int32_t *prio_class, int32_t periodic_link) {
  if (!h) return TS_EINVAL;
  if (h->have_net) return fail(h, TS_EINVAL, "network already loaded");
  if (n_nodes < 1 || n_links < 1) return fail(h, TS_EINVAL, "empty network");
  if (periodic_link >= 0 && n_links != 1)
    return fail(h, TS_EINVAL, "a periodic link must be the only link");
  h->nn = n_nodes;
  h->nl = n_links;
  h->periodic = periodic_link;
  h->nx.assign(node_x_mm, node_x_mm + n_nodes);
  h->ny.assign(node_y_mm, node_y_mm + n_nodes);
  h->from.assign(from, from + n_links);
  h->to.assign(to, to + n_links);
  h->len.assign(length_mm, length_mm + n_links);
  h->lanes.assign(lanes, lanes + n_links);
  h->vmax.assign(vmax, vmax + n_links);
  h->cls.assign(prio_class, prio_class + n_links);
  h->ncell.resize(n_links);
  h->lgid.resize(n_links + 1);
  h->lgid[0] = 0;
  for (int k = 0; k < n_links; k++) {
    if (from[k] < 0 || from[k] >= n_nodes || to[k] < 0 || to[k] >= n_nodes)
      return fail(h, TS_EINVAL, "link %d: dangling node reference", k);
    if (from[k] == to[k] && k != periodic_link) return fail(h, TS_EINVAL, "link %d: from == to", k);
    if (length_mm[k] <= 0) return fail(h, TS_EINVAL, "link %d: non-positive length", k);
    if (lanes[k] < 1 || lanes[k] > kMaxLanes) return fail(h, TS_EINVAL, "link %d: lanes", k);
    if (vmax[k] < 1 || vmax[k] > kGmax) return fail(h, TS_EINVAL, "link %d: vmax", k);
    // R1: round-half-up(length / 7.5 m) in integer mm, at least 1
    int64_t n = std::max<int64_t>(1, (length_mm[k] + 3750) / 7500);
    if (n < 10) return fail(h, TS_EINVAL, "link %d: %lld cells < 10 (R11)", k, (long long)n);
    if (n > 100000000) return fail(h, TS_EINVAL, "link %d: too long", k);
    h->ncell[k] = (int32_t)n;
    h->lgid[k + 1] = h->lgid[k] + lanes[k];
    h->lane_cells += n * lanes[k];
  }
  h->nlanes = h->lgid[n_links];
  // incoming / outgoing links per node in ascending link id
  h->in_off.assign(n_nodes + 1, 0);
  h->out_off.assign(n_nodes + 1, 0);
  for (int k = 0; k < n_links; k++) {
    if (k == periodic_link) continue;
    h->in_off[to[k] + 1]++;
    h->out_off[from[k] + 1]++;
  }
  for (int i = 0; i < n_nodes; i++) {
    if (h->out_off[i + 1] > 15) return fail(h, TS_EINVAL, "node %d: out-degree > 15", i);
    h->in_off[i + 1] += h->in_off[i];
    h->out_off[i + 1] += h->out_off[i];
  }
  h->in_list.assign(std::max(1, h->in_off[n_nodes]), 0);
  h->out_list.assign(std::max(1, h->out_off[n_nodes]), 0);
  h->out_pos.assign(n_links, 0);
  std::vector<int32_t> fi(n_nodes, 0), fo(n_nodes, 0);
  for (int k = 0; k < n_links; k++) {
    if (k == periodic_link) continue;
    h->in_list[h->in_off[to[k]] + fi[to[k]]++] = k;
    h->out_pos[k] = fo[from[k]];
    h->out_list[h->out_off[from[k]] + fo[from[k]]++] = k;
  }
  h->tt.assign(n_links, 0u);
  for (int k = 0; k < n_links; k++) {
    if (k == periodic_link) continue;
    const int nd = to[k];
    for (int s = 0; s < h->out_off[nd + 1] - h->out_off[nd]; s++)
      h->tt[k] |= (uint32_t)turn_type(h, k, h->out_list[h->out_off[nd] + s]) << (2 * s);
  }
  h->have_net = true;
  return TS_OK;
}

int32_t ts_link_cells(const ts_sim *h, int32_t link) {
  if (!h || !h->have_net || link < 0 || link >= h->nl) return -1;
  return h->ncell[link];
}

int ts_load_vehicles(ts_sim *h, int32_t n, const int64_t *route_off, const int32_t *route_links,
                     const int32_t *depart, const int32_t *entry_cell) {
  if (!h) return TS_EINVAL;
  if (!h->have_net) return fail(h, TS_EINVAL, "load the network first");
  if (h->have_veh) return fail(h, TS_EINVAL, "vehicles already loaded");
  if (n < 0) return fail(h, TS_EINVAL, "negative vehicle count");
  if (n > 0 && route_off[0] != 0) return fail(h, TS_EINVAL, "route_off[0] != 0");
  // validation in parallel over vehicles, fused with the conversion of the
  // routes to out-slot sequences (one pass over the route links): error code
  // of vehicle i (0 = ok); the first failing vehicle is reported.  Empty or
  // decreasing route offsets are found first (they size the slot array).
  // per link (from, to, out-slot at its from node) in one 16-byte record:
  // one gather per route entry; raw pointers in locals (the byte stores
  // into the slot array would otherwise force reloads through h)
  struct LinkRec {
    int32_t from, to, slot, pad;
  };
  std::vector<LinkRec> lrec(h->nl);
  for (int k = 0; k < h->nl; k++) lrec[k] = LinkRec{h->from[k], h->to[k], h->out_pos[k], 0};
  const LinkRec *lr = lrec.data();
  const uint32_t nl = (uint32_t)h->nl;
  const int32_t *ncell = h->ncell.data();
  auto check = [&, lr, nl, ncell](int32_t i, uint8_t *slot) -> int {
    const int64_t a = route_off[i], b = route_off[i + 1];
    if (b <= a) return 1;
    const int32_t k0 = route_links[a];
    if ((uint32_t)k0 >= nl) return 2;
    if (slot) slot[a] = 0xFF;
    int32_t at = lr[k0].to;
    for (int64_t j = a + 1; j < b; j++) {
      const int32_t k = route_links[j];
      if ((uint32_t)k >= nl) return 2;
      const LinkRec r = lr[k];
      if (r.from != at) return 3;
      if (slot) slot[j] = (uint8_t)r.slot;
      at = r.to;
    }
    if (entry_cell[i] < 0 || entry_cell[i] >= ncell[k0]) return 4;
    return 0;
  };
  auto first_failing = [&](auto pred) {
    std::vector<int32_t> first_bad(64, INT32_MAX);
    parallel_for(n, [&](int64_t lo, int64_t hi, int t) {
      for (int64_t i = lo; i < hi; i++)
        if (pred((int32_t)i)) {  // (this thread's chunks come in increasing order)
          first_bad[t] = std::min(first_bad[t], (int32_t)i);
          return;
        }
    });
    return *std::min_element(first_bad.begin(), first_bad.end());
  };
  static const char *msg[] = {"", "empty route", "bad link", "route links not consecutive",
                              "entry cell outside link"};
  InitTrace trace("load");
  const int32_t bad_off = first_failing([&](int32_t i) { return route_off[i + 1] <= route_off[i]; });
  if (bad_off != INT32_MAX) return fail(h, TS_EINVAL, "vehicle %d: %s", bad_off, msg[1]);
  trace("offsets");
  h->rslot.resize(n > 0 ? route_off[n] : 0);
  uint8_t *const slot = h->rslot.data();
  // the conversion pass: 8-byte records (from, to | slot << 24) and no
  // branch per route entry (errors accumulate per vehicle; the first
  // failing vehicle is then classified by check); networks with >= 2^24
  // nodes take check itself
  const bool packed = h->nn < (1 << 24) && getenv("TSIM_LOAD_CHECKED") == nullptr;
  std::vector<uint64_t> prec(packed ? h->nl : 0);
  for (int k = 0; k < (packed ? h->nl : 0); k++)
    prec[k] = (uint64_t)(uint32_t)h->from[k] | ((uint64_t)((uint32_t)h->to[k] | ((uint32_t)h->out_pos[k] << 24)) << 32);
  const uint64_t *pr = prec.data();
  auto convert = [&, pr, nl, ncell](int32_t i) -> bool {  // true: vehicle i fails
    const int64_t a = route_off[i], b = route_off[i + 1];
    const uint32_t k0 = (uint32_t)route_links[a];
    if (k0 >= nl) return true;
    slot[a] = 0xFF;
    uint32_t at = (uint32_t)(pr[k0] >> 32) & 0xFFFFFFu, bad = 0u;
    for (int64_t j = a + 1; j < b; j++) {
      const uint32_t k = (uint32_t)route_links[j];
      bad |= k >= nl ? 1u : 0u;
      const uint64_t r = pr[k < nl ? k : 0u];
      bad |= (uint32_t)r != at ? 1u : 0u;
      const uint32_t hi = (uint32_t)(r >> 32);
      slot[j] = (uint8_t)(hi >> 24);
      at = hi & 0xFFFFFFu;
    }
    return bad != 0u || entry_cell[i] < 0 || entry_cell[i] >= ncell[k0];
  };
  const int32_t bad = packed ? first_failing(convert)
                             : first_failing([&](int32_t i) { return check(i, slot) != 0; });
  if (bad != INT32_MAX) {
    decltype(h->rslot)().swap(h->rslot);
    return fail(h, TS_EINVAL, "vehicle %d: %s", bad, msg[check(bad, nullptr)]);
  }
  trace("routes -> out-slots");
  h->nv = n;
  h->roff.resize(n + 1);
  h->roff[0] = 0;
  h->first_link.resize(n);
  h->dep.resize(n);
  h->entry.resize(n);
  parallel_for(n, [&](int64_t lo, int64_t hi, int) {
    for (int64_t f = lo; f < hi; f++) {
      h->roff[f + 1] = route_off[f + 1];
      h->first_link[f] = route_links[route_off[f]];
      h->dep[f] = depart[f];
      h->entry[f] = entry_cell[f];
    }
  });
  h->placed.assign(n, 0);
  h->have_veh = true;
  trace("vehicle arrays");
  return TS_OK;
}

int ts_place_vehicles_at(ts_sim *h, int32_t n, const int32_t *vid, const int32_t *cursor,
                         const int32_t *lane, const int32_t *cell, const int32_t *v) {
  if (!h) return TS_EINVAL;
  if (!h->have_veh) return fail(h, TS_EINVAL, "load vehicles first");
  if (h->inited) return fail(h, TS_EINVAL, "already initialised");
  if (n < 0) return fail(h, TS_EINVAL, "negative placement count");
  InitTrace trace("load");
  // error code of placement i against the loaded routes (0 = ok)
  auto check = [&](int32_t i) -> int {
    const int32_t f = vid[i];
    if (f < 0 || f >= h->nv) return 1;
    const int32_t c = cursor ? cursor[i] : 0;
    if (c < 0 || c >= h->roff[f + 1] - h->roff[f]) return 3;
    const int32_t k = link_at(h, f, c);
    if (lane[i] < 0 || lane[i] >= h->lanes[k] || cell[i] < 0 || cell[i] >= h->ncell[k]) return 4;
    if (v[i] < 0 || v[i] > h->vmax[k]) return 5;
    return 0;
  };
  // parallel pass: validate, claim the vehicles (atomic flag), record the
  // placement at its batch index; any failure undoes the claims and the
  // serial pass below reports the first failing placement in input order
  const size_t base = h->pl_vid.size();
  for (auto *a : {&h->pl_vid, &h->pl_cur, &h->pl_lane, &h->pl_cell, &h->pl_v}) a->resize(base + n);
  std::vector<uint8_t> won(n, 0);
  std::vector<uint8_t> failed(64, 0);
  parallel_for(n, [&](int64_t lo, int64_t hi, int th) {
    for (int64_t i = lo; i < hi; i++) {
      if (check((int32_t)i)) {
        failed[th] = 1;
        return;
      }
      const int32_t f = vid[i];
      if (__atomic_exchange_n(&h->placed[f], (uint8_t)1, __ATOMIC_RELAXED)) {
        failed[th] = 1;
        return;
      }
      won[i] = 1;
      h->pl_vid[base + i] = f;
      h->pl_cur[base + i] = cursor ? cursor[i] : 0;
      h->pl_lane[base + i] = lane[i];
      h->pl_cell[base + i] = cell[i];
      h->pl_v[base + i] = v[i];
    }
  });
  if (std::find(failed.begin(), failed.end(), 1) == failed.end()) {
    trace("placements");
    return TS_OK;
  }
  for (int32_t i = 0; i < n; i++)
    if (won[i]) h->placed[vid[i]] = 0;
  for (auto *a : {&h->pl_vid, &h->pl_cur, &h->pl_lane, &h->pl_cell, &h->pl_v}) a->resize(base);
  static const char *msg[] = {"", "bad vid", "vehicle placed twice", "cursor outside the route",
                              "cell outside link", "velocity"};
  for (int32_t i = 0; i < n; i++) {
    const int32_t f = vid[i];
    const int e = (f < 0 || f >= h->nv) ? 1 : h->placed[f] ? 2 : check(i);
    if (e) {
      for (int32_t j = 0; j < i; j++) h->placed[vid[j]] = 0;
      return fail(h, TS_EINVAL, "placement %d: %s", i, msg[e]);
    }
    h->placed[vid[i]] = 1;
  }
  return fail(h, TS_EINTERNAL, "placement: inconsistent parallel check");
}

int ts_place_vehicles(ts_sim *h, int32_t n, const int32_t *vid, const int32_t *lane,
                      const int32_t *cell, const int32_t *v) {
  return ts_place_vehicles_at(h, n, vid, nullptr, lane, cell, v);
}

int ts_set_arrived(ts_sim *h, int32_t n, const int32_t *vid, const int32_t *t_arrive) {
  if (!h) return TS_EINVAL;
  if (!h->have_veh) return fail(h, TS_EINVAL, "load vehicles first");
  if (h->inited) return fail(h, TS_EINVAL, "already initialised");
  if (h->arr0.empty()) h->arr0.assign(h->nv, -1);
  for (int32_t i = 0; i < n; i++) {
    const int32_t f = vid[i];
    if (f < 0 || f >= h->nv || h->placed[f]) return fail(h, TS_EINVAL, "arrival %d: bad vid", i);
    if (t_arrive[i] < 0) return fail(h, TS_EINVAL, "arrival %d: negative time", i);
    h->placed[f] = 1;
    h->arr0[f] = t_arrive[i];
  }
  return TS_OK;
}

static uint32_t sig_word(int cycle, int shift, int len) {
  return (1u << 31) | (uint32_t)cycle | ((uint32_t)shift << 10) | ((uint32_t)len << 20);
}

int ts_load_network_text(ts_sim *h, const char *text, size_t len) {
  if (!h || !text) return TS_EINVAL;
  int32_t nn = 0, nl = 0, ns = 0;
  char eb[256] = {0};
  if (ts_parse_network_text(text, len, &nn, &nl, &ns, nullptr, nullptr, nullptr, nullptr, nullptr,
                            nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, eb))
    return fail(h, TS_EINVAL, "network text: %s", eb);
  std::vector<int64_t> x(nn), y(nn), len_mm(nl);
  std::vector<int32_t> fr(nl), to(nl), la(nl), vm(nl), cls(nl), ids(nl), sn(ns), sg(ns), sr(ns);
  ts_parse_network_text(text, len, &nn, &nl, &ns, x.data(), y.data(), fr.data(), to.data(),
                        len_mm.data(), la.data(), vm.data(), cls.data(), ids.data(), sn.data(),
                        sg.data(), sr.data(), eb);
  if (int rc = ts_load_network(h, nn, x.data(), y.data(), nl, fr.data(), to.data(), len_mm.data(),
                               la.data(), vm.data(), cls.data(), -1))
    return rc;
  h->text_link_id = ids;
  if (ns > 0) {
    std::vector<int32_t> off(ns, 0);
    return ts_set_signals(h, ns, sn.data(), sg.data(), sr.data(), off.data());
  }
  return TS_OK;
}

int ts_load_plans_text(ts_sim *h, const char *text, size_t len) {
  if (!h || !text) return TS_EINVAL;
  if (!h->have_net) return fail(h, TS_EINVAL, "load the network first");
  std::vector<int32_t> ids = h->text_link_id;
  if (ids.empty())  // network from arrays: link ids are the indices
    for (int32_t k = 0; k < h->nl; k++) ids.push_back(k);
  int32_t nv = 0;
  int64_t ne = 0;
  char eb[256] = {0};
  if (ts_parse_plans_text(text, len, h->nl, ids.data(), &nv, &ne, nullptr, nullptr, nullptr,
                          nullptr, nullptr, eb))
    return fail(h, TS_EINVAL, "plans text: %s", eb);
  std::vector<int64_t> off(nv + 1);
  std::vector<int32_t> route(std::max<int64_t>(ne, 1)), dep(nv), entry(nv);
  ts_parse_plans_text(text, len, h->nl, ids.data(), &nv, &ne, off.data(), route.data(), dep.data(),
                      entry.data(), nullptr, eb);
  return ts_load_vehicles(h, nv, off.data(), route.data(), dep.data(), entry.data());
}

int ts_set_signals(ts_sim *h, int32_t n, const int32_t *node, const int32_t *green0,
                   const int32_t *green1, const int32_t *offset) {
  if (!h) return TS_EINVAL;
  if (!h->have_net) return fail(h, TS_EINVAL, "load the network first");
  if (h->inited) return fail(h, TS_EINVAL, "already initialised");
  if (h->node_sig.empty()) h->node_sig.assign(h->nn, 0u);
  for (int32_t i = 0; i < n; i++) {
    if (node[i] < 0 || node[i] >= h->nn) return fail(h, TS_EINVAL, "signal %d: bad node", i);
    const int g0 = green0[i], g1 = green1[i], c = g0 + g1;
    if (g0 < 0 || g1 < 0 || c < 1 || c > 1023 || offset[i] < 0)
      return fail(h, TS_EINVAL, "signal %d: bad plan", i);
    h->node_sig[node[i]] = sig_word(c, offset[i] % c, g0);
  }
  return TS_OK;
}

int ts_set_domain(ts_sim *h, int32_t k, const int32_t *domain_of_node, int32_t me) {
  if (!h) return TS_EINVAL;
  if (!h->have_net) return fail(h, TS_EINVAL, "load the network first");
  if (h->inited) return fail(h, TS_EINVAL, "already initialised");
  if (k < 1 || me < 0 || me >= k) return fail(h, TS_EINVAL, "bad domain count or index");
  if (k > std::max(1, h->nn)) return fail(h, TS_EINVAL, "more domains than nodes");
  if (k > 1 && h->periodic >= 0) return fail(h, TS_EINVAL, "a ring network has no nodes to cut at");
  if (k > 1 && !domain_of_node) return fail(h, TS_EINVAL, "domain_of_node is NULL");
  for (int i = 0; k > 1 && i < h->nn; i++)
    if (domain_of_node[i] < 0 || domain_of_node[i] >= k)
      return fail(h, TS_EINVAL, "node %d: domain %d out of range", i, domain_of_node[i]);
  h->dom_k = k;
  h->dom_me = me;
  if (k > 1) h->dom_of_node.assign(domain_of_node, domain_of_node + h->nn);
  else h->dom_of_node.assign(h->nn, 0);
  return TS_OK;
}

// pure host: the exchange partners of domain `me` and the strips (one per
// lane of every split link shared with the partner) of one message
int ts_domain_plan(int32_t n_nodes, int32_t n_links, const int32_t *from, const int32_t *to,
                   const int64_t *length_mm, const int32_t *lanes, int32_t k,
                   const int32_t *domain_of_node, int32_t me, int32_t cap, int32_t *nbr_dom,
                   int64_t *nbr_strips, int32_t *n_out) {
  if (k < 1 || me < 0 || me >= k || n_links < 0 || !n_out) return TS_EINVAL;
  std::vector<int64_t> cnt(k, 0);
  for (int32_t j = 0; j < n_links; j++) {
    if (from[j] < 0 || from[j] >= n_nodes || to[j] < 0 || to[j] >= n_nodes) return TS_EINVAL;
    const int a = domain_of_node[from[j]], b = domain_of_node[to[j]];
    if (a == b || (a != me && b != me)) continue;
    const int n = (int)((length_mm[j] + 3750) / 7500);
    if (n < 10) return TS_EINVAL;
    cnt[a == me ? b : a] += lanes[j];
  }
  int32_t m = 0;
  for (int d = 0; d < k; d++)
    if (cnt[d] > 0) {
      if (m < cap) {
        if (nbr_dom) nbr_dom[m] = d;
        if (nbr_strips) nbr_strips[m] = cnt[d];
      }
      m++;
    }
  *n_out = m;
  return TS_OK;
}

// ------------------------------------------------------------------- layout
// cells [lo, hi) of link k owned by domain `me` under a node partition:
// whole links inside the domain; a link whose end nodes lie in different
// domains is cut at h = floor(n/2), the upstream domain owning [0, h)
// (reading R16)
static void owned_range(int n, int dfrom, int dto, int me, int &lo, int &hi) {
  lo = hi = 0;
  if (dfrom == me && dto == me) hi = n;
  else if (dfrom == me) hi = n / 2;
  else if (dto == me) {
    lo = n / 2;
    hi = n;
  }
}

static bool build_tiles(ts_sim *h) {
  const int tc = h->cfg.tile_cells > 0 ? h->cfg.tile_cells : 512;
  const bool dom = h->dom_k > 1;
  h->ring_rows = h->periodic >= 0 && !dom && !(h->cfg.flags & TS_FLAG_GENERAL) &&
                 h->lanes[h->periodic] <= 32 && getenv("TSIM_RING_GENERAL") == nullptr;
  h->tiles.clear();
  h->link_tile0.assign(h->nl + 1, 0);
  h->link_ntiles.assign(h->nl, 0);
  h->own_lo.assign(h->nl, 0);
  h->own_hi.assign(h->nl, 0);
  for (int k = 0; k < h->nl; k++) {
    if (dom && k != h->periodic)
      owned_range(h->ncell[k], h->dom_of_node[h->from[k]], h->dom_of_node[h->to[k]], h->dom_me,
                  h->own_lo[k], h->own_hi[k]);
    else
      h->own_hi[k] = h->ncell[k];
  }
  int64_t off = 0;
  int32_t strip = 0;
  for (int k = 0; k < h->nl; k++) {
    const int n = h->ncell[k], lo = h->own_lo[k], hi = h->own_hi[k], span = hi - lo;
    const bool per = k == h->periodic;
    h->link_tile0[k] = (int32_t)h->tiles.size();
    if (span <= 0) continue;
    const bool split = lo > 0 || hi < n;
    // the ring is one very long link: smaller tiles give its warp-per-tile
    // kernels more warps (config 2: 512 -> 91 us, 256 -> 66 us per step)
    const bool rseg = per && h->ring_rows;  // segments of <= kRowMaxCells cells
    const int tck = rseg ? kRowMaxCells : (per && h->cfg.tile_cells <= 0) ? 256 : tc;
    int nt = (span + tck - 1) / tck;
    if (nt > 1 && span / nt < 10) nt = std::max(1, span / 10);
    h->link_ntiles[k] = nt;
    const bool halo = !rseg && (per || nt > 1 || split);
    int a = lo;
    for (int i = 0; i < nt; i++) {
      const int w = span / nt + (i < span % nt ? 1 : 0);
      TileDesc d{};
      d.off = off;
      d.link = k;
      d.a = a;
      d.lane_gid = h->lgid[k];
      d.n = n;
      d.w = (uint16_t)w;
      d.L = (uint8_t)h->lanes[k];
      uint8_t f = 0;
      if (!per && a == 0) f |= kFirst;
      if (!per && a + w == n) f |= kLast;
      if (per && !rseg) f |= kPeriodic;
      if (rseg) f |= kFirst | kLast | kRingSeg;
      if (halo) {
        f |= kHalo;
        if (per || a > 0) f |= kHasUp;
        if (per || a + w < n) f |= kHasDn;
        if (per && nt == 1) f |= 64;
        d.strip = strip;
        strip += h->lanes[k];
      } else {
        d.strip = -1;
      }
      d.flags = f;
      h->tiles.push_back(d);
      off += tile_cells_padded(w, h->lanes[k]);
      a += w;
    }
  }
  h->link_tile0[h->nl] = (int32_t)h->tiles.size();
  h->total_cells = off + 16;
  // mirror strips: the 5-cell strip of the remote half of every split link
  // (R17), filled by the exchanges
  h->mirror.assign(h->nl, -1);
  for (int k = 0; k < h->nl; k++)
    if (h->own_hi[k] > h->own_lo[k] && (h->own_lo[k] > 0 || h->own_hi[k] < h->ncell[k]) &&
        k != h->periodic) {
      h->mirror[k] = strip;
      strip += h->lanes[k];
    }
  h->nstrips = strip;
  h->halo_up.assign(std::max(1, strip), -1);
  h->halo_dn.assign(std::max(1, strip), -1);
  for (int k = 0; k < h->nl; k++) {
    const int t0 = h->link_tile0[k], nt = h->link_ntiles[k];
    for (int i = 0; i < nt; i++) {
      const TileDesc &d = h->tiles[t0 + i];
      if (d.strip < 0) continue;
      const bool per = k == h->periodic;
      if (d.flags & kHasUp)
        h->halo_up[d.strip] = (i > 0 || per) ? h->tiles[t0 + (i + nt - 1) % nt].strip : h->mirror[k];
      if (d.flags & kHasDn)
        h->halo_dn[d.strip] = (i + 1 < nt || per) ? h->tiles[t0 + (i + 1) % nt].strip : h->mirror[k];
    }
  }
  // exchange plan: per neighbour domain, the split links shared with it in
  // link order, all lanes; each side sends the strip of its boundary tile
  // and receives into the mirror slot (one buffer per neighbour,
  // PAPER.md:897-900)
  h->nbrs.clear();
  h->n_xs = 0;
  if (dom) {
    std::vector<int32_t> nb_index(h->dom_k, -1);
    for (int k = 0; k < h->nl; k++) {
      if (h->mirror[k] < 0) continue;
      const bool up = h->own_lo[k] == 0;  // this domain owns the upstream half
      const int other = up ? h->dom_of_node[h->to[k]] : h->dom_of_node[h->from[k]];
      if (nb_index[other] < 0) {
        nb_index[other] = (int32_t)h->nbrs.size();
        h->nbrs.push_back(ts_sim::Nbr{other, {}, {}, 0});
      }
      ts_sim::Nbr &nb = h->nbrs[nb_index[other]];
      const int t0 = h->link_tile0[k], nt = h->link_ntiles[k];
      const TileDesc &bt = h->tiles[up ? t0 + nt - 1 : t0];
      for (int l = 0; l < h->lanes[k]; l++) {
        nb.send_slot.push_back(bt.strip + l);
        nb.recv_slot.push_back(h->mirror[k] + l);
      }
    }
    std::sort(h->nbrs.begin(), h->nbrs.end(),
              [](const ts_sim::Nbr &a, const ts_sim::Nbr &b) { return a.dom < b.dom; });
    for (ts_sim::Nbr &nb : h->nbrs) {
      nb.off = h->n_xs;
      h->n_xs += (int64_t)nb.send_slot.size();
      if (nb.send_slot.size() != nb.recv_slot.size()) return false;  // one strip each way per lane
    }
  }
  // classify: whole non-periodic links of <= kRowMaxCells cells and <= 32
  // lanes run in k_rows (row tiles, lanes of a link on consecutive slots of
  // one 32-slot group); everything else runs in the general kernels
  const bool allow_rows = !(h->cfg.flags & TS_FLAG_GENERAL);
  h->tile_g.assign(h->tiles.size(), -1);
  h->tile_row.assign(h->tiles.size(), -1);
  h->gtiles.clear();
  h->rows.clear();
  h->gvoff.clear();
  int64_t goff = 0, voff = 0, gbase = 0;
  int slot = 32;
  for (size_t i = 0; i < h->tiles.size(); i++) {
    const TileDesc &d = h->tiles[i];
    const bool row = allow_rows && !(d.flags & kHalo) && (d.flags & kFirst) && (d.flags & kLast) &&
                     d.w <= kRowMaxCells && d.L <= 32;
    if (!row) {
      TileDesc gd = d;
      gd.off = goff;
      goff += tile_cells_padded(d.w, d.L);
      h->tile_g[i] = (int32_t)h->gtiles.size();
      h->gtiles.push_back(gd);
      continue;
    }
    if (slot + d.L > 32) {  // new group: its vid block starts after the last one
      voff = (voff + 3) & ~(int64_t)3;
      gbase = voff;
      h->rows.resize(h->rows.size() + 32, RowDesc{0, 0, 0, 0, 0, 0, 1});
      h->gvoff.push_back((int32_t)gbase);
      slot = 0;
    }
    const size_t base = h->rows.size() - 32;
    h->tile_row[i] = (int32_t)(base + slot);
    for (int l = 0; l < d.L; l++) {
      RowDesc &r = h->rows[base + slot + l];
      r.link = d.link;
      r.lg = d.lane_gid + l;
      r.w = (uint8_t)d.w;
      r.l = (uint8_t)l;
      r.L = (uint8_t)d.L;
      r.vk = (uint8_t)h->vmax[d.link];
      voff += d.w;
    }
    slot += d.L;
  }
  h->ngroups = (int32_t)(h->rows.size() / 32);
  h->gcells = goff + 16;
  h->rvid_entries = voff + 16;
  int nc_max = 32;
  for (const TileDesc &d : h->gtiles) nc_max = std::max(nc_max, (int)d.L * tile_stride(d.w, d.flags));
  h->lay = warp_layout(nc_max);
  h->gfused = (h->cfg.flags & TS_FLAG_FUSED) && h->nstrips == 0;
  // ring segment rows take their lane change in a launch of its own (its
  // neighbour segments must hold S(t))
  h->rfused = (h->cfg.flags & TS_FLAG_FUSED) != 0 && !h->ring_rows;
  return true;
}

// incoming lanes of every node in priority order (R9: major class first,
// then link id, then lane), packed into chunks of <= 32 lanes
static bool build_node_lanes(ts_sim *h, std::vector<NodeLane> &lanes,
                             std::vector<uint32_t> &sig, std::vector<int32_t> &nl_node,
                             std::vector<int32_t> &nl_row, const std::vector<int32_t> &lane_row) {
  lanes.clear();
  sig.clear();
  nl_node.clear();
  nl_row.clear();
  int in_chunk = 0;
  auto close_chunk = [&]() {  // pad the chunk to 32 entries
    while (lanes.size() % 32) {
      lanes.push_back(NodeLane{-1, 0, 0u, 0, 0, 1, 0});
      sig.push_back(0u);
      nl_node.push_back(-1);
      nl_row.push_back(-1);
    }
    in_chunk = 0;
  };
  for (int nd = 0; nd < h->nn; nd++) {
    const int a = h->in_off[nd], b = h->in_off[nd + 1];
    if (a == b || h->dom_of_node[nd] != h->dom_me) continue;
    int maxcls = h->cls[h->in_list[a]], nl = 0;
    for (int i = a; i < b; i++) {
      maxcls = std::max(maxcls, h->cls[h->in_list[i]]);
      nl += h->lanes[h->in_list[i]];
    }
    if (nl > 32) return false;
    if (in_chunk + nl > 32) close_chunk();
    const int node_first = in_chunk;  // the node's first lane in its chunk (match key)
    for (int pass = 0; pass < 2; pass++)
      for (int i = a; i < b; i++) {
        const int j = h->in_list[i];
        if ((h->cls[j] == maxcls) != (pass == 0)) continue;
        for (int l = 0; l < h->lanes[j]; l++) {  // one NodeLane and one signal word per lane
          lanes.push_back(NodeLane{h->lgid[j] + l, h->out_off[nd], h->tt[j], (uint8_t)l,
                                   (uint8_t)(pass == 0), (uint8_t)h->vmax[j],
                                   (uint8_t)node_first});
          nl_node.push_back(nd);
          nl_row.push_back(lane_row[h->lgid[j] + l]);
          uint32_t sw = 0u;  // the lane's phase (R23): 0 = maximal class, 1 = the rest
          const uint32_t s0 = h->node_sig.empty() ? 0u : h->node_sig[nd];
          if (s0 >> 31) {
            const int c = (int)(s0 & 1023u), sh = (int)((s0 >> 10) & 1023u),
                      g0 = (int)((s0 >> 20) & 1023u);
            sw = pass == 0 ? s0 : sig_word(c, ((sh - g0) % c + c) % c, c - g0);
          }
          sig.push_back(sw);
        }
      }
    in_chunk += nl;
  }
  close_chunk();
  return true;
}

// node-lane indices (tail records, node grants): the lane's position in the
// node kernel's lane array, or the identity for the thread-per-node kernel;
// lanes without a node of this domain share a dummy slot at the end
// the periodic link's segments joined by pass-through virtual nodes: node s
// takes the L lanes of segment s to the same lanes of segment s + 1 (mod S)
// -- a straight continuation with a single approach, so the node kernel's
// entry space and crossing are exactly the in-lane gap and move across the
// cut (reading R2 / R10 on a ring, where no vehicle can pass two cuts)
static int setup_ring_nodes(ts_sim *h) {
  const int k = h->periodic, L = h->lanes[k];
  std::vector<int> seg;  // tiles of the ring in cell order
  for (size_t ti = 0; ti < h->tiles.size(); ti++)
    if (h->tiles[ti].flags & kRingSeg) seg.push_back((int)ti);
  const int S = (int)seg.size(), per_chunk = 32 / L;
  std::vector<NodeLane> nlanes;
  std::vector<int32_t> nl_row;  // row slot per node-lane index
  auto pad = [&]() {
    while (nlanes.size() % 32) {
      nlanes.push_back(NodeLane{-1, 0, 0u, 0, 0, 1, 0});
      nl_row.push_back(-1);
    }
  };
  h->ring_nodeout.assign(S, NodeOut{});
  std::vector<int32_t> nxt(h->rows.size(), -1), prv(h->rows.size(), -1), ra(h->rows.size(), 0);
  for (int s = 0; s < S; s++) {
    if (s % per_chunk == 0) pad();
    const int first = (int)(nlanes.size() % 32);
    const TileDesc &d = h->tiles[seg[s]];
    const TileDesc &dn = h->tiles[seg[(s + 1) % S]], &dp = h->tiles[seg[(s + S - 1) % S]];
    for (int l = 0; l < L; l++) {
      const int row = h->tile_row[seg[s]] + l;
      nl_row.push_back(row);
      RowDesc &r = h->rows[row];
      r.nli = (int32_t)nlanes.size();
      r.lg = s * L + l;  // node-out-lane index: segment s is the target of node s - 1
      nxt[row] = h->tile_row[seg[(s + 1) % S]] + l;
      prv[row] = (h->tile_row[seg[(s + S - 1) % S]] + l) | ((int32_t)dp.w << 24);
      ra[row] = d.a;
      // pass-through (major | 2): out-slot 0 is the next segment, straight on
      nlanes.push_back(NodeLane{k, s, 0u, (uint8_t)l, (uint8_t)(1 | 2), (uint8_t)h->vmax[k],
                                (uint8_t)first});
    }
    h->ring_nodeout[s] = NodeOut{((s + 1) % S) * L, (int16_t)L, (int16_t)dn.w,
                                 h->tile_row[seg[(s + 1) % S]]};
  }
  pad();
  h->node_warp = true;
  h->nchunks = (int32_t)(nlanes.size() / 32);
  h->n_nli = (int64_t)nlanes.size() + 1;
  h->n_nlo = (int64_t)S * L + 1;
  h->nli.assign(h->nlanes, 0);
  h->nlo.assign(h->nlanes, 0);
  h->d_lane_sig = nullptr;
  int rc;
  if ((rc = upload(h, &h->d_nlanes, nlanes))) return rc;
  if ((rc = upload(h, &h->d_nl_row, nl_row))) return rc;
  if ((rc = upload(h, &h->d_ring_next, nxt))) return rc;
  if ((rc = upload(h, &h->d_ring_prev, prv))) return rc;
  if ((rc = upload(h, &h->d_row_a, ra))) return rc;
  return 0;
}

// row slot of every global lane id (-1: not a row-kernel lane); the node
// kernels write the grants and entrant records of these lanes by row slot too
static std::vector<int32_t> lane_rows(const ts_sim *h) {
  std::vector<int32_t> lr(std::max<int64_t>(h->nlanes, 1), -1);
  if (h->ring_rows) return lr;  // ring segments: by node lane (setup_ring_nodes)
  for (size_t ti = 0; ti < h->tiles.size(); ti++)
    if (h->tile_row[ti] >= 0)
      for (int l = 0; l < h->tiles[ti].L; l++) lr[h->tiles[ti].lane_gid + l] = h->tile_row[ti] + l;
  return lr;
}

static int setup_node_lanes(ts_sim *h) {
  int rc;
  const std::vector<int32_t> lane_row = lane_rows(h);
  if ((rc = upload(h, &h->d_lane_row, lane_row))) return rc;
  h->lane_row0.resize(h->nl);
  for (int k = 0; k < h->nl; k++) h->lane_row0[k] = lane_row[h->lgid[k]];
  if (h->ring_rows) return setup_ring_nodes(h);
  std::vector<NodeLane> nlanes;
  std::vector<uint32_t> lsig;
  std::vector<int32_t> nl_node, nl_row;
  h->node_warp = h->periodic < 0 && !(h->cfg.flags & (TS_FLAG_GENERAL | TS_FLAG_NODE_GENERAL)) &&
                 build_node_lanes(h, nlanes, lsig, nl_node, nl_row, lane_row);
  h->nli.assign(h->nlanes, 0);
  if (h->node_warp) {
    h->nchunks = (int32_t)(nlanes.size() / 32);
    h->n_nli = std::max<int64_t>((int64_t)nlanes.size(), 1) + 1;
    for (int32_t &x : h->nli) x = (int32_t)(h->n_nli - 1);
    for (size_t i = 0; i < nlanes.size(); i++)
      if (nlanes[i].lane_gid >= 0) h->nli[nlanes[i].lane_gid] = (int32_t)i;
    if ((rc = upload(h, &h->d_nlanes, nlanes))) return rc;
    if ((rc = upload(h, &h->d_nl_node, nl_node))) return rc;
    if ((rc = upload(h, &h->d_nl_row, nl_row))) return rc;
    if (h->node_sig.empty()) h->d_lane_sig = nullptr;
    else if ((rc = upload(h, &h->d_lane_sig, lsig))) return rc;
  } else {
    h->n_nli = std::max<int64_t>(h->nlanes, 1);
    for (int i = 0; i < h->nlanes; i++) h->nli[i] = i;
  }
  // node-out-lane indices (head occupancy, entrant records): the outgoing
  // lanes of every node of this domain contiguous, in node order, so the
  // node kernel's target lookups stay within a few sectors per node
  h->nlo.assign(h->nlanes, 0);
  if (h->node_warp) {
    int32_t cnt = 0;
    std::vector<int32_t> map(h->nlanes, -1);
    for (int nd = 0; nd < h->nn; nd++) {
      if (h->dom_of_node[nd] != h->dom_me) continue;
      for (int i = h->out_off[nd]; i < h->out_off[nd + 1]; i++) {
        const int k = h->out_list[i];
        for (int l = 0; l < h->lanes[k]; l++) map[h->lgid[k] + l] = cnt++;
      }
    }
    h->n_nlo = (int64_t)cnt + 1;
    for (int i = 0; i < h->nlanes; i++) h->nlo[i] = map[i] >= 0 ? map[i] : cnt;
  } else {
    h->n_nlo = std::max<int64_t>(h->nlanes, 1);
    for (int i = 0; i < h->nlanes; i++) h->nlo[i] = i;
  }
  for (RowDesc &r : h->rows)
    if (r.w > 0) {
      r.nli = h->nli[r.lg];
      r.lg = h->nlo[r.lg];
    }
  return 0;
}

static int tile_of(const ts_sim *h, int k, int x) {
  int t0 = h->link_tile0[k], nt = h->link_ntiles[k];
  for (int i = 0; i < nt; i++) {
    const TileDesc &d = h->tiles[t0 + i];
    if (x >= d.a && x < d.a + d.w) return t0 + i;
  }
  return -1;
}


StepParams step_params(ts_sim *h, int t, int mode) {
  StepParams P{};
  if (h->capturing) {
    P.tdev = h->d_clock;
    t -= h->graph_t0;
  }
  P.tiles = h->d_tiles;
  P.ntiles = (int32_t)h->gtiles.size();
  P.t = t;
  P.mode = mode;
  P.D = h->cfg.desperation_D;
  P.Dmul = (uint32_t)((0x100000000ull + (uint64_t)P.D - 1) / (uint64_t)P.D);
  P.k0 = (uint32_t)(h->cfg.seed & 0xffffffffu);
  P.k1 = (uint32_t)(h->cfg.seed >> 32);
  for (int r = 0; r < 10; r++) {  // Philox4x32-10 key schedule (curand's Weyl constants)
    P.rk[2 * r] = P.k0 + (uint32_t)r * 0x9E3779B9u;
    P.rk[2 * r + 1] = P.k1 + (uint32_t)r * 0xBB67AE85u;
  }
  P.p32 = h->p32;
  P.lay = h->lay;
  P.code_in = h->d_code[h->gcur];
  P.code_out = h->d_code[h->gcur ^ 1];
  P.vid_in = h->d_vid[h->gcur];
  P.vid_out = h->d_vid[h->gcur ^ 1];
  P.strip_in = h->d_strip[h->gcur];
  P.strip_out = h->d_strip[h->gcur ^ 1];
  P.halo_up = h->d_halo_up;
  P.halo_dn = h->d_halo_dn;
  P.vmax_link = h->d_vmax;
  P.tt_link = h->d_tt;
  P.out_pos = h->d_out_pos;
  P.rslot = h->d_rslot;
  P.vpos = h->d_vpos;
  P.dep = h->d_dep;
  P.entry = h->d_entry;
  P.inj_time = h->d_inj;
  P.arr_time = h->d_arr;
  P.pend_off = h->d_pend_off;
  P.pend_list = h->d_pend_list;
  P.pend_head = h->d_pend_head;
  P.nli = h->d_nli;
  P.nlo = h->d_nlo;
  P.tail_rec = h->d_tail;
  P.head_occ = h->d_head;
  P.ext = h->d_ext;
  P.entr = h->d_entr;
  P.ext_row = h->d_ext_row;
  P.entr_row = h->d_entr_row;
  P.stats = h->d_stats;
  P.link_work = h->d_work;
  return P;
}

static NodeParams node_params(ts_sim *h, int t) {
  NodeParams N{};
  if (h->capturing) {
    N.tdev = h->d_clock;
    t -= h->graph_t0;
  }
  N.nnodes = h->periodic >= 0 ? 0 : (int32_t)h->my_nodes.size();
  N.node_ids = h->d_node_ids;
  N.t = t;
  N.G = h->cfg.gap_accept_G;
  N.k0 = (uint32_t)(h->cfg.seed & 0xffffffffu);
  N.k1 = (uint32_t)(h->cfg.seed >> 32);
  N.p32 = h->p32;
  N.in_off = h->d_in_off;
  N.in_list = h->d_in_list;
  N.out_off = h->d_out_off;
  N.out_list = h->d_out_list;
  N.link_ncell = h->d_ncell;
  N.link_lanes = h->d_lanes;
  N.link_lgid = h->d_lgid;
  N.link_cls = h->d_cls;
  N.vmax_link = h->d_vmax;
  N.tt_link = h->d_tt;
  N.out_pos = h->d_out_pos;
  N.rslot = h->d_rslot;
  N.nodeout = h->d_nodeout;
  N.node_sig = h->d_node_sig;
  N.vpos = h->d_vpos;
  N.tail_rec = h->d_tail;
  N.head_occ = h->d_head;
  N.ext = h->d_ext;
  N.entr = h->d_entr;
  N.ext_row = h->d_ext_row;
  N.entr_row = h->d_entr_row;
  N.lane_row = h->d_lane_row;
  N.stats = h->d_stats;
  N.node_work = (h->cfg.flags & TS_FLAG_LINK_WORK) && h->periodic < 0 ? h->d_node_work : nullptr;
  return N;
}

RowsParams rows_params(ts_sim *h) {
  RowsParams r{};
  r.rows = h->d_rows;
  r.ring_next = h->ring_rows ? h->d_ring_next : nullptr;
  r.ring_prev = h->ring_rows ? h->d_ring_prev : nullptr;
  r.row_a = h->ring_rows ? h->d_row_a : nullptr;
  r.gvoff = h->d_gvoff;
  r.planes_in = h->d_planes[h->rcur];
  r.planes_out = h->d_planes[h->rcur ^ 1];
  r.vid_in = h->d_rvid[h->rcur];
  r.vid_out = h->d_rvid[h->rcur ^ 1];
  r.inj_scratch = h->d_inj_scratch;
  r.gcnt_in = h->d_gcnt[h->rcur];
  r.gcnt_out = h->d_gcnt[h->rcur ^ 1];
  r.ngroups = h->ngroups;
  r.cap = h->rows_cap;
  r.gctr = h->d_gctr;
  r.gbase = h->gctr_base;
  return r;
}

// k_rows launch; the work counter advances by the groups: every warp takes
// its first group by its index, then one fetch per further group and one
// failed fetch (warps without a first group fetch nothing)
static void rows_launch(ts_sim *h, const StepParams &p, bool pdl = false) {
  launch_rows(p, rows_params(h), h->rows_blocks, h->rows_threads, h->rows_smem, h->stream, pdl);
  h->gctr_base += (unsigned long long)h->ngroups +
                  (TS_ROWS_FIRST_STATIC ? 0ull
                                        : (unsigned long long)h->rows_blocks * (h->rows_threads / 32));
}

static int base_mode(const ts_sim *h) {
  // injection only while this domain still has pending trips (the count
  // only falls; a stale host count errs on the side of injecting)
  int m = kModeMove | (h->n_pending0 - h->injected > 0 ? kModeInject : 0);
  if (h->cfg.flags & TS_FLAG_HASH) m |= kModeHash;
  if (h->cfg.flags & TS_FLAG_LINK_WORK) m |= kModeWork;
  return m;
}

static int zero_stats(ts_sim *h, int32_t t_from, int32_t n) {
  // slots t_from .. t_from+n-1 (mod kHist)
  if (n >= kHist) {
    CK(h, cudaMemsetAsync(h->d_stats, 0, sizeof(unsigned long long) * kHist * ST_N, h->stream));
    return TS_OK;
  }
  int s = t_from & (kHist - 1);
  int n1 = std::min(n, kHist - s);
  CK(h, cudaMemsetAsync(h->d_stats + (size_t)s * ST_N, 0, sizeof(unsigned long long) * ST_N * n1,
                        h->stream));
  if (n > n1)
    CK(h, cudaMemsetAsync(h->d_stats, 0, sizeof(unsigned long long) * ST_N * (n - n1), h->stream));
  return TS_OK;
}


// host staging of the initial placement (TSIM_HOST_INIT=1, and the exact
// report of a cell claimed twice): codes + compact vid lists per tile, then
// the row planes and vid blocks, uploaded
static int place_host(ts_sim *h, HostVec<int32_t> &cur0, std::vector<uint8_t> &gcode,
                      std::vector<int32_t> &gvid) {
  // cells of other domains are skipped
  HostVec<uint8_t> code = filled<uint8_t>(h->total_cells, kEmpty);
  HostVec<int32_t> cellvid = filled<int32_t>(h->total_cells, -1);
  // placements in parallel: a cell claimed twice is found by the
  // compare-and-swap on its vehicle slot (the first placement in input
  // order is reported)
  std::vector<int64_t> taken(64, INT64_MAX);
  std::vector<int64_t> placed_cnt(64, 0);
  parallel_for((int64_t)h->pl_vid.size(), [&](int64_t lo, int64_t hi, int th) {
    for (int64_t i = lo; i < hi; i++) {
      const int f = h->pl_vid[i], c = h->pl_cur[i];
      const int k = link_at(h, f, c);
      cur0[f] = c;
      const int ti = tile_of(h, k, h->pl_cell[i]);
      if (ti < 0) continue;  // another domain's cell
      const TileDesc &d = h->tiles[ti];
      const int64_t pos = d.off + (int64_t)h->pl_lane[i] * row_pitch(d.w) + (h->pl_cell[i] - d.a);
      int32_t expect = -1;
      if (!__atomic_compare_exchange_n(&cellvid[pos], &expect, (int32_t)f, false, __ATOMIC_RELAXED,
                                       __ATOMIC_RELAXED)) {
        taken[th] = std::min(taken[th], i);
        continue;
      }
      const int64_t ro = h->roff[f];
      // ring segment rows: every vehicle goes straight on through the virtual
      // nodes (out-slot 0, all lanes allowed) instead of being on a final link
      const int slot = h->ring_rows ? 0
                       : c + 1 < h->roff[f + 1] - ro ? (int)h->rslot[ro + c + 1] : kSlotFinal;
      code[pos] = (uint8_t)(h->pl_v[i] | (slot << 3));
      placed_cnt[th]++;
    }
  });
  {
    const int64_t bad = *std::min_element(taken.begin(), taken.end());
    if (bad != INT64_MAX) {  // the first placement (input order) on a taken cell
      std::unordered_set<int64_t> seen;
      for (size_t i = 0; i < h->pl_vid.size(); i++) {
        const int k = link_at(h, h->pl_vid[i], h->pl_cur[i]);
        const int ti = tile_of(h, k, h->pl_cell[i]);
        if (ti < 0) continue;
        const TileDesc &d = h->tiles[ti];
        if (!seen.insert(d.off + (int64_t)h->pl_lane[i] * row_pitch(d.w) + (h->pl_cell[i] - d.a)).second)
          return fail(h, TS_EINVAL, "placement %zu: cell taken", i);
      }
      return fail(h, TS_EINVAL, "placement %lld: cell taken", (long long)bad);
    }
    for (int64_t c : placed_cnt) h->n_placed += c;
  }
  HostVec<int32_t> vids = filled<int32_t>(h->total_cells, -1);
  parallel_for((int64_t)h->tiles.size(), [&](int64_t lo, int64_t hi, int) {
    for (int64_t ti = lo; ti < hi; ti++) {  // per-row vid lists in cell order
      const TileDesc &d = h->tiles[ti];
      const int Wp = row_pitch(d.w);
      for (int l = 0; l < d.L; l++) {
        const int64_t rb = d.off + (int64_t)l * Wp;
        int64_t r = rb;
        for (int x = 0; x < d.w; x++)
          if (code[rb + x] != kEmpty) vids[r++] = cellvid[rb + x];
      }
    }
  });
  HostVec<int32_t>().swap(cellvid);
  // general tiles: the byte layout at their own device offsets
  gcode.assign(h->gcells, kEmpty);
  gvid.assign(h->gcells, -1);
  for (size_t ti = 0; ti < h->tiles.size(); ti++) {
    if (h->tile_g[ti] < 0) continue;
    const TileDesc &d = h->tiles[ti], &gd = h->gtiles[h->tile_g[ti]];
    const int64_t n = (int64_t)d.L * row_pitch(d.w);
    std::copy(code.begin() + d.off, code.begin() + d.off + n, gcode.begin() + gd.off);
    std::copy(vids.begin() + d.off, vids.begin() + d.off + n, gvid.begin() + gd.off);
  }
  // row tiles: bit-planes O, V0..V2, A0, A1 per row (group-interleaved);
  // list entries vid | slot << 27
  HostVec<uint32_t> planes = filled<uint32_t>(group_plane_base(h->ngroups), 0u);
  HostVec<int32_t> rvid = filled<int32_t>(h->rvid_entries, -1);
  std::vector<int32_t> row_tile(h->rows.size(), -1);  // row slot -> tile
  for (size_t ti = 0; ti < h->tiles.size(); ti++)
    if (h->tile_row[ti] >= 0)
      for (int l = 0; l < h->tiles[ti].L; l++) row_tile[h->tile_row[ti] + l] = (int32_t)ti;
  std::vector<int32_t> gcnt(std::max(1, h->ngroups), 0);
  parallel_for(h->ngroups, [&](int64_t glo, int64_t ghi, int) {
  for (int g = (int)glo; g < (int)ghi; g++) {
    const int64_t k0 = h->gvoff[g];
    int64_t k = k0;  // the group's block: rows in slot order
    for (int sl = 0; sl < 32; sl++) {
      const int s = g * 32 + sl;
      if (row_tile[s] < 0) continue;
      const TileDesc &d = h->tiles[row_tile[s]];
      const int l = h->rows[s].l, Wp = row_pitch(d.w);
      uint32_t *pl = planes.data() + group_plane_base(g) + sl;
      int64_t r = d.off + (int64_t)l * Wp;
      for (int x = 0; x < d.w; x++) {
        const uint8_t c = code[d.off + (int64_t)l * Wp + x];
        if (c == kEmpty) continue;
        const uint32_t bit = 1u << (x & 31);
        const int wd = x >> 5;
        pl[(0 * kRowWords + wd) * 32] |= bit;
        for (int b = 0; b < 3; b++)
          if ((c >> b) & 1) pl[((1 + b) * kRowWords + wd) * 32] |= bit;
        // allowed-lane class (R7): 0 all, 1 curb (right turn), 2 median (left)
        const int slot = c >> 3;
        int cls = 0;
        if (slot != kSlotFinal) {
          const int tty = (h->tt[d.link] >> (2 * slot)) & 3;
          cls = tty == 0 ? 0 : (tty == 2 ? 1 : 2);
        }
        for (int b = 0; b < 2; b++)
          if ((cls >> b) & 1) pl[((4 + b) * kRowWords + wd) * 32] |= bit;
        rvid[k++] = (int32_t)((uint32_t)vids[r++] | ((uint32_t)slot << kSlotShift));
      }
    }
    gcnt[g] = (int32_t)(k - k0);
  }
  });
  if (h->ngroups > 0) {
    CK(h, cudaMemcpyAsync(h->d_planes[0], planes.data(), planes.size() * 4, cudaMemcpyHostToDevice,
                          h->stream));
    CK(h, cudaMemcpyAsync(h->d_rvid[0], rvid.data(), rvid.size() * 4, cudaMemcpyHostToDevice,
                          h->stream));
    CK(h, cudaMemcpyAsync(h->d_gcnt[0], gcnt.data(), gcnt.size() * 4, cudaMemcpyHostToDevice,
                          h->stream));
    CK(h, cudaStreamSynchronize(h->stream));  // the staging arrays are freed on return
  }
  return TS_OK;
}

// ------------------------------------------------ device-side placement
// The row-tile placements become one record each (row slot s and cell x as
// s << 7 | x, the list entry vid | slot << 27, velocity | lane class << 3);
// k_place_bits ORs each into the bit-planes (an occupancy bit already set
// is a cell claimed twice: flagged, and the host path reports it),
// k_place_rows turns each group's occupancy popcounts into row offsets
// (warp scan) and the group count, k_place_lists writes each entry at its
// rank within its row (popcount of the occupancy below its cell) -- the
// layout the host path builds, without staging planes and lists in host
// memory.
constexpr int kPlaceHost = -1000;       // place_device: use the host path
constexpr uint32_t kNoPlace = 0xFFFFFFFFu;

__global__ void k_place_bits(const uint32_t *__restrict__ pos, const uint8_t *__restrict__ vc, int64_t n,
                             uint32_t *planes, uint32_t *conflict) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || pos[i] == kNoPlace) return;
  const uint32_t s = pos[i] >> 7, x = pos[i] & 127u, q = vc[i];
  uint32_t *pl = planes + group_plane_base(s >> 5) + (s & 31u) + (x >> 5) * 32;
  const uint32_t bit = 1u << (x & 31u);
  if (atomicOr(pl, bit) & bit) atomicExch(conflict, 1u);
  for (int p = 1; p <= 5; p++)  // V0..V2 (q bits 0-2), A0, A1 (q bits 3-4)
    if ((q >> (p - 1)) & 1u) atomicOr(pl + p * kRowWords * 32, bit);
}

__global__ void k_place_rows(const uint32_t *__restrict__ planes, const int32_t *__restrict__ gvoff, int ngroups,
                             int32_t *rowoff, int32_t *gcnt) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int g = (int)(s >> 5), lane = threadIdx.x & 31;
  if (g >= ngroups) return;  // whole warps (blockDim a multiple of 32)
  const uint32_t *pl = planes + group_plane_base(g) + lane;
  int c = 0;
  for (int w = 0; w < kRowWords; w++) c += __popc(pl[w * 32]);
  int inc = c;
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += o;
  }
  rowoff[s] = gvoff[g] + inc - c;
  if (lane == 31) gcnt[g] = inc;
}

__global__ void k_place_lists(const uint32_t *__restrict__ pos, const uint32_t *__restrict__ ent, int64_t n,
                              const uint32_t *__restrict__ planes, const int32_t *__restrict__ rowoff,
                              int32_t *rvid) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || pos[i] == kNoPlace) return;
  const uint32_t s = pos[i] >> 7, x = pos[i] & 127u;
  const uint32_t *pl = planes + group_plane_base(s >> 5) + (s & 31u);
  int r = __popc(pl[(x >> 5) * 32] & ((1u << (x & 31u)) - 1u));
  for (uint32_t w = 0; w < (x >> 5); w++) r += __popc(pl[w * 32]);
  rvid[rowoff[s] + r] = (int32_t)ent[i];
}

// per-vehicle words of a fresh start (no restored arrivals) built on the
// device from the route offsets (uploaded once, also used by the read-back),
// the initial cursors and the placed flags: route position, injection word
// (placed: INT_MIN, pending: INT_MAX), arrival time -1
__global__ void k_init_vehicles(int nv, const int64_t *__restrict__ roff, const int32_t *__restrict__ cur0,
                                const uint8_t *__restrict__ placed, VehPos *vpos, int32_t *inj,
                                int32_t *arr) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nv) return;
  vpos[f] = VehPos{roff[f] + cur0[f], roff[f + 1]};
  inj[f] = placed[f] ? INT_MIN : INT_MAX;
  arr[f] = -1;
}

// the placement with the row tiles built on the device (general tiles on
// the host, at their own offsets); kPlaceHost when the host path must run
static int place_device(ts_sim *h, HostVec<int32_t> &cur0, std::vector<uint8_t> &gcode,
                        std::vector<int32_t> &gvid) {
  InitTrace trace;
  const int64_t n = (int64_t)h->pl_vid.size();
  if (h->rows.size() > ((size_t)1 << 25)) return kPlaceHost;  // s << 7 | x in 32 bits
  HostVec<uint32_t> pos(std::max<int64_t>(n, 1)), ent(std::max<int64_t>(n, 1));
  HostVec<uint8_t> vc(std::max<int64_t>(n, 1));
  gcode.assign(h->gcells, kEmpty);
  std::vector<int32_t> gcell(h->gcells, -1);
  std::vector<int64_t> placed_cnt(64, 0);
  std::vector<uint8_t> taken(64, 0);
  parallel_for(n, [&](int64_t lo, int64_t hi, int th) {
    for (int64_t i = lo; i < hi; i++) {
      pos[i] = kNoPlace;
      const int f = h->pl_vid[i], c = h->pl_cur[i];
      const int k = link_at(h, f, c);
      cur0[f] = c;
      const int ti = tile_of(h, k, h->pl_cell[i]);
      if (ti < 0) continue;  // another domain's cell
      const TileDesc &d = h->tiles[ti];
      const int64_t ro = h->roff[f];
      // ring segment rows: straight on through the virtual nodes (out-slot 0)
      const int slot = h->ring_rows ? 0
                       : c + 1 < h->roff[f + 1] - ro ? (int)h->rslot[ro + c + 1] : kSlotFinal;
      const int x = h->pl_cell[i] - d.a;
      if (h->tile_row[ti] >= 0) {
        // allowed-lane class (R7): 0 all, 1 curb (right turn), 2 median (left)
        int cls = 0;
        if (slot != kSlotFinal) {
          const int tty = (h->tt[d.link] >> (2 * slot)) & 3;
          cls = tty == 0 ? 0 : (tty == 2 ? 1 : 2);
        }
        pos[i] = ((uint32_t)(h->tile_row[ti] + h->pl_lane[i]) << 7) | (uint32_t)x;
        ent[i] = (uint32_t)f | ((uint32_t)slot << kSlotShift);
        vc[i] = (uint8_t)(h->pl_v[i] | (cls << 3));
      } else {
        const TileDesc &gd = h->gtiles[h->tile_g[ti]];
        const int64_t p = gd.off + (int64_t)h->pl_lane[i] * row_pitch(d.w) + x;
        int32_t expect = -1;
        if (!__atomic_compare_exchange_n(&gcell[p], &expect, (int32_t)f, false, __ATOMIC_RELAXED,
                                         __ATOMIC_RELAXED)) {
          taken[th] = 1;
          continue;
        }
        gcode[p] = (uint8_t)(h->pl_v[i] | (slot << 3));
      }
      placed_cnt[th]++;
    }
  });
  for (uint8_t t : taken)
    if (t) return kPlaceHost;
  trace("  records");
  // general tiles: per-row vid lists in cell order
  gvid.assign(h->gcells, -1);
  parallel_for((int64_t)h->gtiles.size(), [&](int64_t lo, int64_t hi, int) {
    for (int64_t gi = lo; gi < hi; gi++) {
      const TileDesc &d = h->gtiles[gi];
      const int Wp = row_pitch(d.w);
      for (int l = 0; l < d.L; l++) {
        const int64_t rb = d.off + (int64_t)l * Wp;
        int64_t r = rb;
        for (int x = 0; x < d.w; x++)
          if (gcode[rb + x] != kEmpty) gvid[r++] = gcell[rb + x];
      }
    }
  });
  // row tiles on the device (stream-ordered scratch)
  const int64_t nrows = (int64_t)h->ngroups * 32;
  uint32_t *d_pos = nullptr, *d_ent = nullptr, *d_flag = nullptr;
  uint8_t *d_vc = nullptr;
  int32_t *d_rowoff = nullptr;
  const size_t nb = (size_t)std::max<int64_t>(n, 1);
  CK(h, cudaMallocAsync(&d_pos, nb * 4, h->stream));
  CK(h, cudaMallocAsync(&d_ent, nb * 4, h->stream));
  CK(h, cudaMallocAsync(&d_vc, nb, h->stream));
  CK(h, cudaMallocAsync(&d_rowoff, (size_t)nrows * 4, h->stream));
  CK(h, cudaMallocAsync(&d_flag, 4, h->stream));
  CK(h, cudaMemsetAsync(d_flag, 0, 4, h->stream));
  CK(h, cudaMemcpyAsync(d_pos, pos.data(), nb * 4, cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(d_ent, ent.data(), nb * 4, cudaMemcpyHostToDevice, h->stream));
  CK(h, cudaMemcpyAsync(d_vc, vc.data(), nb, cudaMemcpyHostToDevice, h->stream));
  trace("  general lists + uploads");
  const int nblk = (int)((n + 255) / 256);
  if (n > 0) k_place_bits<<<nblk, 256, 0, h->stream>>>(d_pos, d_vc, n, h->d_planes[0], d_flag);
  k_place_rows<<<(int)((nrows + 255) / 256), 256, 0, h->stream>>>(h->d_planes[0], h->d_gvoff, h->ngroups,
                                                                  d_rowoff, h->d_gcnt[0]);
  if (n > 0)
    k_place_lists<<<nblk, 256, 0, h->stream>>>(d_pos, d_ent, n, h->d_planes[0], d_rowoff, h->d_rvid[0]);
  CK(h, cudaGetLastError());
  uint32_t conflict = 0;
  CK(h, cudaMemcpyAsync(&conflict, d_flag, 4, cudaMemcpyDeviceToHost, h->stream));
  for (void *p : {(void *)d_pos, (void *)d_ent, (void *)d_vc, (void *)d_rowoff, (void *)d_flag})
    CK(h, cudaFreeAsync(p, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));  // the host records are freed on return
  trace("  kernels");
  if (conflict) {  // planes and lists are rebuilt by the host path
    CK(h, cudaMemsetAsync(h->d_planes[0], 0, group_plane_base(h->ngroups) * 4, h->stream));
    return kPlaceHost;
  }
  for (int64_t c : placed_cnt) h->n_placed += c;
  return TS_OK;
}

static int init_impl(ts_sim *h, int32_t t0, bool inject0);
static void pack_strips(ts_sim *h);

int ts_init(ts_sim *h, int32_t t0) { return init_impl(h, t0, true); }
int ts_resume(ts_sim *h, int32_t t) { return init_impl(h, t, false); }

static int init_impl(ts_sim *h, int32_t t0, bool inject0) {
  InitTrace trace;
  if (!h) return TS_EINVAL;
  if (!h->have_veh) return fail(h, TS_EINVAL, "load vehicles first");
  if (h->inited) return fail(h, TS_EINVAL, "already initialised");
  if (t0 < 0) return fail(h, TS_EINVAL, "t0 must be >= 0");
  CK(h, cudaSetDevice(h->dev));
  if (h->dom_of_node.empty()) h->dom_of_node.assign(h->nn, 0);
  if (!build_tiles(h)) return fail(h, TS_EINTERNAL, "asymmetric exchange plan");
  trace("tiles");

  // the routes (out-slot sequences built at load, GBs at the largest
  // configs) go to the device on a host thread of their own through pinned
  // double-buffered staging, overlapping the placement and plane build below
  struct RouteUpload {
    std::thread th;
    cudaError_t err = cudaSuccess;
    double secs = 0, setup_secs = 0;
    // the DMA starts once the placement's own uploads are done (they would
    // otherwise queue behind GBs of route data); the host copies into the
    // pinned buffers start at once
    std::atomic<bool> go{getenv("TSIM_ROUTE_UNGATED") != nullptr};
    ~RouteUpload() {
      go = true;
      if (th.joinable()) th.join();
    }
  } rup;
  {
    const size_t nb = h->rslot.size();
    int rc;
    if ((rc = dalloc(h, &h->d_rslot, std::max<size_t>(nb, 1)))) return rc;
    rup.th = std::thread([h, nb, &rup]() {
      cudaError_t &e = rup.err;
      const auto t_start = std::chrono::steady_clock::now();
      struct Done {
        RouteUpload &r;
        std::chrono::steady_clock::time_point t;
        ~Done() { r.secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t).count(); }
      } done_{rup, t_start};
      if ((e = cudaSetDevice(h->dev)) != cudaSuccess || nb == 0) return;
      const size_t chunk = (size_t)64 << 20;
      uint8_t *pin[2] = {nullptr, nullptr};
      cudaEvent_t done[2] = {nullptr, nullptr};
      cudaStream_t st = nullptr;
      const bool pinned = nb > chunk && cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) == cudaSuccess &&
                          cudaMallocHost(&pin[0], chunk) == cudaSuccess &&
                          cudaMallocHost(&pin[1], chunk) == cudaSuccess &&
                          cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming) == cudaSuccess &&
                          cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming) == cudaSuccess;
      rup.setup_secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
      if (pinned) {  // fill one buffer while the other copies
        for (size_t o = 0, i = 0; o < nb && e == cudaSuccess; o += chunk, i++) {
          const size_t m = std::min(chunk, nb - o);
          uint8_t *b = pin[i & 1];
          if (i >= 2) cudaEventSynchronize(done[i & 1]);
          {  // a few copy threads: one host thread alone cannot keep up with the DMA
            constexpr int kCp = 6;
            std::thread cp[kCp];
            for (int q = 0; q < kCp; q++)
              cp[q] = std::thread([=]() {
                std::memcpy(b + m * q / kCp, h->rslot.data() + o + m * q / kCp, m * (q + 1) / kCp - m * q / kCp);
              });
            for (auto &t : cp) t.join();
          }
          while (!rup.go.load()) std::this_thread::sleep_for(std::chrono::microseconds(200));
          if ((e = cudaMemcpyAsync(h->d_rslot + o, b, m, cudaMemcpyHostToDevice, st)) == cudaSuccess)
            e = cudaEventRecord(done[i & 1], st);
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      } else {
        while (!rup.go.load()) std::this_thread::sleep_for(std::chrono::microseconds(200));
        e = cudaMemcpy(h->d_rslot, h->rslot.data(), nb, cudaMemcpyHostToDevice);
      }
      for (int i = 0; i < 2; i++)
        if (done[i]) cudaEventDestroy(done[i]);
      if (pin[0] && pin[1] && !h->pin_rd[0]) {  // kept as the read-back staging
        h->pin_rd[0] = pin[0];
        h->pin_rd[1] = pin[1];
        h->pin_rd_bytes = chunk;
      } else {
        for (int i = 0; i < 2; i++)
          if (pin[i]) cudaFreeHost(pin[i]);
      }
      if (st) cudaStreamDestroy(st);
    });
  }

  h->entry_h = h->entry;

  trace("route upload started");
  if (h->ngroups > 0 && h->nv > (int32_t)kVidMask)
    return fail(h, TS_EINVAL, "too many vehicles for the row kernel");
  if (h->rvid_entries > INT32_MAX) return fail(h, TS_EINVAL, "network too large for one device");
  int rc;
  for (int b = 0; b < 2; b++) {  // device state (both buffers)
    if ((rc = dalloc(h, &h->d_code[b], h->gtiles.empty() ? 16 : h->gcells, 0xFF))) return rc;
    if ((rc = dalloc(h, &h->d_vid[b], h->gtiles.empty() ? 16 : h->gcells, 0xFF))) return rc;
    if ((rc = dalloc(h, &h->d_strip[b], std::max(1, h->nstrips), 0xFF))) return rc;
    if ((rc = dalloc(h, &h->d_planes[b], std::max<size_t>(16, group_plane_base(h->ngroups)), 0))) return rc;
    if ((rc = dalloc(h, &h->d_rvid[b], h->rvid_entries, 0xFF))) return rc;
    if ((rc = dalloc(h, &h->d_gcnt[b], std::max(1, h->ngroups), 0))) return rc;
    if (b == 0 && (rc = dalloc(h, &h->d_gctr, 1, 0))) return rc;
  }
  if (h->ngroups > 0 && (rc = upload(h, &h->d_gvoff, h->gvoff))) return rc;
  trace("device state");
  // the initial placement: row tiles built on the device (TSIM_HOST_INIT=1:
  // on the host, as are a doubly claimed cell's exact report and an
  // oversized row table)
  HostVec<int32_t> cur0 = filled<int32_t>(h->nv, 0);
  std::vector<uint8_t> gcode;
  std::vector<int32_t> gvid;
  h->n_placed = 0;
  rc = kPlaceHost;
  if (h->ngroups > 0 && getenv("TSIM_HOST_INIT") == nullptr) {
    rc = place_device(h, cur0, gcode, gvid);
    if (rc != TS_OK && rc != kPlaceHost) return rc;
  }
  if (rc == kPlaceHost) {
    h->n_placed = 0;
    if ((rc = place_host(h, cur0, gcode, gvid))) return rc;
  }
  rup.go = true;  // the route DMA may start
  trace("placement");
  // pending lists per first link in (departure, vid) order (R13)
  std::vector<int32_t> pend_off(h->nl + 1, 0), pend_list;
  auto mine = [&](int f) {  // pending vehicle whose entry cell this domain owns
    const int k = h->first_link[f];
    return !h->placed[f] && h->entry[f] >= h->own_lo[k] && h->entry[f] < h->own_hi[k];
  };
  // which vehicles are this domain's pending trips: flags in parallel, then
  // a counting sort by first link (input order kept, stable-sorted below)
  HostVec<uint8_t> pend_me(h->nv);
  parallel_for(h->nv, [&](int64_t lo, int64_t hi, int) {
    for (int64_t f = lo; f < hi; f++) pend_me[f] = mine((int)f) ? 1 : 0;
  });
  h->n_pending0 = 0;
  for (int f = 0; f < h->nv; f++)
    if (pend_me[f]) {
      pend_off[h->first_link[f] + 1]++;
      h->n_pending0++;
    }
  for (int k = 0; k < h->nl; k++) pend_off[k + 1] += pend_off[k];
  pend_list.assign(std::max(1, pend_off[h->nl]), 0);
  if (h->n_pending0 > 0) {
    std::vector<int32_t> fill(h->nl, 0);
    for (int f = 0; f < h->nv; f++)
      if (pend_me[f]) {
        int k = h->first_link[f];
        pend_list[pend_off[k] + fill[k]++] = f;
      }
    for (int k = 0; k < h->nl; k++)
      std::stable_sort(pend_list.begin() + pend_off[k], pend_list.begin() + pend_off[k + 1],
                       [&](int a, int b) { return h->dep[a] < h->dep[b] || (h->dep[a] == h->dep[b] && a < b); });
  }
  trace("pending lists");
  // a fresh start builds the per-vehicle words on the device (below)
  const bool dev_veh = h->arr0.empty() && h->nv > 0 && getenv("TSIM_HOST_INIT") == nullptr;
  HostVec<int32_t> inj, arr;
  if (!dev_veh) {
    inj.resize(h->nv);
    arr = filled<int32_t>(h->nv, -1);
    parallel_for(h->nv, [&](int64_t lo, int64_t hi, int) {
      for (int64_t f = lo; f < hi; f++) inj[f] = h->placed[f] ? INT_MIN : INT_MAX;
    });
  }
  h->n_arrived0 = 0;
  if (!h->arr0.empty()) {
    for (int f = 0; f < h->nv; f++) {
      arr[f] = h->arr0[f];
      if (arr[f] >= 0) cur0[f] = (int32_t)(h->roff[f + 1] - h->roff[f] - 1);  // on its final link
      if (arr[f] >= 0 && h->dom_me == 0) h->n_arrived0++;  // counted once over the domains
    }
  }
  std::vector<uint8_t> vmax8(h->nl);
  for (int k = 0; k < h->nl; k++) vmax8[k] = (uint8_t)h->vmax[k];
  // device
  if ((rc = setup_node_lanes(h))) return rc;
  trace("node lanes");
  if (h->ngroups > 0 && (rc = upload(h, &h->d_rows, h->rows))) return rc;  // node lanes resolved
  if ((rc = upload(h, &h->d_nli, h->nli))) return rc;
  if ((rc = upload(h, &h->d_nlo, h->nlo))) return rc;
  if ((rc = upload(h, &h->d_tiles, h->gtiles))) return rc;
  if (!h->gtiles.empty()) {
    CK(h, cudaMemcpyAsync(h->d_code[0], gcode.data(), gcode.size(), cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemcpyAsync(h->d_vid[0], gvid.data(), gvid.size() * 4, cudaMemcpyHostToDevice, h->stream));
  }
  trace("uploads");
  {  // injection scratch of the row kernel: needed only if a row link has pending trips
    bool need = false;
    for (size_t ti = 0; ti < h->tiles.size() && !need; ti++)
      if (h->tile_row[ti] >= 0 && pend_off[h->tiles[ti].link + 1] > pend_off[h->tiles[ti].link])
        need = true;
    if ((rc = dalloc(h, &h->d_inj_scratch, need ? h->rows.size() * kRowMaxCells : 16, 0xFF)))
      return rc;
  }
  if ((rc = upload(h, &h->d_halo_up, h->halo_up))) return rc;
  if ((rc = upload(h, &h->d_halo_dn, h->halo_dn))) return rc;
  if ((rc = upload(h, &h->d_vmax, vmax8))) return rc;
  if (h->ring_rows) h->tt[h->periodic] = 0u;  // straight on through the virtual nodes
  if ((rc = upload(h, &h->d_tt, h->tt))) return rc;
  if ((rc = upload(h, &h->d_out_pos, h->out_pos))) return rc;
  {  // routes as out-slot sequences: the upload started above
    rup.th.join();
    trace("route upload joined");
    if (trace.on)
      fprintf(stderr, "[tsim init]   (route upload took %.3f s, its pinned staging set up in %.3f s)\n",
              rup.secs, rup.setup_secs);
    if (rup.err != cudaSuccess)
      return fail(h, TS_EINTERNAL, "route upload: %s", cudaGetErrorString(rup.err));
    cudaGetLastError();
    std::vector<NodeOut> nodeout(h->out_list.size());
    for (size_t i = 0; i < h->out_list.size(); i++) {
      const int k = h->out_list[i];
      nodeout[i] = NodeOut{h->nlo[h->lgid[k]], (int16_t)h->lanes[k],
                           (int16_t)std::min(h->ncell[k], 32767), h->lane_row0[k]};
    }
    if ((rc = upload(h, &h->d_nodeout, h->ring_rows ? h->ring_nodeout : nodeout))) return rc;
  }
  trace("  node outs");
  if (dev_veh) {  // 12 bytes per vehicle cross PCIe instead of 24
    if (!h->d_roff && (rc = upload(h, &h->d_roff, h->roff))) return rc;
    trace("  route offsets up");
    if ((rc = dalloc(h, &h->d_vpos, h->nv))) return rc;
    if ((rc = dalloc(h, &h->d_inj, h->nv))) return rc;
    if ((rc = dalloc(h, &h->d_arr, h->nv))) return rc;
    trace("  vehicle arrays allocated");
    int32_t *d_cur = nullptr;
    uint8_t *d_placed = nullptr;
    CK(h, cudaMallocAsync(&d_cur, (size_t)h->nv * 4, h->stream));
    CK(h, cudaMallocAsync(&d_placed, (size_t)h->nv, h->stream));
    CK(h, cudaMemcpyAsync(d_cur, cur0.data(), (size_t)h->nv * 4, cudaMemcpyHostToDevice, h->stream));
    CK(h, cudaMemcpyAsync(d_placed, h->placed.data(), (size_t)h->nv, cudaMemcpyHostToDevice, h->stream));
    trace("  cursors up");
    k_init_vehicles<<<(h->nv + 255) / 256, 256, 0, h->stream>>>(h->nv, h->d_roff, d_cur, d_placed,
                                                                h->d_vpos, h->d_inj, h->d_arr);
    CK(h, cudaGetLastError());
    CK(h, cudaFreeAsync(d_cur, h->stream));
    CK(h, cudaFreeAsync(d_placed, h->stream));
  } else {
    HostVec<VehPos> vp(h->nv);
    parallel_for(h->nv, [&](int64_t lo, int64_t hi, int) {
      for (int64_t f = lo; f < hi; f++) vp[f] = VehPos{h->roff[f] + cur0[f], h->roff[f + 1]};
    });
    if ((rc = upload(h, &h->d_vpos, vp))) return rc;
    if ((rc = upload(h, &h->d_inj, inj))) return rc;
    if ((rc = upload(h, &h->d_arr, arr))) return rc;
  }
  trace("node outs + vehicle positions");
  if ((rc = upload(h, &h->d_dep, h->dep))) return rc;
  if ((rc = upload(h, &h->d_entry, h->entry))) return rc;
  if ((rc = upload(h, &h->d_pend_off, pend_off))) return rc;
  if ((rc = upload(h, &h->d_pend_list, pend_list))) return rc;
  {  // absolute head index into pend_list per link
    std::vector<int32_t> head(pend_off.begin(), pend_off.begin() + h->nl);
    if ((rc = upload(h, &h->d_pend_head, head))) return rc;
  }
  if ((rc = dalloc(h, &h->d_tail, h->n_nli, 0))) return rc;
  // entrant records start (and are reset to) all ones: vid 0xFFFFFFFF is
  // no vehicle, so a record never matches before it is written
  if ((rc = dalloc(h, &h->d_entr, h->n_nlo, 0xFF))) return rc;
  if ((rc = dalloc(h, &h->d_head, h->n_nlo, 0))) return rc;
  if ((rc = dalloc(h, &h->d_ext, h->n_nli, 0))) return rc;
  if ((rc = dalloc(h, &h->d_ext_row, (size_t)h->ngroups * 32 + 1, 0))) return rc;
  if ((rc = dalloc(h, &h->d_entr_row, (size_t)h->ngroups * 32 + 1, 0xFF))) return rc;
  if ((rc = dalloc(h, &h->d_stats, (size_t)kHist * ST_N, 0))) return rc;
  if ((rc = dalloc(h, &h->d_work, h->nl, 0))) return rc;
  if ((rc = dalloc(h, &h->d_node_work, h->nn, 0))) return rc;
  if ((rc = dalloc(h, &h->d_hash, 2, 0))) return rc;
  if ((rc = upload(h, &h->d_in_off, h->in_off))) return rc;
  if ((rc = upload(h, &h->d_in_list, h->in_list))) return rc;
  if ((rc = upload(h, &h->d_out_off, h->out_off))) return rc;
  if ((rc = upload(h, &h->d_out_list, h->out_list))) return rc;
  if ((rc = upload(h, &h->d_ncell, h->ncell))) return rc;
  if ((rc = upload(h, &h->d_lanes, h->lanes))) return rc;
  if ((rc = upload(h, &h->d_lgid, h->lgid))) return rc;
  if ((rc = upload(h, &h->d_cls, h->cls))) return rc;
  trace("routes + node tables");
  // launch geometry
  h->smem = h->lay.bytes;
  int wpb = std::max(1, std::min(8, (200 * 1024) / h->lay.bytes));
  h->threads = 32 * wpb;
  h->smem = wpb * h->lay.bytes;
  CK(h, set_smem_attrs(std::max(h->smem, 1)));
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->dev);
  int occ = std::max(1, occupancy_blocks(h->threads, h->smem));
  const int need = (int)((h->gtiles.size() + wpb - 1) / wpb);
  h->blocks = std::max(1, std::min(need, occ * nsm));
  // row kernel: one warp per 32-row group, 4 warps per block; each warp
  // stages its group's vid blocks (in + out) in shared memory
  // staging capacity per warp: 4 blocks of 4 warps per SM (128 registers)
  // leave ~55 KB of shared memory per block; group_cells overrides (tuning)
  h->rows_cap = h->cfg.group_cells > 0 ? (h->cfg.group_cells + 3) & ~3 : 1344;
  h->pdl = getenv("TSIM_NO_PDL") == nullptr;
  h->no_xoverlap = getenv("TSIM_NO_XOVERLAP") != nullptr;
  h->rows_threads = TS_ROWS_TPB;
  h->rows_smem = (h->rows_threads / 32) * rows_stage_words(h->rows_cap) * 4;
  CK(h, set_rows_smem(h->rows_smem));
  {  // persistent grid: every resident warp loops over groups
    const int wpb = h->rows_threads / 32;
    const int rocc = std::max(1, occupancy_rows(h->rows_threads, h->rows_smem));
    h->rows_blocks = std::max(1, std::min((h->ngroups + wpb - 1) / wpb, rocc * nsm));
  }
  if (!h->node_sig.empty() && (rc = upload(h, &h->d_node_sig, h->node_sig))) return rc;
  // the nodes of this domain (nodes are never split)
  h->my_nodes.clear();
  for (int nd = 0; nd < h->nn; nd++)
    if (h->dom_of_node[nd] == h->dom_me) h->my_nodes.push_back(nd);
  if ((rc = upload(h, &h->d_node_ids, h->my_nodes))) return rc;
  // exchange buffers: one contiguous segment of Strips per neighbour
  if (h->n_xs > 0) {
    std::vector<int32_t> ss, rs;
    for (const ts_sim::Nbr &nb : h->nbrs) {
      ss.insert(ss.end(), nb.send_slot.begin(), nb.send_slot.end());
      rs.insert(rs.end(), nb.recv_slot.begin(), nb.recv_slot.end());
    }
    if ((rc = upload(h, &h->d_send_slot, ss))) return rc;
    if ((rc = upload(h, &h->d_recv_slot, rs))) return rc;
    if ((rc = dalloc(h, &h->d_send, h->n_xs, 0xFF))) return rc;
    if ((rc = dalloc(h, &h->d_recv, h->n_xs, 0xFF))) return rc;
  }
  trace("launch geometry + node lanes");
  // S(t0) into buffer 1: the initial injection of departure <= t0 (O1
  // §Init), or (resume) a plain pass that writes strips and counters
  h->gcur = 0;
  h->rcur = 0;
  h->rows_s1 = false;
  h->gen_s1 = false;
  if (zero_stats(h, t0, 1)) return TS_EINTERNAL;
  int mode = (inject0 ? kModeInject : 0) | (base_mode(h) & kModeHash);
  StepParams P = step_params(h, t0 - 1, mode);
  if (h->ngroups > 0) {
    rows_launch(h, P);
    h->rcur ^= 1;
  }
  if (!h->gtiles.empty()) {
    launch_step(P, h->blocks, h->threads, h->smem, h->stream);
    h->gcur ^= 1;
  }
  CK(h, cudaGetLastError());
  h->t = t0;
  h->folded_t = t0;
  if (h->n_xs > 0) pack_strips(h);  // the caller exchanges, then ts_step_phase(h, 2, 0)
  CK(h, cudaStreamSynchronize(h->stream));
  unsigned long long st[ST_N];
  CK(h, cudaMemcpy(st, h->d_stats + (size_t)(t0 & (kHist - 1)) * ST_N, sizeof st, cudaMemcpyDeviceToHost));
  h->injected = (int64_t)st[ST_INJ];
  trace("initial kernels");
  // the host copies of the plans are no longer needed (all on the device)
  std::vector<uint8_t, UninitAlloc<uint8_t>>().swap(h->rslot);
  decltype(h->pl_vid)().swap(h->pl_vid);
  decltype(h->pl_cur)().swap(h->pl_cur);
  decltype(h->pl_lane)().swap(h->pl_lane);
  decltype(h->pl_cell)().swap(h->pl_cell);
  decltype(h->pl_v)().swap(h->pl_v);
  h->inited = true;
  trace("host plans freed");
  return TS_OK;
}

// --------------------------------------------------------------------- step
// strips of the boundary tiles -> send buffer (after k_lc / k_step)
static void pack_strips(ts_sim *h) {
  if (h->direct) return;  // delivered straight from the strip buffers (ts_local_step)
  launch_strip_copy(h->d_strip[h->gcur], h->d_send_slot, h->d_send, nullptr, h->n_xs, h->stream);
}
// receive buffer -> mirror strips, read as halos by the next kernel
static void unpack_strips(ts_sim *h, cudaStream_t st = nullptr) {
  if (h->direct) return;
  launch_strip_copy(h->d_recv, nullptr, h->d_strip[h->gcur], h->d_recv_slot, h->n_xs, st ? st : h->stream);
}

// Phase 0 of step t: lane change on S(t) (H1) of the
// general tiles and, unless already fused into the previous move, of the
// row tiles; pack exchange #1 (H2).
static void phase_lc(ts_sim *h) {
  const int t = h->t;
  if (!h->gtiles.empty() && !h->gen_s1) {
    launch_lc(step_params(h, t, 0), h->blocks, h->threads, h->smem, h->stream);
    h->gcur ^= 1;
  }
  if (h->ngroups > 0 && !h->rows_s1) {
    rows_launch(h, step_params(h, t, kModeLC | (h->ring_rows ? kModeHalo : 0)));
    h->rcur ^= 1;
  }
  h->gen_s1 = h->rows_s1 = true;
  if (h->n_xs > 0) pack_strips(h);
}

// Phase 1: intersections (H3), velocity update + move (H4/H5), injection
// (H6); with `more`, the lane change of step t+1 is fused into the move
// kernels whose tiles need no exchange for it.  Pack exchange #2 (H7).
// xside: exchange #1 and its unpack were enqueued on the side stream (native
// multi-rank step): only the general tiles read the mirror strips, so the
// node kernel and the row kernel run on the main stream meanwhile and the
// general-tile kernel follows the unpack on the side stream
static void phase_move(ts_sim *h, bool more, cudaEvent_t e0, cudaEvent_t e1, bool xside = false) {
  const int t = h->t;
  const int mode = base_mode(h);
  if (h->n_xs > 0 && !xside) unpack_strips(h);
  if (h->node_warp)
    launch_node_warp(node_params(h, t),
                     NodeWarpParams{h->d_lane_sig, h->d_nlanes, h->nchunks, h->d_nl_node,
                                    h->d_nl_row}, h->stream,
                     h->pdl);
  else
    launch_node(node_params(h, t), h->stream);
  // row tiles and general tiles are disjoint: with both present, the
  // general kernel runs on the side stream next to the row kernel
  const bool fork = h->ngroups > 0 && !h->gtiles.empty() && h->side;
  if (!h->gtiles.empty()) {
    const bool f = more && h->gfused;
    const StepParams gp = step_params(h, t, mode | (f ? kModeLC : 0));
    if (fork) {
      cudaEventRecord(h->ev_fork, h->stream);
      cudaStreamWaitEvent(h->side, h->ev_fork, 0);
      launch_step(gp, h->blocks, h->threads, h->smem, h->side);
      cudaEventRecord(h->ev_join, h->side);
    }
    h->gen_s1 = f;
    if (!fork) launch_step(gp, h->blocks, h->threads, h->smem, h->stream);
    h->gcur ^= 1;
  }
  if (e0) cudaEventRecord(e0, h->stream);
  if (h->ngroups > 0) {
    const bool f = more && h->rfused;
    rows_launch(h, step_params(h, t, mode | (f ? kModeLC : 0)), h->pdl && h->node_warp && !fork);
    h->rcur ^= 1;
    h->rows_s1 = f;
  }
  if (e1) cudaEventRecord(e1, h->stream);
  if (fork) cudaStreamWaitEvent(h->stream, h->ev_join, 0);
  h->t = t + 1;
  if (h->n_xs > 0) pack_strips(h);
}

constexpr int kTimingStride = 8;
// Steps are enqueued in blocks of at most kStepBlock: the per-step counters
// live in a ring of kHist slots, which must be folded into the host totals
// before a slot is reused (a longer run is finished block by block).
constexpr int kStepBlock = kHist / 2;
// steps per CUDA graph: odd, so that the row buffers return to their parity
// (one lane-change-only launch + kGraphSteps move launches flip them)
constexpr int kGraphSteps = 15;

// both tile kinds hold S(t) with its lane change pending (bits 1: rows, 2:
// general tiles; a kind without tiles counts as pending)
static int pending_lc(const ts_sim *h) {
  return ((h->ngroups == 0 || !h->rows_s1) ? 1 : 0) | ((h->gtiles.empty() || !h->gen_s1) ? 2 : 0);
}

// capture kGraphSteps steps from the current state (lane change of S(t)
// pending) into h->graph_exec; false if the capture is not possible
static int graph_key(const ts_sim *h) { return (h->rcur & 1) | ((h->gcur & 1) << 1); }

static bool capture_graph(ts_sim *h) {
  if (!h->d_clock && dalloc(h, &h->d_clock, 1, 0)) return false;
  const int key = graph_key(h);
  const int t0 = h->t, rc0 = h->rcur, gc0 = h->gcur;
  const bool rs0 = h->rows_s1, gs0 = h->gen_s1;
  const unsigned long long gb0 = h->gctr_base;
  h->capturing = true;
  h->graph_t0 = t0;
  h->gctr_base = 0;
  cudaGraph_t graph = nullptr;
  bool ok = cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    cudaMemsetAsync(h->d_gctr, 0, sizeof(unsigned long long), h->stream);
    launch_clock(h->d_clock, h->d_stats, kGraphSteps + 1, false, h->stream);
    for (int i = 0; i < kGraphSteps; i++) {
      phase_lc(h);
      phase_move(h, i < kGraphSteps - 1, nullptr, nullptr);
    }
    launch_clock(h->d_clock, h->d_stats, kGraphSteps, true, h->stream);
    const cudaError_t e = cudaStreamEndCapture(h->stream, &graph);
    ok = e == cudaSuccess && graph;
    if (!ok && getenv("TSIM_TRACE")) fprintf(stderr, "[tsim] end capture: %s\n", cudaGetErrorString(e));
  }
  const bool parity = h->rcur == rc0 && h->gcur == gc0 && pending_lc(h) == 3;
  if (!parity && getenv("TSIM_TRACE"))
    fprintf(stderr, "[tsim] graph parity: rcur %d->%d gcur %d->%d rows_s1 %d->%d gen_s1 %d->%d\n", rc0,
            h->rcur, gc0, h->gcur, rs0, h->rows_s1, gs0, h->gen_s1);
  ok = ok && parity;
  if (ok) {
    const cudaError_t e = cudaGraphInstantiate(&h->graph_exec[key], graph, 0);
    ok = e == cudaSuccess;
    if (!ok && getenv("TSIM_TRACE")) fprintf(stderr, "[tsim] instantiate: %s\n", cudaGetErrorString(e));
  }
  if (graph) cudaGraphDestroy(graph);
  h->graph_gctr_end[key] = h->gctr_base;
  h->capturing = false;
  h->t = t0;
  h->rcur = rc0;
  h->gcur = gc0;
  h->rows_s1 = rs0;
  h->gen_s1 = gs0;
  h->gctr_base = gb0;
  cudaGetLastError();  // a failed capture leaves no sticky error
  if (getenv("TSIM_TRACE"))
    fprintf(stderr, "[tsim] graph capture of %d steps at t=%d: %s\n", kGraphSteps, t0,
            ok ? "ok" : "failed (steps launched one by one)");
  if (!ok) {
    if (h->graph_exec[key]) cudaGraphExecDestroy(h->graph_exec[key]);
    h->graph_exec[key] = nullptr;
    h->graph_off = true;
  }
  return ok;
}

static int enqueue_steps(ts_sim *h, int32_t n) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "call ts_init first");
  if (n < 0) return fail(h, TS_EINVAL, "negative step count");
  if (h->n_xs > 0 && !h->comm)
    return fail(h, TS_EINVAL, "domain with neighbours: ts_nccl_init, or ts_step_phase and an exchange");
  if (n == 0) return TS_OK;
  if (n > kStepBlock) return fail(h, TS_EINTERNAL, "step block too long");
  CK(h, cudaSetDevice(h->dev));
  if (h->n_xs > 0) {  // whole steps with the native exchange (G1): LC, #1, move, #2
    if (zero_stats(h, h->t + 1, std::min(n + 1, kHist))) return TS_EINTERNAL;
    // both exchanges of every kTimingStride-th step are bracketed by events
    // (exchange time reported separately from the step, BASELINE config 5)
    const int nt = h->timing ? (n + kTimingStride - 1) / kTimingStride : 0;
    while ((int)h->mv_ev.size() < 4 * nt) {
      cudaEvent_t e;
      CK(h, cudaEventCreate(&e));
      h->mv_ev.push_back(e);
    }
    CK(h, cudaEventRecord(h->ev0, h->stream));
    int ne = 0;
    // exchange #1 overlaps the node and row kernels when the domain has
    // both kinds of tiles (the row tiles never read the strips)
    const bool xov = h->side && h->ngroups > 0 && !h->gtiles.empty() && !h->no_xoverlap;
    for (int i = 0; i < n; i++) {
      const bool tm = h->timing && i % kTimingStride == 0;
      phase_lc(h);
      const cudaStream_t xs = xov ? h->side : h->stream;
      if (xov) {
        CK(h, cudaEventRecord(h->ev_lc, h->stream));
        CK(h, cudaStreamWaitEvent(h->side, h->ev_lc, 0));
      }
      if (tm) CK(h, cudaEventRecord(h->mv_ev[2 * ne], xs));
      if (int rc = nccl_exchange(h, xs)) return rc;
      if (tm) CK(h, cudaEventRecord(h->mv_ev[2 * ne + 1], xs));
      ne += tm;
      if (xov) unpack_strips(h, h->side);
      phase_move(h, i < n - 1, nullptr, nullptr, xov);
      if (tm) CK(h, cudaEventRecord(h->mv_ev[2 * ne], h->stream));
      if (int rc = nccl_exchange(h)) return rc;
      if (tm) CK(h, cudaEventRecord(h->mv_ev[2 * ne + 1], h->stream));
      ne += tm;
      unpack_strips(h);
    }
    CK(h, cudaEventRecord(h->ev1, h->stream));
    CK(h, cudaGetLastError());
    h->last_move_launches = 0;
    h->last_xchg_n = ne;
    return TS_OK;
  }
  // TS_FLAG_GRAPH: whole kGraphSteps blocks of steps replay one CUDA graph
  int reps = 0;
  if ((h->cfg.flags & TS_FLAG_GRAPH) && !h->graph_off && n >= kGraphSteps && pending_lc(h) == 3 &&
      (h->graph_exec[graph_key(h)] || capture_graph(h)))
    reps = n / kGraphSteps;
  CK(h, cudaEventRecord(h->ev0, h->stream));
  if (reps) {
    CK(h, cudaMemcpyAsync(h->d_clock, &h->t, sizeof(int32_t), cudaMemcpyHostToDevice, h->stream));
    const int key = graph_key(h);  // the buffer parity is the same after every replay
    for (int r = 0; r < reps; r++) CK(h, cudaGraphLaunch(h->graph_exec[key], h->stream));
    h->t += reps * kGraphSteps;
    h->gctr_base = h->graph_gctr_end[key];
    n -= reps * kGraphSteps;
  }
  if (n > 0 && zero_stats(h, h->t + 1, std::min(n + 1, kHist))) return TS_EINTERNAL;
  if ((int)h->mv_ev.size() < 2 * n && h->timing) {
    while ((int)h->mv_ev.size() < 2 * n) {
      cudaEvent_t e;
      CK(h, cudaEventCreate(&e));
      h->mv_ev.push_back(e);
    }
  }
  // the move kernel is timed on every kTimingStride-th step only: events
  // between two kernels would serialise their programmatic overlap
  int ns = 0;
  for (int i = 0; i < n; i++) {
    phase_lc(h);
    const bool tm = h->timing && i % kTimingStride == 0;
    phase_move(h, i < n - 1, tm ? h->mv_ev[2 * ns] : nullptr, tm ? h->mv_ev[2 * ns + 1] : nullptr);
    ns += tm;
  }
  CK(h, cudaEventRecord(h->ev1, h->stream));
  CK(h, cudaGetLastError());
  h->last_move_launches = ns;
  h->last_xchg_n = 0;
  return TS_OK;
}

// fold the per-step counters of steps whose result time is in
// (folded_t, t] into the host totals
int fold_stats(ts_sim *h) {
  const int n = h->t - h->folded_t;
  if (n <= 0) return TS_OK;
  if (n < kHist) {
    std::vector<unsigned long long> st((size_t)kHist * ST_N);
    CK(h, cudaMemcpy(st.data(), h->d_stats, st.size() * 8, cudaMemcpyDeviceToHost));
    for (int tt = h->folded_t + 1; tt <= h->t; tt++) {
      const unsigned long long *a = &st[(size_t)(tt & (kHist - 1)) * ST_N];
      const unsigned long long *p = &st[(size_t)((tt - 1) & (kHist - 1)) * ST_N];
      h->veh_updates += (int64_t)p[ST_ACTIVE];
      h->arrived += (int64_t)a[ST_ARR];
      h->injected += (int64_t)a[ST_INJ];
    }
  }
  h->folded_t = h->t;
  return TS_OK;
}

static int finish_steps(ts_sim *h) {
  CK(h, cudaStreamSynchronize(h->stream));
  float ms = 0;
  CK(h, cudaEventElapsedTime(&ms, h->ev0, h->ev1));
  h->last_total_ms = ms;
  h->busy_ms += ms;
  double mv = 0;
  if (h->timing)
    for (int i = 0; i < h->last_move_launches; i++) {
      float m = 0;
      CK(h, cudaEventElapsedTime(&m, h->mv_ev[2 * i], h->mv_ev[2 * i + 1]));
      mv += m;
    }
  h->last_move_ms = mv;
  double xm = 0;
  for (int64_t i = 0; i < h->last_xchg_n; i++) {
    float m = 0;
    CK(h, cudaEventElapsedTime(&m, h->mv_ev[2 * i], h->mv_ev[2 * i + 1]));
    xm += m;
  }
  h->last_xchg_ms = xm;
  return fold_stats(h);
}

struct StepTotals {
  double ms = 0, move_ms = 0, xchg_ms = 0;
  int64_t move_launches = 0, xchg_n = 0;
  void add(const ts_sim *h) {
    ms += h->last_total_ms;
    move_ms += h->last_move_ms;
    xchg_ms += h->last_xchg_ms;
    move_launches += h->last_move_launches;
    xchg_n += h->last_xchg_n;
  }
  void store(ts_sim *h) const {
    h->last_total_ms = ms;
    h->last_move_ms = move_ms;
    h->last_xchg_ms = xchg_ms;
    h->last_move_launches = move_launches;
    h->last_xchg_n = xchg_n;
  }
};

// run all but the last block of n steps to completion (totals in *acc);
// returns the size of the last block, or < 0 on error
static int run_leading_blocks(ts_sim *h, int32_t n, StepTotals *acc) {
  while (n > kStepBlock) {
    if (int rc = enqueue_steps(h, kStepBlock)) return -rc;
    if (int rc = finish_steps(h)) return -rc;
    acc->add(h);
    n -= kStepBlock;
  }
  return n;
}

int ts_step(ts_sim *h, int32_t n_steps) {
  if (!h) return TS_EINVAL;
  if (n_steps < 0) return fail(h, TS_EINVAL, "negative step count");
  StepTotals acc;
  const int last = run_leading_blocks(h, n_steps, &acc);
  if (last < 0) return -last;
  if (int rc = enqueue_steps(h, last)) return rc;
  if (n_steps == 0) return TS_OK;
  if (last > 0) {
    if (int rc = finish_steps(h)) return rc;
    acc.add(h);
  }
  acc.store(h);
  return TS_OK;
}

// asynchronous steps: per-handle state (several handles may interleave);
// a run longer than kStepBlock finishes its leading blocks before returning
int ts_step_async(ts_sim *h, int32_t n_steps) {
  if (!h) return TS_EINVAL;
  if (h->async_n > 0) return fail(h, TS_EINVAL, "ts_step_async: previous steps not synced");
  if (n_steps < 0) return fail(h, TS_EINVAL, "negative step count");
  StepTotals acc;
  const int last = run_leading_blocks(h, n_steps, &acc);
  if (last < 0) return -last;
  h->async_ms = acc.ms;
  h->async_move_ms = acc.move_ms;
  h->async_move_launches = acc.move_launches;
  h->async_from = h->t;
  if (int rc = enqueue_steps(h, last)) return rc;
  h->async_n = last;
  return TS_OK;
}

int ts_sync(ts_sim *h) {
  if (!h) return TS_EINVAL;
  CK(h, cudaSetDevice(h->dev));
  if (h->async_n > 0) {
    h->async_n = 0;
    if (int rc = finish_steps(h)) return rc;
    h->last_total_ms += h->async_ms;
    h->last_move_ms += h->async_move_ms;
    h->last_move_launches += h->async_move_launches;
    h->async_ms = h->async_move_ms = 0;
    h->async_move_launches = 0;
    return TS_OK;
  }
  CK(h, cudaStreamSynchronize(h->stream));
  return fold_stats(h);
}

static int fold_busy(ts_sim *h) {
  if (h->ph_used == 0) return TS_OK;
  CK(h, cudaStreamSynchronize(h->stream));
  for (size_t i = 0; i + 1 < h->ph_used; i += 2) {
    float m = 0;
    CK(h, cudaEventElapsedTime(&m, h->ph_ev[i], h->ph_ev[i + 1]));
    h->busy_ms += m;
  }
  h->ph_used = 0;
  return TS_OK;
}

int ts_busy_time(ts_sim *h, double *ms) {
  if (!h || !h->inited || !ms) return TS_EINVAL;
  CK(h, cudaSetDevice(h->dev));
  if (int rc = fold_busy(h)) return rc;
  *ms = h->busy_ms;
  h->busy_ms = 0;
  return TS_OK;
}

int ts_step_phase(ts_sim *h, int32_t phase, int32_t more) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "call ts_init first");
  CK(h, cudaSetDevice(h->dev));
  if (h->ph_used >= 8192)
    if (int rc = fold_busy(h)) return rc;
  while (h->ph_ev.size() < h->ph_used + 2) {
    cudaEvent_t e;
    CK(h, cudaEventCreate(&e));
    h->ph_ev.push_back(e);
  }
  CK(h, cudaEventRecord(h->ph_ev[h->ph_used], h->stream));
  switch (phase) {
    case 0:
      if (h->t + 1 - h->folded_t >= kStepBlock) {  // fold before the stats ring wraps
        CK(h, cudaStreamSynchronize(h->stream));
        if (int rc = fold_stats(h)) return rc;
      }
      if (zero_stats(h, h->t + 1, 1)) return TS_EINTERNAL;
      phase_lc(h);
      break;
    case 1:
      if (!h->gen_s1 || !h->rows_s1) return fail(h, TS_EINVAL, "phase 1 before phase 0");
      phase_move(h, more != 0, nullptr, nullptr);
      break;
    case 2:
      if (h->n_xs > 0) unpack_strips(h);
      break;
    default:
      return fail(h, TS_EINVAL, "phase must be 0, 1 or 2");
  }
  CK(h, cudaEventRecord(h->ph_ev[h->ph_used + 1], h->stream));
  h->ph_used += 2;
  CK(h, cudaGetLastError());
  return TS_OK;
}

int ts_exchange_plan(const ts_sim *h, int32_t cap, int32_t *nbr_dom, int64_t *nbr_strips,
                     int64_t *nbr_off, int32_t *n_out) {
  if (!h || !h->inited || !n_out) return TS_EINVAL;
  const int32_t m = (int32_t)h->nbrs.size();
  for (int32_t i = 0; i < m && i < cap; i++) {
    if (nbr_dom) nbr_dom[i] = h->nbrs[i].dom;
    if (nbr_strips) nbr_strips[i] = (int64_t)h->nbrs[i].send_slot.size();
    if (nbr_off) nbr_off[i] = h->nbrs[i].off;
  }
  *n_out = m;
  return TS_OK;
}

int ts_exchange_buffers(ts_sim *h, void **send_dev, void **recv_dev) {
  if (!h || !h->inited) return TS_EINVAL;
  if (send_dev) *send_dev = h->d_send;
  if (recv_dev) *recv_dev = h->d_recv;
  return TS_OK;
}

int32_t ts_strip_bytes(void) { return (int32_t)sizeof(Strip); }

void *ts_stream(const ts_sim *h) { return h ? (void *)h->stream : nullptr; }

// in-process exchange between the domains of one partition (all handles of
// the same k-way partition, any devices): every send segment is copied into
// the partner's receive segment, ordered after the sender's pack and before
// the receiver's unpack by events
// the exchange among the handles of one partition, by_dom[d] = domain d:
// every send segment into its partner's receive segment (device copies,
// peer copies across devices), ordered by the handles' reusable events
static int exchange_local_enqueue(const std::vector<ts_sim *> &by_dom) {
  const int k = (int)by_dom.size();
  // ordering by each handle's reusable events: the receivers' copies wait
  // for their senders' packs; the senders' next work waits for the copies
  for (int i = 0; i < k; i++) {
    ts_sim *a = by_dom[i];
    if (!a) return TS_EINVAL;  // checked by by_domain
    CK(a, cudaSetDevice(a->dev));
    CK(a, cudaEventRecord(a->ev_packed, a->stream));
  }
  for (int i = 0; i < k; i++) {
    ts_sim *b = by_dom[i];  // receiver
    CK(b, cudaSetDevice(b->dev));
    for (const ts_sim::Nbr &nb : b->nbrs) {
      ts_sim *a = by_dom[nb.dom];
      const ts_sim::Nbr *back = nullptr;
      for (const ts_sim::Nbr &x : a->nbrs)
        if (x.dom == b->dom_me) back = &x;
      if (!back || back->send_slot.size() != nb.recv_slot.size())
        return fail(b, TS_EINTERNAL, "exchange plans of domains %d and %d disagree", a->dom_me,
                    b->dom_me);
      CK(b, cudaStreamWaitEvent(b->stream, a->ev_packed, 0));
      CK(b, cudaMemcpyPeerAsync(b->d_recv + nb.off, b->dev, a->d_send + back->off, a->dev,
                                nb.recv_slot.size() * sizeof(Strip), b->stream));
    }
  }
  // a sender may not overwrite its send buffer before the receivers copied
  for (int i = 0; i < k; i++) {
    ts_sim *b = by_dom[i];
    CK(b, cudaSetDevice(b->dev));
    CK(b, cudaEventRecord(b->ev_copied, b->stream));
    for (const ts_sim::Nbr &nb : b->nbrs) {
      ts_sim *a = by_dom[nb.dom];
      CK(a, cudaSetDevice(a->dev));
      CK(a, cudaStreamWaitEvent(a->stream, b->ev_copied, 0));
    }
  }
  return TS_OK;
}


// the k handles of one partition indexed by domain (TS_EINVAL otherwise)
static int by_domain(ts_sim **hs, int32_t k, std::vector<ts_sim *> &by_dom) {
  if (!hs || k < 1) return TS_EINVAL;
  by_dom.assign(k, nullptr);
  for (int i = 0; i < k; i++) {
    if (!hs[i] || !hs[i]->inited || hs[i]->dom_k != k || by_dom[hs[i]->dom_me])
      return hs[i] ? fail(hs[i], TS_EINVAL, "not the %d initialised domains of one partition", k)
                   : TS_EINVAL;
    by_dom[hs[i]->dom_me] = hs[i];
  }
  return TS_OK;
}

int ts_exchange_local(ts_sim **hs, int32_t k) {
  std::vector<ts_sim *> by_dom;
  if (int rc = by_domain(hs, k, by_dom)) return rc;
  return exchange_local_enqueue(by_dom);
}

// direct exchange plans of in-process partitions: per partition (handle
// set), every (sender, its strip slot) -> (receiver, mirror slot), grouped
// by the receiver's device.  One kernel per receiving device pulls its
// receivers' strips straight from the senders' strip buffers -- over
// NVLink through peer pointers (UVA) when a sender is on another device --
// ordered after every domain's last work and before its next by events.
// TSIM_DIRECT_SPLIT=1 groups by receiving handle instead (one kernel per
// domain: the multi-device structure exercised on one device, tests).
struct DirectPlan {
  struct Sub {
    ts_sim *rep;  // a receiving handle on the group's device: stream, events, plan memory
    int4 *d_plan = nullptr;
    int64_t n = 0;
  };
  std::vector<ts_sim *> ds;
  std::vector<Sub> subs;
};
static std::vector<DirectPlan> g_direct_plans;

static const DirectPlan *direct_plan(const std::vector<ts_sim *> &ds) {
  for (const DirectPlan &p : g_direct_plans)
    if (p.ds == ds) return &p;
  if ((int)ds.size() > kDirectMax) return nullptr;
  const bool split = getenv("TSIM_DIRECT_SPLIT") != nullptr;
  // peer access from every receiving device to every sending device
  for (ts_sim *b : ds)
    for (const ts_sim::Nbr &nb : b->nbrs) {
      ts_sim *a = ds[nb.dom];
      if (a->dev == b->dev) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, b->dev, a->dev) != cudaSuccess || !can) return nullptr;
      if (cudaSetDevice(b->dev) != cudaSuccess) return nullptr;
      const cudaError_t e = cudaDeviceEnablePeerAccess(a->dev, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return nullptr;
      cudaGetLastError();
    }
  DirectPlan p;
  p.ds = ds;
  std::vector<std::vector<int4>> plans;
  for (size_t bi = 0; bi < ds.size(); bi++) {
    ts_sim *b = ds[bi];
    size_t g = 0;  // the receiver's group
    while (g < p.subs.size() && (split ? p.subs[g].rep != b : p.subs[g].rep->dev != b->dev)) g++;
    if (g == p.subs.size()) {
      p.subs.push_back(DirectPlan::Sub{b});
      plans.emplace_back();
    }
    for (const ts_sim::Nbr &nb : b->nbrs) {
      ts_sim *a = ds[nb.dom];
      const ts_sim::Nbr *back = nullptr;
      for (const ts_sim::Nbr &x : a->nbrs)
        if (x.dom == b->dom_me) back = &x;
      if (!back || back->send_slot.size() != nb.recv_slot.size()) return nullptr;
      for (size_t j = 0; j < nb.recv_slot.size(); j++)
        plans[g].push_back(int4{nb.dom, back->send_slot[j], (int)bi, nb.recv_slot[j]});
    }
  }
  for (size_t g = 0; g < p.subs.size(); g++) {
    DirectPlan::Sub &sb = p.subs[g];
    sb.n = (int64_t)plans[g].size();
    // owned by the group's handle (freed with it; the plan is dropped then)
    if (!plans[g].empty() &&
        (cudaSetDevice(sb.rep->dev) != cudaSuccess || upload(sb.rep, &sb.d_plan, plans[g])))
      return nullptr;
  }
  g_direct_plans.push_back(p);
  return &g_direct_plans.back();
}

static void drop_direct_plans(const ts_sim *h) {
  for (size_t i = 0; i < g_direct_plans.size();) {
    if (std::find(g_direct_plans[i].ds.begin(), g_direct_plans[i].ds.end(), h) !=
        g_direct_plans[i].ds.end())
      g_direct_plans.erase(g_direct_plans.begin() + i);
    else
      i++;
  }
}

// the exchange as one kernel per receiving device, after every domain's
// last work and before its next (the strips of the handles' current buffers)
static int exchange_direct_enqueue(const std::vector<ts_sim *> &ds, const DirectPlan &pl) {
  DirectParams P{};
  for (size_t i = 0; i < ds.size(); i++) {
    P.src[i] = ds[i]->d_strip[ds[i]->gcur];
    P.dst[i] = ds[i]->d_strip[ds[i]->gcur];
    CK(ds[i], cudaSetDevice(ds[i]->dev));
    CK(ds[i], cudaEventRecord(ds[i]->ev_packed, ds[i]->stream));
  }
  for (const DirectPlan::Sub &sb : pl.subs) {
    ts_sim *r = sb.rep;
    CK(r, cudaSetDevice(r->dev));
    for (ts_sim *h : ds)
      if (h != r) CK(r, cudaStreamWaitEvent(r->stream, h->ev_packed, 0));
    P.plan = sb.d_plan;
    P.n = sb.n;
    launch_strip_direct(P, r->stream);
    CK(r, cudaEventRecord(r->ev_copied, r->stream));
  }
  for (ts_sim *h : ds) {
    CK(h, cudaSetDevice(h->dev));
    for (const DirectPlan::Sub &sb : pl.subs)
      if (sb.rep != h) CK(h, cudaStreamWaitEvent(h->stream, sb.rep->ev_copied, 0));
  }
  return TS_OK;
}

// one whole step of all domains: lane change + pack #1,
// exchange, unpack + intersections + move + injection + pack #2, exchange,
// unpack; every phase of a domain bracketed by its busy-time events unless
// capturing
static int local_step_enqueue(const std::vector<ts_sim *> &ds, bool more,
                              const DirectPlan *dp = nullptr) {
  auto exchange = [&]() { return dp ? exchange_direct_enqueue(ds, *dp) : exchange_local_enqueue(ds); };
  auto timed = [&](ts_sim *h, auto &&fn) -> int {
    const bool ev = !h->capturing;
    if (ev) {
      if (h->ph_used >= 8192)
        if (int rc = fold_busy(h)) return rc;
      while (h->ph_ev.size() < h->ph_used + 2) {
        cudaEvent_t e;
        CK(h, cudaEventCreate(&e));
        h->ph_ev.push_back(e);
      }
      CK(h, cudaEventRecord(h->ph_ev[h->ph_used], h->stream));
    }
    fn();
    if (ev) {
      CK(h, cudaEventRecord(h->ph_ev[h->ph_used + 1], h->stream));
      h->ph_used += 2;
    }
    return TS_OK;
  };
  for (ts_sim *h : ds) {
    CK(h, cudaSetDevice(h->dev));
    if (int rc = timed(h, [&]() { phase_lc(h); })) return rc;
  }
  if (int rc = exchange()) return rc;
  for (ts_sim *h : ds) {
    CK(h, cudaSetDevice(h->dev));
    if (int rc = timed(h, [&]() { phase_move(h, more, nullptr, nullptr); })) return rc;
  }
  if (int rc = exchange()) return rc;
  for (ts_sim *h : ds) {
    CK(h, cudaSetDevice(h->dev));
    if (int rc = timed(h, [&]() {
          if (h->n_xs > 0) unpack_strips(h);
        }))
      return rc;
  }
  return TS_OK;
}

// capture kGraphSteps steps of all domains into one CUDA graph (the
// domains' streams forked from / joined into domain 0's stream); false if
// the capture is not possible
struct LocalGraph {
  std::vector<ts_sim *> ds;
  cudaGraphExec_t exec = nullptr;
  int key = -1;
  std::vector<unsigned long long> gctr_end;
};
static std::vector<LocalGraph> g_local_graphs;  // per partition (handle set) and parity

// a destroyed handle's graphs go with it (their nodes use its buffers)
static void drop_local_graphs(const ts_sim *h) {
  for (size_t i = 0; i < g_local_graphs.size();) {
    LocalGraph &g = g_local_graphs[i];
    if (std::find(g.ds.begin(), g.ds.end(), h) != g.ds.end()) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g_local_graphs.erase(g_local_graphs.begin() + i);
    } else {
      i++;
    }
  }
}

static bool capture_local(std::vector<ts_sim *> &ds, LocalGraph &lg, const DirectPlan *dp) {
  ts_sim *h0 = ds[0];
  struct Saved {
    int32_t t;
    int rcur, gcur;
    bool rs, gs;
    unsigned long long gb;
  };
  std::vector<Saved> sv;
  for (ts_sim *h : ds) {
    if (!h->d_clock && dalloc(h, &h->d_clock, 1, 0)) return false;
    sv.push_back(Saved{h->t, h->rcur, h->gcur, h->rows_s1, h->gen_s1, h->gctr_base});
  }
  cudaGraph_t graph = nullptr;
  bool ok = cudaStreamBeginCapture(h0->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    cudaEventRecord(h0->ev_packed, h0->stream);  // fork every domain's stream into the capture
    for (ts_sim *h : ds) {
      if (h != h0) cudaStreamWaitEvent(h->stream, h0->ev_packed, 0);
      h->capturing = true;
      h->graph_t0 = h->t;
      h->gctr_base = 0;
      cudaMemsetAsync(h->d_gctr, 0, sizeof(unsigned long long), h->stream);
      launch_clock(h->d_clock, h->d_stats, kGraphSteps + 1, false, h->stream);
    }
    for (int i = 0; i < kGraphSteps && ok; i++)
      ok = local_step_enqueue(ds, i < kGraphSteps - 1, dp) == TS_OK;
    for (ts_sim *h : ds) {
      launch_clock(h->d_clock, h->d_stats, kGraphSteps, true, h->stream);
      if (h != h0) {  // join
        cudaEventRecord(h->ev_copied, h->stream);
        cudaStreamWaitEvent(h0->stream, h->ev_copied, 0);
      }
    }
    const cudaError_t e = cudaStreamEndCapture(h0->stream, &graph);
    ok = ok && e == cudaSuccess && graph;
    if (!ok && getenv("TSIM_TRACE")) fprintf(stderr, "[tsim] local capture: %s\n", cudaGetErrorString(e));
  }
  for (size_t i = 0; i < ds.size(); i++) {
    ts_sim *h = ds[i];
    ok = ok && h->rcur == sv[i].rcur && h->gcur == sv[i].gcur && pending_lc(h) == 3;
    lg.gctr_end.push_back(h->gctr_base);
    h->capturing = false;
    h->t = sv[i].t;
    h->rcur = sv[i].rcur;
    h->gcur = sv[i].gcur;
    h->rows_s1 = sv[i].rs;
    h->gen_s1 = sv[i].gs;
    h->gctr_base = sv[i].gb;
  }
  if (ok) ok = cudaGraphInstantiate(&lg.exec, graph, 0) == cudaSuccess;
  if (graph) cudaGraphDestroy(graph);
  cudaGetLastError();
  if (getenv("TSIM_TRACE"))
    fprintf(stderr, "[tsim] local graph capture of %d steps, %zu domains: %s\n", kGraphSteps, ds.size(),
            ok ? "ok" : "failed (steps launched one by one)");
  return ok;
}

int ts_local_step(ts_sim **hs, int32_t k, int32_t n_steps) {
  std::vector<ts_sim *> ds;
  if (int rc = by_domain(hs, k, ds)) return rc;
  if (n_steps < 0) return fail(ds[0], TS_EINVAL, "negative step count");
  // the strips go straight from the senders' to the receivers' strip
  // buffers, one kernel per receiving device and exchange (peer pointers
  // across devices; TSIM_LOCAL_COPIES=1 or no peer access: device / peer
  // copies)
  const DirectPlan *dp = getenv("TSIM_LOCAL_COPIES") ? nullptr : direct_plan(ds);
  struct DirectGuard {
    std::vector<ts_sim *> &ds;
    ~DirectGuard() {
      for (ts_sim *h : ds) h->direct = false;
    }
  } guard{ds};
  for (ts_sim *h : ds) h->direct = dp != nullptr;
  bool graph = true;
  for (ts_sim *h : ds) {
    if (h->comm) return fail(h, TS_EINVAL, "a domain with a native communicator");
    if (pending_lc(h) != 3) return fail(h, TS_EINVAL, "domain in the middle of a step");
    if (h->t != ds[0]->t) return fail(h, TS_EINVAL, "domains at different times");
    graph = graph && (h->cfg.flags & TS_FLAG_GRAPH) && !h->graph_off && h->dev == ds[0]->dev;
  }
  while (n_steps > 0) {
    const int32_t m = std::min<int32_t>(n_steps, kStepBlock);
    for (ts_sim *h : ds) {
      CK(h, cudaSetDevice(h->dev));
      if (zero_stats(h, h->t + 1, std::min(m + 1, kHist))) return TS_EINTERNAL;
    }
    int done = 0;
    if (graph && m >= kGraphSteps) {  // whole blocks replay one graph of all domains
      int key = 0;
      for (size_t i = 0; i < ds.size(); i++) key |= (graph_key(ds[i]) << (2 * (i % 16)));
      LocalGraph *lg = nullptr;
      for (LocalGraph &x : g_local_graphs)
        if (x.ds == ds && x.key == key) lg = &x;
      if (!lg) {
        LocalGraph nl;
        nl.ds = ds;
        nl.key = key;
        if (capture_local(ds, nl, dp)) {
          g_local_graphs.push_back(nl);
          lg = &g_local_graphs.back();
        } else {
          for (ts_sim *h : ds) h->graph_off = true;
          graph = false;
        }
      }
      if (lg) {
        const int reps = m / kGraphSteps;
        ts_sim *h0 = ds[0];
        CK(h0, cudaSetDevice(h0->dev));
        for (ts_sim *h : ds) {  // clocks, after each domain's previous work
          CK(h0, cudaEventRecord(h->ev_packed, h->stream));
          CK(h0, cudaStreamWaitEvent(h0->stream, h->ev_packed, 0));
          CK(h0, cudaMemcpyAsync(h->d_clock, &h->t, sizeof(int32_t), cudaMemcpyHostToDevice, h0->stream));
        }
        for (int r = 0; r < reps; r++) CK(h0, cudaGraphLaunch(lg->exec, h0->stream));
        CK(h0, cudaEventRecord(h0->ev_copied, h0->stream));
        for (size_t i = 0; i < ds.size(); i++) {
          ts_sim *h = ds[i];
          CK(h, cudaStreamWaitEvent(h->stream, h0->ev_copied, 0));  // later work after the graph
          h->t += reps * kGraphSteps;
          h->gctr_base = lg->gctr_end[i];
        }
        done = reps * kGraphSteps;
        CK(h0, cudaStreamSynchronize(h0->stream));  // the host clock values were read
      }
    }
    for (int i = done; i < m; i++)
      if (int rc = local_step_enqueue(ds, i < m - 1, dp)) return rc;
    for (ts_sim *h : ds) {
      CK(h, cudaSetDevice(h->dev));
      CK(h, cudaStreamSynchronize(h->stream));
      if (int rc = fold_stats(h)) return rc;
    }
    n_steps -= m;
  }
  return TS_OK;
}

int32_t ts_time(const ts_sim *h) { return h ? h->t : -1; }

}  // extern "C"
