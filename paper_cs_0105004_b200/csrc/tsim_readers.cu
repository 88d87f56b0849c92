// tsim_readers.cu -- host side of libtsim: read-back of the simulation
// state (vehicles, cells, hashes, history, totals, timings) and the ORB /
// work-weighted partition entry points.  C-ABI declared in include/tsim.h.
#include "tsim_host.h"

// ------------------------------------------------- device-side read-back
// Per-vehicle state gathered on the device (single-domain handles): every
// vehicle found in the row planes / vid blocks or the general tiles writes
// its link, lane, cell, velocity by vid and counts itself in `seen` (a
// count > 1 is a corrupt state); then one thread per vehicle derives
// status, route cursor and arrival time.  Only the caller's arrays cross
// PCIe.
struct ReadOut {
  int32_t *link, *lane, *cell, *v;
  uint32_t *seen;
};

__global__ void __launch_bounds__(128) k_read_rows(const RowsParams R, ReadOut o) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = gid >> 5, lane = gid & 31;
  const bool act = g < R.ngroups;
  const uint32_t *pl = R.planes_in + group_plane_base(act ? g : 0) + lane;
  int n = 0;
  uint32_t O[kRowWords];
  for (int i = 0; i < kRowWords; i++) {
    O[i] = act ? pl[i * 32] : 0u;
    n += __popc(O[i]);
  }
  int off = n;  // exclusive warp prefix of the row counts
  for (int d = 1; d < 32; d <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, off, d);
    if (lane >= d) off += y;
  }
  off -= n;
  if (!act || n == 0) return;
  const RowDesc rd = R.rows[gid];
  const int a = R.row_a ? R.row_a[gid] : 0;
  const int32_t *lst = R.vid_in + R.gvoff[g] + off;
  int k = 0;
  for (int i = 0; i < kRowWords; i++) {
    uint32_t m = O[i];
    while (m) {
      const int x = __ffs(m) - 1;
      m &= m - 1u;
      const int v = (int)((pl[(kRowWords + i) * 32] >> x) & 1u) |
                    (int)(((pl[(2 * kRowWords + i) * 32] >> x) & 1u) << 1) |
                    (int)(((pl[(3 * kRowWords + i) * 32] >> x) & 1u) << 2);
      const int f = (int)((uint32_t)lst[k++] & kVidMask);
      atomicAdd(o.seen + f, 1u);
      o.link[f] = rd.link;
      o.lane[f] = rd.l;
      o.cell[f] = a + 32 * i + x;
      o.v[f] = v;
    }
  }
}

// general tiles: one thread per lane of a tile (byte codes, per-lane lists)
__global__ void __launch_bounds__(128) k_read_tiles(const TileDesc *tiles, int ntiles,
                                                    const uint8_t *code, const int32_t *vid,
                                                    ReadOut o) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int ti = (int)(i >> 3), l = (int)(i & 7);
  if (ti >= ntiles) return;
  const TileDesc d = tiles[ti];
  if (l >= d.L) return;
  const int Wp = row_pitch(d.w);
  const int64_t rb = d.off + (int64_t)l * Wp;
  int64_t r = rb;
  for (int x = 0; x < d.w; x++) {
    const uint8_t c = code[rb + x];
    if (c & 0x80) continue;
    const int f = vid[r++];
    atomicAdd(o.seen + f, 1u);
    o.link[f] = d.link;
    o.lane[f] = l;
    o.cell[f] = d.a + x;
    o.v[f] = c & 7;
  }
}

// per vehicle: status / cursor / arrival (single domain); bad[0] = the
// smallest vid seen twice, bad[1] = the smallest vid that is nowhere
__global__ void __launch_bounds__(256) k_read_status(int32_t nv, ReadOut o, const int32_t *inj,
                                                     const int32_t *arr, const VehPos *vpos,
                                                     const int64_t *roff, int8_t *status,
                                                     int32_t *cursor, int32_t *tarr,
                                                     int32_t *bad) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= nv) return;
  const uint32_t sn = o.seen[f];
  int8_t st;
  if (sn > 1) atomicMin(bad, f);
  if (sn) st = TS_ACTIVE;
  else if (arr[f] >= 0) st = TS_ARRIVED;
  else if (inj[f] == INT_MAX) st = TS_PENDING;
  else {
    atomicMin(bad + 1, f);
    st = TS_ABSENT;
  }
  status[f] = st;
  cursor[f] = (st == TS_ACTIVE || st == TS_ARRIVED) ? (int32_t)(vpos[f].p - roff[f]) : -1;
  tarr[f] = st == TS_ARRIVED ? arr[f] : -1;
  if (!sn) {
    o.link[f] = -1;
    o.lane[f] = -1;
    o.cell[f] = -1;
    o.v[f] = -1;
  }
}

// device -> host copies of several arrays through the handle's pinned
// double buffer: the DMA of one chunk overlaps the host cores' copy of the
// previous one into the caller's (pageable) memory, whose first-touch page
// faults are then taken by all cores instead of the driver's one staging
// thread.  Small totals (or TSIM_PAGEABLE_READ) use plain cudaMemcpy.
struct D2H {
  void *dst;
  const void *src;
  size_t n;
};
static int d2h_staged(ts_sim *h, const std::vector<D2H> &segs) {
  size_t total = 0;
  for (const D2H &d : segs) total += d.dst ? d.n : 0;
  const bool staged = total >= ((size_t)64 << 20) && getenv("TSIM_PAGEABLE_READ") == nullptr;
  if (staged && !h->pin_rd[0]) {  // (no route staging kept: a network without routes to upload)
    h->pin_rd_bytes = (size_t)32 << 20;
    for (int i = 0; i < 2 && h->pin_rd_bytes; i++)
      if (cudaMallocHost(&h->pin_rd[i], h->pin_rd_bytes) != cudaSuccess) {
        cudaGetLastError();
        for (int j = 0; j < 2; j++) {
          if (h->pin_rd[j]) cudaFreeHost(h->pin_rd[j]);
          h->pin_rd[j] = nullptr;
        }
        h->pin_rd_bytes = 0;
      }
  }
  if (staged && h->pin_rd[0] && !h->ev_rd[0])
    for (int i = 0; i < 2; i++)
      if (cudaEventCreateWithFlags(&h->ev_rd[i], cudaEventDisableTiming) != cudaSuccess) {
        cudaGetLastError();
        h->ev_rd[i] = nullptr;
      }
  if (!staged || !h->pin_rd[0] || !h->ev_rd[0] || !h->ev_rd[1]) {
    for (const D2H &d : segs)
      if (d.dst && d.n) CK(h, cudaMemcpy(d.dst, d.src, d.n, cudaMemcpyDeviceToHost));
    return TS_OK;
  }
  struct Chunk {
    uint8_t *dst;
    const uint8_t *src;
    size_t n;
  };
  std::vector<Chunk> ch;
  for (const D2H &d : segs)
    if (d.dst)
      for (size_t o = 0; o < d.n; o += h->pin_rd_bytes)
        ch.push_back(Chunk{static_cast<uint8_t *>(d.dst) + o, static_cast<const uint8_t *>(d.src) + o,
                           std::min(h->pin_rd_bytes, d.n - o)});
  auto issue = [&](size_t c) -> cudaError_t {
    cudaError_t e = cudaMemcpyAsync(h->pin_rd[c & 1], ch[c].src, ch[c].n, cudaMemcpyDeviceToHost, h->stream);
    return e == cudaSuccess ? cudaEventRecord(h->ev_rd[c & 1], h->stream) : e;
  };
  CK(h, issue(0));
  for (size_t c = 0; c < ch.size(); c++) {
    if (c + 1 < ch.size()) CK(h, issue(c + 1));  // its buffer was emptied in the last iteration
    CK(h, cudaEventSynchronize(h->ev_rd[c & 1]));
    const uint8_t *b = h->pin_rd[c & 1];
    uint8_t *dst = ch[c].dst;
    parallel_for((int64_t)ch[c].n,
                 [&](int64_t lo, int64_t hi, int) { std::memcpy(dst + lo, b + lo, (size_t)(hi - lo)); });
  }
  return TS_OK;
}

static int read_vehicles_device(ts_sim *h, int8_t *status, int32_t *link, int32_t *lane,
                                int32_t *cell, int32_t *v, int32_t *cursor, int32_t *t_arrive) {
  const size_t nv = (size_t)std::max(h->nv, 1);
  if (!h->d_roff) {
    int rc;
    if ((rc = upload(h, &h->d_roff, h->roff))) return rc;
  }
  if (!h->d_rd) {  // scratch: 7 int32 arrays + the status bytes + 2 error words
    int rc;
    if ((rc = dalloc(h, &h->d_rd, nv * 7 + nv / 4 + 4))) return rc;
  }
  ReadOut o{h->d_rd, h->d_rd + nv, h->d_rd + 2 * nv, h->d_rd + 3 * nv,
            reinterpret_cast<uint32_t *>(h->d_rd + 4 * nv)};
  int32_t *dcur = h->d_rd + 5 * nv, *darr = h->d_rd + 6 * nv;
  int8_t *dst = reinterpret_cast<int8_t *>(h->d_rd + 7 * nv);
  int32_t *dbad = h->d_rd + 7 * nv + nv / 4 + 1;
  CK(h, cudaMemsetAsync(o.seen, 0, nv * 4, h->stream));
  CK(h, cudaMemsetAsync(dbad, 0x7f, 8, h->stream));
  if (h->ngroups > 0) {
    RowsParams R = rows_params(h);
    R.planes_in = h->d_planes[h->rcur];
    R.vid_in = h->d_rvid[h->rcur];
    const int n = h->ngroups * 32;
    k_read_rows<<<(n + 127) / 128, 128, 0, h->stream>>>(R, o);
  }
  if (!h->gtiles.empty()) {
    const int64_t n = (int64_t)h->gtiles.size() * 8;
    k_read_tiles<<<(unsigned)((n + 127) / 128), 128, 0, h->stream>>>(
        h->d_tiles, (int)h->gtiles.size(), h->d_code[h->gcur], h->d_vid[h->gcur], o);
  }
  if (h->nv > 0)
    k_read_status<<<(h->nv + 255) / 256, 256, 0, h->stream>>>(h->nv, o, h->d_inj, h->d_arr,
                                                              h->d_vpos, h->d_roff, dst, dcur,
                                                              darr, dbad);
  CK(h, cudaGetLastError());
  int32_t bad[2];
  CK(h, cudaMemcpyAsync(bad, dbad, 8, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  if (bad[0] != 0x7f7f7f7f) return fail(h, TS_EINTERNAL, "corrupt state: vid %d held twice", bad[0]);
  if (bad[1] != 0x7f7f7f7f) return fail(h, TS_EINTERNAL, "corrupt state: vehicle %d lost", bad[1]);
  const size_t b4 = (size_t)h->nv * 4;
  if (h->nv == 0) return TS_OK;
  return d2h_staged(h, {{status, dst, (size_t)h->nv}, {link, o.link, b4}, {lane, o.lane, b4},
                        {cell, o.cell, b4}, {v, o.v, b4}, {cursor, dcur, b4}, {t_arrive, darr, b4}});
}

extern "C" {

// ------------------------------------------------------------------ readers
// State of tiles [t0, t1) in the byte-code layout (codes at off + l*Wp + x,
// per-row vid lists) starting at element 0 = cell off(t0).  Row mode:
// decoded from the bit-planes and the vid | slot << 27 list entries.
static int download_tiles(ts_sim *h, int t0, int t1, HostVec<uint8_t> &code,
                          HostVec<int32_t> &vids) {
  const int64_t c0 = h->tiles[t0].off;
  const int64_t c1 = t1 < (int)h->tiles.size() ? h->tiles[t1].off : h->total_cells;
  code = filled<uint8_t>(c1 - c0, kEmpty);
  vids = filled<int32_t>(c1 - c0, -1);
  // general tiles of the range: one contiguous device range
  int g0 = -1, g1 = -1, s0 = -1, s1 = -1;
  for (int ti = t0; ti < t1; ti++) {
    if (h->tile_g[ti] >= 0) {
      if (g0 < 0) g0 = h->tile_g[ti];
      g1 = h->tile_g[ti] + 1;
    }
    if (h->tile_row[ti] >= 0) {
      if (s0 < 0) s0 = h->tile_row[ti];
      s1 = h->tile_row[ti] + h->tiles[ti].L;
    }
  }
  if (g0 >= 0) {
    const TileDesc &la = h->gtiles[g1 - 1];
    const int64_t a = h->gtiles[g0].off, b = la.off + tile_cells_padded(la.w, la.L);
    std::vector<uint8_t> gc(b - a);
    std::vector<int32_t> gv(b - a);
    CK(h, cudaMemcpy(gc.data(), h->d_code[h->gcur] + a, b - a, cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(gv.data(), h->d_vid[h->gcur] + a, (b - a) * 4, cudaMemcpyDeviceToHost));
    for (int ti = t0; ti < t1; ti++) {
      if (h->tile_g[ti] < 0) continue;
      const TileDesc &d = h->tiles[ti];
      const int64_t n = (int64_t)d.L * row_pitch(d.w), src = h->gtiles[h->tile_g[ti]].off - a;
      std::copy(gc.begin() + src, gc.begin() + src + n, code.begin() + (d.off - c0));
      std::copy(gv.begin() + src, gv.begin() + src + n, vids.begin() + (d.off - c0));
    }
  }
  if (s0 >= 0) {
    // row tiles: planes and vid blocks of the covering groups; a row's list
    // starts at the prefix of the vehicle counts of the rows before it
    const int gr0 = s0 >> 5, gr1 = ((s1 - 1) >> 5) + 1;
    const int64_t va = h->gvoff[gr0];
    const int64_t vb = gr1 < h->ngroups ? h->gvoff[gr1] : h->rvid_entries;
    std::vector<uint32_t> pl(group_plane_base(gr1) - group_plane_base(gr0));
    std::vector<int32_t> rv(vb - va);
    CK(h, cudaMemcpy(pl.data(), h->d_planes[h->rcur] + group_plane_base(gr0), pl.size() * 4,
                     cudaMemcpyDeviceToHost));
    CK(h, cudaMemcpy(rv.data(), h->d_rvid[h->rcur] + va, rv.size() * 4, cudaMemcpyDeviceToHost));
    std::vector<int64_t> roff((size_t)(gr1 - gr0) * 32);
    for (int g = gr0; g < gr1; g++) {
      int64_t k = h->gvoff[g] - va;
      for (int sl = 0; sl < 32; sl++) {
        roff[(size_t)(g - gr0) * 32 + sl] = k;
        const uint32_t *P = pl.data() + (group_plane_base(g) - group_plane_base(gr0)) + sl;
        for (int wd = 0; wd < kRowWords; wd++) k += __builtin_popcount(P[wd * 32]);
      }
    }
    parallel_for(t1 - t0, [&](int64_t lo, int64_t hi, int) {
    for (int ti = t0 + (int)lo; ti < t0 + (int)hi; ti++) {
      if (h->tile_row[ti] < 0) continue;
      const TileDesc &d = h->tiles[ti];
      const int Wp = row_pitch(d.w);
      for (int l = 0; l < d.L; l++) {
        const int s = h->tile_row[ti] + l;
        const uint32_t *P = pl.data() + (group_plane_base(s >> 5) - group_plane_base(gr0)) + (s & 31);
        const int32_t *lst = rv.data() + roff[(size_t)(s - gr0 * 32)];
        const int64_t rb = d.off - c0 + (int64_t)l * Wp;
        int64_t r = rb, k = 0;
        for (int x = 0; x < d.w; x++) {
          const int wd = x >> 5, bt = x & 31;
          if (!((P[wd * 32] >> bt) & 1u)) continue;
          const int v = (int)((P[(kRowWords + wd) * 32] >> bt) & 1u) |
                        (int)(((P[(2 * kRowWords + wd) * 32] >> bt) & 1u) << 1) |
                        (int)(((P[(3 * kRowWords + wd) * 32] >> bt) & 1u) << 2);
          const uint32_t e = (uint32_t)lst[k++];
          code[rb + x] = (uint8_t)(v | ((e >> kSlotShift) << 3));
          vids[r++] = (int32_t)(e & kVidMask);
        }
      }
    }
    });
  }
  return TS_OK;
}

int ts_read_vehicles(ts_sim *h, int8_t *status, int32_t *link, int32_t *lane, int32_t *cell,
                     int32_t *v, int32_t *cursor, int32_t *t_arrive) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  CK(h, cudaSetDevice(h->dev));
  // one domain: gathered on the device; domains (pending vehicles are
  // reported by the owner of their entry cell): on the host
  if (h->dom_k == 1 && !getenv("TSIM_HOST_READ"))
    return read_vehicles_device(h, status, link, lane, cell, v, cursor, t_arrive);
  CK(h, cudaStreamSynchronize(h->stream));
  HostVec<uint8_t> code;
  HostVec<int32_t> vids, inj(h->nv), arr(h->nv), cur(h->nv);
  std::vector<VehPos> vp(h->nv);
  if (int rc = download_tiles(h, 0, (int)h->tiles.size(), code, vids)) return rc;
  CK(h, cudaMemcpy(inj.data(), h->d_inj, inj.size() * 4, cudaMemcpyDeviceToHost));
  CK(h, cudaMemcpy(arr.data(), h->d_arr, arr.size() * 4, cudaMemcpyDeviceToHost));
  CK(h, cudaMemcpy(vp.data(), h->d_vpos, vp.size() * sizeof(VehPos), cudaMemcpyDeviceToHost));
  parallel_for(h->nv, [&](int64_t lo, int64_t hi, int) {
    for (int64_t f = lo; f < hi; f++) cur[f] = (int32_t)(vp[f].p - h->roff[f]);
  });
  HostVec<int32_t> lk = filled<int32_t>(h->nv, -1), ln = filled<int32_t>(h->nv, -1),
                   ce = filled<int32_t>(h->nv, -1), vv = filled<int32_t>(h->nv, -1);
  HostVec<uint8_t> seen = filled<uint8_t>(h->nv, 0);
  std::vector<int64_t> bad(64, -1);  // per thread: a corrupt entry (vid << 32 | link)
  parallel_for((int64_t)h->tiles.size(), [&](int64_t lo, int64_t hi, int th) {
    for (int64_t ti = lo; ti < hi; ti++) {
      const TileDesc &d = h->tiles[ti];
      for (int l = 0; l < d.L; l++) {
        const int64_t rb = d.off + (int64_t)l * row_pitch(d.w);
        int64_t r = rb;
        for (int x = 0; x < d.w; x++) {
          uint8_t c = code[rb + x];
          if (c & 0x80) continue;
          int f = vids[r++];
          if (f < 0 || f >= h->nv || __atomic_exchange_n(&seen[f], (uint8_t)1, __ATOMIC_RELAXED)) {
            bad[th] = ((int64_t)f << 32) | (uint32_t)d.link;
            return;
          }
          lk[f] = d.link;
          ln[f] = l;
          ce[f] = d.a + x;
          vv[f] = c & 7;
        }
      }
    }
  });
  for (int64_t b : bad)
    if (b != -1)
      return fail(h, TS_EINTERNAL, "corrupt state: vid %d at link %d", (int)(b >> 32), (int)(int32_t)b);
  std::vector<int32_t> lost(64, INT32_MAX);
  parallel_for(h->nv, [&](int64_t lo, int64_t hi, int th) {
    for (int f = (int)lo; f < (int)hi; f++) {
      int8_t s = TS_ACTIVE;
      if (seen[f]) s = TS_ACTIVE;
      else if (arr[f] >= 0) s = TS_ARRIVED;
      else if (inj[f] == INT_MAX) {
        // pending: reported by the domain owning its entry cell
        const int k = h->first_link[f];
        s = (h->entry_h[f] >= h->own_lo[k] && h->entry_h[f] < h->own_hi[k]) ? TS_PENDING : TS_ABSENT;
      } else {
        s = TS_ABSENT;  // on a cell of another domain
      }
      if (s == TS_ABSENT && h->dom_k == 1) {
        lost[th] = std::min(lost[th], f);
        return;
      }
      if (status) status[f] = s;
      if (link) link[f] = lk[f];
      if (lane) lane[f] = ln[f];
      if (cell) cell[f] = ce[f];
      if (v) v[f] = vv[f];
      if (cursor) cursor[f] = (s == TS_ACTIVE || s == TS_ARRIVED) ? cur[f] : -1;
      if (t_arrive) t_arrive[f] = s == TS_ARRIVED ? arr[f] : -1;
    }
  });
  if (const int32_t f = *std::min_element(lost.begin(), lost.end()); f != INT32_MAX)
    return fail(h, TS_EINTERNAL, "corrupt state: vehicle %d lost", f);
  return TS_OK;
}

int ts_read_cells(ts_sim *h, int32_t link, int32_t *vid_out) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  if (link < 0 || link >= h->nl) return fail(h, TS_EINVAL, "bad link");
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaStreamSynchronize(h->stream));
  const int n = h->ncell[link], L = h->lanes[link];
  for (int i = h->link_tile0[link]; i < h->link_tile0[link + 1]; i++) {
    const TileDesc &d = h->tiles[i];
    const int Wp = row_pitch(d.w);
    HostVec<uint8_t> code;
    HostVec<int32_t> vids;
    if (int rc = download_tiles(h, i, i + 1, code, vids)) return rc;
    for (int l = 0; l < L; l++) {
      int r = l * Wp;
      for (int x = 0; x < d.w; x++) {
        uint8_t c = code[(size_t)l * Wp + x];
        vid_out[(size_t)l * n + d.a + x] = (c & 0x80) ? -1 : vids[r++];
      }
    }
  }
  return TS_OK;
}

int ts_read_raw(ts_sim *h, int32_t link, uint8_t *code_out, int32_t *vid_out, int32_t *pitch) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  if (link < 0 || link >= h->nl) return fail(h, TS_EINVAL, "bad link");
  if (h->link_ntiles[link] != 1) return fail(h, TS_EINVAL, "link spans several tiles");
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaStreamSynchronize(h->stream));
  const int ti = h->link_tile0[link];
  const TileDesc &d = h->tiles[ti];
  const int Wp = row_pitch(d.w);
  *pitch = Wp;
  HostVec<uint8_t> code;
  HostVec<int32_t> vids;
  if (int rc = download_tiles(h, ti, ti + 1, code, vids)) return rc;
  memcpy(code_out, code.data(), (size_t)d.L * Wp);
  memcpy(vid_out, vids.data(), (size_t)d.L * Wp * 4);
  return TS_OK;
}

int ts_state_hash(ts_sim *h, uint64_t *out) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaMemsetAsync(h->d_hash, 0, 16, h->stream));
  StepParams P = step_params(h, h->t, 0);
  if (h->ngroups > 0) launch_rows_hash(P, rows_params(h), h->stream, h->d_hash);
  if (!h->gtiles.empty()) launch_hash(P, h->blocks, h->threads, h->smem, h->stream, h->d_hash);
  CK(h, cudaGetLastError());
  unsigned long long r[2];
  CK(h, cudaMemcpyAsync(r, h->d_hash, 16, cudaMemcpyDeviceToHost, h->stream));
  CK(h, cudaStreamSynchronize(h->stream));
  *out = r[0];
  return TS_OK;
}

int ts_read_history(ts_sim *h, int32_t t_from, int32_t n, uint64_t *hash, int64_t *active,
                    int64_t *arrivals, int64_t *injections, int64_t *lane_changes,
                    int64_t *crossings) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  if (n < 0 || n > kHist || t_from + n - 1 > h->t || t_from < h->t - kHist + 2)
    return fail(h, TS_EINVAL, "history range not available");
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaStreamSynchronize(h->stream));
  std::vector<unsigned long long> st((size_t)kHist * ST_N);
  CK(h, cudaMemcpy(st.data(), h->d_stats, st.size() * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; i++) {
    const unsigned long long *s = &st[(size_t)((t_from + i) & (kHist - 1)) * ST_N];
    if (hash) hash[i] = s[ST_HASH];
    if (active) active[i] = (int64_t)s[ST_ACTIVE];
    if (arrivals) arrivals[i] = (int64_t)s[ST_ARR];
    if (injections) injections[i] = (int64_t)s[ST_INJ];
    if (lane_changes) lane_changes[i] = (int64_t)s[ST_LC];
    if (crossings) crossings[i] = (int64_t)s[ST_CROSS];
  }
  return TS_OK;
}

int ts_read_flow(ts_sim *h, int32_t t_from, int32_t n, int64_t *sumv) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  if (n < 0 || n > kHist || t_from + n - 1 > h->t || t_from < h->t - kHist + 2)
    return fail(h, TS_EINVAL, "history range not available");
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaStreamSynchronize(h->stream));
  std::vector<unsigned long long> st((size_t)kHist * ST_N);
  CK(h, cudaMemcpy(st.data(), h->d_stats, st.size() * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; i++)
    sumv[i] = (int64_t)st[(size_t)((t_from + i) & (kHist - 1)) * ST_N + ST_SUMV];
  return TS_OK;
}

int ts_get_totals(ts_sim *h, int64_t out[8]) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  CK(h, cudaStreamSynchronize(h->stream));
  if (int rc = fold_stats(h)) return rc;
  unsigned long long st[ST_N];
  CK(h, cudaMemcpy(st, h->d_stats + (size_t)(h->t & (kHist - 1)) * ST_N, sizeof st,
                   cudaMemcpyDeviceToHost));
  const int64_t active = (int64_t)st[ST_ACTIVE];
  out[0] = active;
  out[1] = h->n_pending0 - h->injected;
  out[2] = h->n_arrived0 + h->arrived;
  out[3] = h->veh_updates;
  out[4] = h->lane_cells;
  out[5] = (int64_t)h->tiles.size();
  out[6] = (int64_t)h->dev_bytes;
  out[7] = 2 * h->lane_cells + 8 * active;
  return TS_OK;
}

int ts_get_link_work(ts_sim *h, int64_t *link_work) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  CK(h, cudaStreamSynchronize(h->stream));
  CK(h, cudaMemcpy(link_work, h->d_work, sizeof(int64_t) * h->nl, cudaMemcpyDeviceToHost));
  return TS_OK;
}

int ts_get_load(ts_sim *h, int64_t *link_work, int64_t *node_work) {
  if (!h || !h->inited) return fail(h, TS_EINVAL, "not initialised");
  CK(h, cudaSetDevice(h->dev));
  CK(h, cudaStreamSynchronize(h->stream));
  if (link_work) CK(h, cudaMemcpy(link_work, h->d_work, sizeof(int64_t) * h->nl, cudaMemcpyDeviceToHost));
  if (node_work) CK(h, cudaMemcpy(node_work, h->d_node_work, sizeof(int64_t) * h->nn, cudaMemcpyDeviceToHost));
  return TS_OK;
}

int ts_last_exchange_timing(ts_sim *h, double *ms, int64_t *n) {
  if (!h) return TS_EINVAL;
  if (ms) *ms = h->last_xchg_ms;
  if (n) *n = h->last_xchg_n;
  return TS_OK;
}

int ts_last_timing(ts_sim *h, double *total_ms, double *move_ms, int64_t *move_launches) {
  if (!h) return TS_EINVAL;
  if (total_ms) *total_ms = h->last_total_ms;
  if (move_ms) *move_ms = h->last_move_ms;
  if (move_launches) *move_launches = h->last_move_launches;
  return TS_OK;
}

// --------------------------------------------------------------- partition
// Orthogonal recursive bisection: a vertical line halves
// the load, then the larger piece is cut by a horizontal line, and so on
// until k pieces; non-power-of-two k splits in proportion.
static void orb_rec(std::vector<int32_t> &idx, size_t lo, size_t hi, const int64_t *x,
                    const int64_t *y, const std::vector<double> &w, int k, int dom0, bool vertical,
                    int32_t *out) {
  if (k == 1) {
    for (size_t i = lo; i < hi; i++) out[idx[i]] = dom0;
    return;
  }
  const int64_t *c = vertical ? x : y;
  std::stable_sort(idx.begin() + lo, idx.begin() + hi, [&](int a, int b) {
    return c[a] < c[b] || (c[a] == c[b] && a < b);
  });
  const int kl = (k + 1) / 2, kr = k - kl;
  double tot = 0;
  for (size_t i = lo; i < hi; i++) tot += w[idx[i]];
  const double target = tot * kl / k;
  double acc = 0, best = 1e300;
  size_t cut = lo + 1;
  for (size_t i = lo; i + 1 < hi + 1 && i < hi; i++) {
    acc += w[idx[i]];
    const size_t c1 = i + 1;
    if (c1 - lo < (size_t)kl || hi - c1 < (size_t)kr) continue;
    const double dev = std::fabs(acc - target);
    if (dev < best) {
      best = dev;
      cut = c1;
    }
  }
  orb_rec(idx, lo, cut, x, y, w, kl, dom0, !vertical, out);
  orb_rec(idx, cut, hi, x, y, w, kr, dom0 + kl, !vertical, out);
}

int ts_orb_partition(int32_t n_nodes, const int64_t *node_x_mm, const int64_t *node_y_mm,
                     const double *node_weight, int32_t k, int32_t *domain_of_node) {
  if (n_nodes < 1 || k < 1 || k > n_nodes) return TS_EINVAL;
  std::vector<double> w(n_nodes, 1.0);
  if (node_weight)
    for (int i = 0; i < n_nodes; i++) w[i] = std::max(0.0, node_weight[i]);
  std::vector<int32_t> idx(n_nodes);
  std::iota(idx.begin(), idx.end(), 0);
  orb_rec(idx, 0, n_nodes, node_x_mm, node_y_mm, w, k, 0, true, domain_of_node);
  return TS_OK;
}

}  // extern "C"

extern "C" {
// ORB partition of the handle's own network with the paper's default node
// weights (half of cells x lanes of every attached link)
// or the given ones, and this handle set up as domain `me` (ts_set_domain).
int ts_partition(ts_sim *h, int32_t k, const double *node_weight, int32_t me,
                 int32_t *domain_of_node_out) {
  if (!h) return TS_EINVAL;
  if (!h->have_net) return fail(h, TS_EINVAL, "load the network first");
  std::vector<double> w(h->nn, 1e-9);
  if (node_weight) {
    w.assign(node_weight, node_weight + h->nn);
  } else {
    for (int j = 0; j < h->nl; j++) {
      const double lw = 0.5 * (double)h->ncell[j] * h->lanes[j];
      w[h->from[j]] += lw;
      w[h->to[j]] += lw;
    }
  }
  std::vector<int32_t> dom(h->nn);
  if (ts_orb_partition(h->nn, h->nx.data(), h->ny.data(), w.data(), k, dom.data()))
    return fail(h, TS_EINVAL, "bad partition: k = %d for %d nodes", k, h->nn);
  if (domain_of_node_out) std::copy(dom.begin(), dom.end(), domain_of_node_out);
  return ts_set_domain(h, k, dom.data(), me);
}
}
