// tsim_rows.cu -- fast path of the TRANSIMS CA step on sm_100a: k_rows.
//
// One warp per group of consecutive whole-link tiles (<= 32 lane-rows,
// ~2K cells).  The group's int8 codes are staged in shared memory with
// 128-bit coalesced loads and an occupancy bitmap (one bit per lane-cell)
// is built; a warp scan enumerates the vehicles in (row, cell) order and
// keeps per-word popcount prefixes, so the rank of any cell is two loads
// and a popc.  All per-vehicle work is vehicle-parallel (32 vehicles per
// warp step), never row-serial:
//   1. move (H4/H5): gap from the bitmap, NaSch velocity
//      with the Philox slowdown, placement; the vid of a vehicle is read at
//      its rank within its row.  Node entrants, injection (H6)  -> S(t+1)
//   2. (fused) lane change of step t+1 (H1): bit-parallel
//      prefilter per 32-cell word (target cell, the cell ahead of it and
//      the V cells behind it free, or desperation zone), exact rule on the
//      candidates only, applied in place                     -> S1(t+1)
//   3. vid lists: a row that gained or lost no vehicle except exits at its
//      front keeps a prefix of its list (128-bit copy); in the other rows
//      every vehicle's output slot is its rank in the final bitmap and its
//      vid is found by rank in the input list (order is preserved).
#include "tsim_device.cuh"

namespace tsim {

// rank of position q in a flat bitmap with per-word exclusive prefixes wp
static __device__ __forceinline__ int flat_rank(const uint32_t *bits, const uint16_t *wp, int q) {
  return wp[q >> 5] + __popc(bits[(q >> 5) + 1] & low_mask(q & 31));
}
// same for the bitmap (b1 & ~b2)
static __device__ __forceinline__ int flat_rank2(const uint32_t *b1, const uint32_t *b2,
                                                 const uint16_t *wp, int q) {
  const int j = (q >> 5) + 1;
  return wp[q >> 5] + __popc(b1[j] & ~b2[j] & low_mask(q & 31));
}

// warp scan over the words of (b1 & ~b2) (b2 may be null): wp[j] = bits
// before word j; optionally vpos[rank] = position.  Returns the total.
static __device__ __forceinline__ int scan_words(const uint32_t *b1, const uint32_t *b2, int nw,
                                                 uint16_t *wp, uint16_t *vpos, int lane) {
  int total = 0;
  for (int j0 = 0; j0 < nw; j0 += 32) {
    const int j = j0 + lane;
    uint32_t m = 0u;
    if (j < nw) m = b2 ? (b1[j + 1] & ~b2[j + 1]) : b1[j + 1];
    const int c = __popc(m);
    int sc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, sc, o);
      if (lane >= o) sc += y;
    }
    int r = total + sc - c;
    if (j < nw) wp[j] = (uint16_t)r;
    if (vpos)
      while (m) {
        vpos[r++] = (uint16_t)(32 * j + __ffs(m) - 1);
        m &= m - 1u;
      }
    total += __shfl_sync(FULL, sc, 31);
  }
  if (lane == 0) wp[nw] = (uint16_t)total;
  __syncwarp();
  return total;
}

// any bit of a row set?
static __device__ __forceinline__ bool row_any(const uint32_t *bits, int s, int w) {
  uint32_t a = 0u;
  for (int wj = 0; wj * 32 < w; wj++) a |= win_at(bits, s + 32 * wj) & low_mask(w - 32 * wj);
  return a != 0u;
}

// vid of an entrant / injected vehicle of row `row` at cell x
static __device__ __forceinline__ int special_vid(const int32_t *ent, const int32_t *injx,
                                                  const int32_t *injv, int ninj, int row, int x) {
  if (ent[32 + row] == x) return ent[row];
  const int key = (row << 16) | x;
  for (int k = 0; k < ninj; k++)
    if (injx[k] == key) return injv[k];
  return -1;
}

__global__ void __launch_bounds__(128, 8) k_rows(const StepParams P, const RowsParams R) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long red[4 * 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  const RowsLayout &Y = R.lay;
  uint8_t *base = smem + warp * Y.bytes;
  uint8_t *cin = base + Y.o_cin, *cout = base + Y.o_cout, *rowof = base + Y.o_rowof;
  uint32_t *bin = reinterpret_cast<uint32_t *>(base + Y.o_bin);
  uint32_t *bmid = reinterpret_cast<uint32_t *>(base + Y.o_bmid);
  uint32_t *bspec = reinterpret_cast<uint32_t *>(base + Y.o_bspec);
  uint32_t *blv = reinterpret_cast<uint32_t *>(base + Y.o_bleave);
  uint32_t *bfin = reinterpret_cast<uint32_t *>(base + Y.o_bfin);
  uint16_t *vpos = reinterpret_cast<uint16_t *>(base + Y.o_vpos);
  uint16_t *wp_in = reinterpret_cast<uint16_t *>(base + Y.o_wp);
  uint16_t *wp_fin = wp_in + Y.NW;
  uint16_t *wp_mid = wp_in + 2 * Y.NW;
  int32_t *ent = reinterpret_cast<int32_t *>(base + Y.o_ent);
  int32_t *injx = reinterpret_cast<int32_t *>(base + Y.o_injx);
  int32_t *injv = reinterpret_cast<int32_t *>(base + Y.o_injv);
  int32_t *misc = reinterpret_cast<int32_t *>(base + Y.o_misc);
  int32_t *row_s = reinterpret_cast<int32_t *>(base + Y.o_rows);
  int32_t *row_w = row_s + 32;       // cells
  int32_t *row_link = row_s + 64;    // link
  int32_t *row_lv = row_s + 96;      // lane | vmax << 8
  int32_t *row_lg = row_s + 128;     // global lane id
  int32_t *row_nfin = row_s + 160;   // vehicles in the final state
  int32_t *row_front = row_s + 192;  // vid of the front vehicle (final state)
  int32_t *row_r0 = row_s + 224;     // rank of the row start in bin
  int32_t *row_f0 = row_s + 256;     // ... in bfin
  int32_t *row_m0 = row_s + 288;     // ... in (bmid & ~bspec)
  const bool hash = (P.mode & kModeHash) != 0;
  const bool lc_next = (P.mode & kModeLC) != 0;
  const bool work = (P.mode & kModeWork) && P.link_work;
  const int dir = ((P.t + 1) & 1) ? -1 : +1;  // R4, lane change of step t+1
  Acc acc = {};
  Acc acc_next = {};

  for (int g = blockIdx.x * (blockDim.x >> 5) + warp; g < R.ngroups; g += nwarps_total) {
    const GroupDesc G = R.groups[g];
    const int64_t off0 = P.tiles[G.t0].off;
    const int nw = (G.bytes + 31) >> 5;
    // ---- rows of the group (thread i describes row i)
    const bool active = lane < G.nrows;
    TileDesc d;
    d.w = 0;
    d.L = 1;
    d.link = 0;
    d.lane_gid = 0;
    int l = 0, s = 0, Wp = 4, Vk = 1;
    if (active) {
      const int rm = R.rowmap[(size_t)g * 32 + lane];
      l = rm & 7;
      d = P.tiles[G.t0 + (rm >> 3)];
      Wp = row_pitch(d.w);
      s = (int)(d.off - off0) + l * Wp;
      Vk = P.vmax_link[d.link];
    }
    // ---- stage the group's codes, clear the work bitmaps, row table
    {
      const uint4 *src = reinterpret_cast<const uint4 *>(P.code_in + off0);
      uint4 *dst = reinterpret_cast<uint4 *>(cin);
      uint4 *dco = reinterpret_cast<uint4 *>(cout);
      const uint4 e = make_uint4(FULL, FULL, FULL, FULL);
      const int n16 = G.bytes >> 4;
      for (int i = lane; i < 2 * nw; i += 32) {
        dst[i] = i < n16 ? __ldcs(src + i) : e;
        dco[i] = e;
      }
      for (int i = lane; i < nw + 3; i += 32) {
        bmid[i] = 0u;
        bspec[i] = 0u;
        blv[i] = 0u;
      }
      if (lane == 0) misc[0] = 0;
      ent[32 + lane] = -1;
      row_s[lane] = s;
      row_w[lane] = d.w;
      row_link[lane] = d.link;
      row_lv[lane] = l | (Vk << 8);
      row_lg[lane] = d.lane_gid + l;
      if (active) {  // row id of every cell of the row
        uint32_t *ro = reinterpret_cast<uint32_t *>(rowof + s);
        const uint32_t id4 = (uint32_t)lane * 0x01010101u;
        for (int i = 0; i < (Wp >> 2); i++) ro[i] = id4;
      }
    }
    __syncwarp();
    build_bits(cin, bin, nw, lane);
    __syncwarp();
    const int nveh = scan_words(bin, nullptr, nw, wp_in, vpos, lane);
    row_r0[lane] = active ? flat_rank(bin, wp_in, s) : 0;
    __syncwarp();
    // ---- 1. velocity update + move (H4/H5), 32 vehicles per warp step
    if (P.mode & kModeMove) {
      for (int r = lane; r < nveh; r += 32) {
        const int p = vpos[r];
        const int row = rowof[p];
        const int rs = row_s[row], w = row_w[row], lv = row_lv[row];
        const int x = p - rs;
        const int code = cin[p];
        const int v = code & 7, slot = code >> 3;
        const int vid = P.vid_in[off0 + rs + (r - row_r0[row])];  // rank within the row
        const int lim = min(kGmax, w - 1 - x);
        const uint32_t ma = win_ahead(bin, p) & low_mask(lim);
        int gp;
        if (ma) gp = __ffs(ma) - 1;
        else if (lim == kGmax || slot == kSlotFinal) gp = kGmax;  // R12 open end
        else gp = min(kGmax, lim + (int)P.ext[row_lg[row]]);      // node grant (H3)
        const int v3 = nasch_v3(v, lv >> 8, gp, (uint32_t)P.t, (uint32_t)vid, P.k0, P.k1, P.p32);
        const int y = x + v3;
        if (y < w) {
          cout[rs + y] = (uint8_t)(v3 | (slot << 3));
          set_bit(bmid, rs + y);
          acc_place(acc, hash, vid, row_link[row], lv & 255, y, v3);
        } else if (slot == kSlotFinal) {  // exit to parking
          P.arr_time[vid] = P.t + 1;
          acc.arr++;
        }  // else: crossed the node; the node kernel placed it on the next link
        acc.work++;
        if (work) atomicAdd(P.link_work + row_link[row], 1ull);
      }
      __syncwarp();
      if (active) {
        // entrant granted by the node kernel (lands in front of every vehicle)
        const uint64_t rec = P.entr[d.lane_gid + l];
        if ((uint32_t)(rec >> 43) == ((uint32_t)(P.t + 1) & 0x1FFFFFu)) {
          const int evid = (int)(uint32_t)rec;
          const uint8_t code = (uint8_t)(rec >> 32);
          const int y = (int)((rec >> 40) & 7);
          cout[s + y] = code;
          set_bit(bmid, s + y);
          set_bit(bspec, s + y);
          ent[lane] = evid;
          ent[32 + lane] = y;
          acc_place(acc, hash, evid, d.link, l, y, code & 7);
        }
        if ((P.mode & kModeInject) && l == 0 && P.pend_off[d.link + 1] > P.pend_head[d.link]) {
          const int row = lane;
          inject_link(
              P, d.link, 0, d.w, true, [&](int xx) { return cout[s + xx] == kEmpty; },
              [&](int xx, uint8_t code, int ivid) {
                cout[s + xx] = code;
                set_bit(bmid, s + xx);
                set_bit(bspec, s + xx);
                const int k = atomicAdd(misc, 1);
                injx[k] = (row << 16) | xx;
                injv[k] = ivid;
                acc.inj++;
                acc_place(acc, hash, ivid, d.link, 0, xx, 0);
              });
        }
      }
    }
    __syncwarp();
    // ---- 2. lane change of step t+1 on S(t+1) (H1, fused)
    const int l2 = l + dir;
    const bool can_lc = active && lc_next && l2 >= 0 && l2 < d.L;
    const int s2 = s + dir * Wp;
    if (can_lc) {
      const uint32_t tt = P.tt_link[d.link];
      for (int x0 = 0; x0 < d.w; x0 += 32) {
        const uint32_t own = win_at(bmid, s + x0) & low_mask(d.w - x0);
        if (!own) continue;
        // target lane cells x0-5 .. x0+58 as one 64-bit window
        uint64_t W = (uint64_t)win_at(bmid, s2 + x0 - kGmax) |
                     ((uint64_t)win_at(bmid, s2 + x0 + 27) << 32);
        if (x0 == 0) W &= ~(uint64_t)31u;  // before the link start: empty (R2)
        const int endb = d.w - x0 + kGmax;  // first bit at or beyond the link end
        const uint64_t Wend = endb < 64 ? (W | (~0ull << endb)) : W;
        const uint32_t T = (uint32_t)(W >> kGmax);            // target cell
        const uint32_t Tn = (uint32_t)(Wend >> (kGmax + 1));  // cell ahead of it
        uint32_t B = 0u;                                      // Vk cells behind it
        for (int k = 1; k <= Vk; k++) B |= (uint32_t)(W >> (kGmax - k));
        const uint32_t DZ = range_mask(d.w - P.D - x0, 32);  // desperation zone
        uint32_t cand = own & ~T & ((~Tn & ~B) | DZ);
        while (cand) {
          const int x = x0 + __ffs(cand) - 1;
          cand &= cand - 1u;
          if (lc_rule(bmid, s + x, s2 + x, s, s + d.w, s2, s2 + d.w, cout[s + x], l, l2, d.L,
                      dir, d.w - 1 - x, tt, false, Vk, P.D)) {
            set_bit(blv, s + x);
            acc_next.lc++;
          }
        }
      }
    }
    __syncwarp();
    for (int i = lane; i < nw + 3; i += 32) bfin[i] = bmid[i] & ~blv[i];
    __syncwarp();
    if (can_lc) {  // apply: sideways moves into cells that were empty
      for (int x0 = 0; x0 < d.w; x0 += 32) {
        uint32_t m = win_at(blv, s + x0) & low_mask(d.w - x0);
        while (m) {
          const int x = x0 + __ffs(m) - 1;
          m &= m - 1u;
          cout[s2 + x] = cout[s + x];
          cout[s + x] = kEmpty;
          set_bit(bfin, s2 + x);
        }
      }
    }
    // ---- 3. vid lists of the final state
    for (int i = lane; i < nw + 3; i += 32) bin[i] = 0u;  // becomes: changed rows' cells
    __syncwarp();
    bool changed = false;
    if (active) {
      changed = row_any(bspec, s, d.w) || (lc_next && row_any(blv, s, d.w));
      int nfin = 0;
      uint32_t diff = 0u;
      for (int x0 = 0; x0 < d.w; x0 += 32) {
        const uint32_t f = win_at(bfin, s + x0) & low_mask(d.w - x0);
        nfin += __popc(f);
        diff |= f ^ (win_at(bmid, s + x0) & low_mask(d.w - x0));
      }
      changed |= diff != 0u;  // arrivals
      row_nfin[lane] = nfin;
      if (!changed) {
        // input vehicles minus exits at the front: a prefix of the input list
        const uint4 *src = reinterpret_cast<const uint4 *>(P.vid_in + off0 + s);
        uint4 *dst = reinterpret_cast<uint4 *>(P.vid_out + off0 + s);
        uint4 bufv = make_uint4(0, 0, 0, 0);
        for (int i = 0; i < nfin; i += 4) {
          bufv = __ldg(src + (i >> 2));
          __stcs(dst + (i >> 2), bufv);
        }
        const int k = (nfin - 1) & 3;
        row_front[lane] = (int)(k == 0 ? bufv.x : k == 1 ? bufv.y : k == 2 ? bufv.z : bufv.w);
      } else {
        for (int x0 = 0; x0 < d.w; x0 += 32) {  // mark the row's cells
          const uint32_t m = low_mask(d.w - x0);
          const int q = s + x0, sh = q & 31;
          atomicOr(bin + (q >> 5) + 1, m << sh);
          if (sh) atomicOr(bin + (q >> 5) + 2, m >> (32 - sh));
        }
      }
    }
    if (__ballot_sync(FULL, changed)) {
      __syncwarp();
      for (int i = lane; i < nw; i += 32) bin[i + 1] &= bfin[i + 1];
      scan_words(bfin, nullptr, nw, wp_fin, nullptr, lane);
      scan_words(bmid, bspec, nw, wp_mid, nullptr, lane);
      const int nch = scan_words(bin, nullptr, nw, wp_in, vpos, lane);
      row_f0[lane] = active ? flat_rank(bfin, wp_fin, s) : 0;
      row_m0[lane] = active ? flat_rank2(bmid, bspec, wp_mid, s) : 0;
      __syncwarp();
      for (int r = lane; r < nch; r += 32) {
        const int p = vpos[r];
        const int row = rowof[p];
        const int rs = row_s[row];
        const int x = p - rs;
        const int j = flat_rank(bfin, wp_fin, p) - row_f0[row];  // output slot
        int vid;
        if (occupied(bmid, p)) {  // own post-move vehicle
          if (occupied(bspec, p)) vid = special_vid(ent, injx, injv, misc[0], row, x);
          else vid = P.vid_in[off0 + rs + flat_rank2(bmid, bspec, wp_mid, p) - row_m0[row]];
        } else {  // arrived from the row l - dir of the same link
          const int wpr = row_pitch(row_w[row]);
          const int ps = p - dir * wpr, srow = row - dir;
          if (occupied(bspec, ps)) vid = special_vid(ent, injx, injv, misc[0], srow, x);
          else
            vid = P.vid_in[off0 + (rs - dir * wpr) + flat_rank2(bmid, bspec, wp_mid, ps) -
                           row_m0[srow]];
        }
        P.vid_out[off0 + rs + j] = vid;
        if (j == row_nfin[row] - 1) row_front[row] = vid;  // front vehicle
      }
    }
    __syncwarp();
    if (active && lc_next) {  // the output is S1(t+1): node records for k_node_warp
      const uint32_t fin = win_at(bfin, s + d.w - kGmax) & 31u;  // bit i = cell w-5+i
      uint64_t rec = (uint64_t)(__brev(fin) >> 27) << 44;          // bit i = cell n-1-i
      if (fin) {
        const int xf = d.w - kGmax + 31 - __clz(fin);
        rec |= (uint64_t)(uint32_t)row_front[lane] | ((uint64_t)cout[s + xf] << 32) |
               ((uint64_t)(d.w - 1 - xf) << 40) | (1ull << 43);
      }
      P.tail_rec[d.lane_gid + l] = rec;
      P.head_occ[d.lane_gid + l] = (uint8_t)(win_at(bfin, s) & 31u);
    }
    {
      uint4 *dst = reinterpret_cast<uint4 *>(P.code_out + off0);
      const uint4 *src = reinterpret_cast<const uint4 *>(cout);
      for (int i = lane; i < (G.bytes >> 4); i += 32) __stcs(dst + i, src[i]);
    }
    __syncwarp();
  }
  flush_acc(P, acc, P.t + 1, red);
  if (lc_next) flush_acc(P, acc_next, P.t + 2, red);
}

void launch_rows(const StepParams &p, const RowsParams &r, int blocks, int threads, int smem,
                 void *stream) {
  k_rows<<<blocks, threads, smem, (cudaStream_t)stream>>>(p, r);
}
cudaError_t set_rows_smem(int bytes) {
  return cudaFuncSetAttribute(k_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
int occupancy_rows(int threads, int smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows, threads, smem);
  return nb;
}

}  // namespace tsim
