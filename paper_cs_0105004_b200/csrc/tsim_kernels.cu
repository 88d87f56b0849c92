// tsim_kernels.cu -- general-path and node kernels of the TRANSIMS CA step
// on sm_100a (Nagel & Rickert, §3-§4; readings R1-R22 in
// DESIGN.md §3).  The fast row kernel lives in tsim_rows.cu.
//
// State: one int8 code per lane-cell (0xFF empty, else velocity | out-slot
// << 3) and, per lane-row, the vids of its vehicles in cell order.
//
// General path (any tile, incl. tiles with 5-cell halos: long, periodic or
// split links): one warp per tile; the tile's codes are staged in shared
// memory, vehicles are enumerated by rank (prefix popcount).
//   k_lc    S(t)  -> S1(t)   lane change (H1), node records + strips
//   k_step  S1(t) -> S(t+1)  velocity update + move (H4/H5), entrants,
//                            injection (H6), ghost moves across tile seams,
//                            optionally the lane change of step t+1
//   k_hash  state hash of S(t)
// Intersections (H3):
//   k_node_warp  one thread per incoming lane; __match_any_sync picks the
//                winner of every target lane
//   k_node       one thread per node (fallback for > 32 incoming lanes)
#include "tsim_device.cuh"

// checked build (-DTS_CHECKED): invariants of a node crossing (H3/H5) and
// of the general tiles' output state, counted per device and read by
// ts_debug_checks (csrc/tsim_rows.cu).  Bits: 256 a crosser landing on or
// past the first occupied cell of its target lane, 512 a
// crossing velocity above the link's vmax, 1024 a
// crossing by a vehicle with no next link on its route, 2048 an occupied
// tile cell without a vehicle id, 4096 a tile vehicle above its link's vmax
#ifdef TS_CHECKED
__device__ unsigned int g_ts_chk_node[2] = {0u, 0u};  // bits, count
#define TS_CHK_NODE(cond, bit)                        \
  do {                                                \
    if (!(cond)) {                                    \
      atomicOr(&g_ts_chk_node[0], (unsigned)(bit));   \
      atomicAdd(&g_ts_chk_node[1], 1u);               \
    }                                                 \
  } while (0)
#else
#define TS_CHK_NODE(cond, bit) ((void)0)
#endif

namespace tsim {

// ====================================================================
// General path
// ====================================================================
struct TileCtx {
  TileDesc d;
  int S, HP, nwords, L, w, Wp;
  int has_up, has_dn, ghosts;
  uint8_t *cin, *cout;
  uint32_t *bin, *bout;
  int32_t *vout, *lf;
  uint16_t *vpos, *dpos, *vrow;
};

__device__ __forceinline__ void tile_setup(TileCtx &T, const TileDesc *tiles, int ti,
                                           const WarpLayout &lay, uint8_t *base) {
  T.d = tiles[ti];
  T.L = T.d.L;
  T.w = T.d.w;
  T.Wp = row_pitch(T.w);
  T.S = tile_stride(T.w, T.d.flags);
  T.HP = (T.d.flags & kHalo) ? kHaloPad : 0;
  T.nwords = (T.L * T.S + 31) >> 5;
  T.has_up = (T.d.flags & kHasUp) != 0;
  T.has_dn = (T.d.flags & kHasDn) != 0;
  T.ghosts = T.has_up && !(T.d.flags & 64);  // 64: the neighbour is the tile itself
  T.cin = base + lay.o_cin;
  T.cout = base + lay.o_cout;
  T.bin = reinterpret_cast<uint32_t *>(base + lay.o_bin);
  T.bout = reinterpret_cast<uint32_t *>(base + lay.o_bout);
  T.vout = reinterpret_cast<int32_t *>(base + lay.o_vout);
  T.vpos = reinterpret_cast<uint16_t *>(base + lay.o_vpos);
  T.dpos = T.vpos + lay.NC;
  T.vrow = T.vpos + 2 * lay.NC;
  T.lf = reinterpret_cast<int32_t *>(base + lay.o_lf);
}

__device__ __forceinline__ int lane_of(const TileCtx &T, int p) {
  int l = 0;
  while (l + 1 < T.L && p >= (l + 1) * T.S) l++;
  return l;
}

// owned positions of word j; a word spans every row it intersects (rows can
// be as short as 12 cells)
__device__ __forceinline__ uint32_t owned_mask(const TileCtx &T, int j) {
  const int p0 = 32 * j;
  const int k1 = min(T.L - 1, (p0 + 31) / T.S);
  uint32_t m = 0u;
  for (int k = p0 / T.S; k <= k1; k++)
    m |= range_mask(k * T.S + T.HP - p0, k * T.S + T.HP + T.w - p0);
  return m;
}

// rank -> position for the owned vehicles of `bits` (lane-major order);
// also vrow[r] = index of the vehicle within its lane-row.  Returns count.
__device__ int enumerate(const TileCtx &T, const uint32_t *bits, uint16_t *vpos, int lane) {
  int total = 0;
  for (int j0 = 0; j0 < T.nwords; j0 += 32) {
    int j = j0 + lane;
    uint32_t m = j < T.nwords ? (bits[j + 1] & owned_mask(T, j)) : 0u;
    int c = __popc(m);
    int s = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    int r = total + s - c;
    while (m) {
      int b = __ffs(m) - 1;
      m &= m - 1u;
      vpos[r++] = (uint16_t)(32 * j + b);
    }
    total += __shfl_sync(FULL, s, 31);
  }
  __syncwarp();
  for (int r = lane; r < total; r += 32) {
    const int l = lane_of(T, vpos[r]);
    if (r == 0 || lane_of(T, vpos[r - 1]) != l) T.lf[l] = r;
  }
  __syncwarp();
  for (int r = lane; r < total; r += 32) T.vrow[r] = (uint16_t)(r - T.lf[lane_of(T, vpos[r])]);
  __syncwarp();
  return total;
}

__device__ __forceinline__ int64_t vid_index(const TileCtx &T, int q, int r) {
  return T.d.off + (int64_t)lane_of(T, q) * T.Wp + T.vrow[r];
}

// stage the codes of the tile (+ 5-cell halos from strips) into smem
__device__ void load_codes(const TileCtx &T, const uint8_t *gcode, const Strip *strips,
                           const int32_t *halo_up, const int32_t *halo_dn, int lane) {
  const int nb = T.nwords * 32;
  if (!T.HP) {
    const int n16 = (T.L * T.Wp + 15) >> 4;
    const uint4 *src = reinterpret_cast<const uint4 *>(gcode + T.d.off);
    uint4 *dst = reinterpret_cast<uint4 *>(T.cin);
    for (int i = lane; i < n16; i += 32) dst[i] = __ldcs(src + i);
    for (int i = 16 * n16 + lane; i < nb; i += 32) T.cin[i] = kEmpty;
  } else {
    uint32_t *c32 = reinterpret_cast<uint32_t *>(T.cin);
    for (int i = lane; i < nb / 4; i += 32) c32[i] = 0xFFFFFFFFu;
    __syncwarp();
    for (int l = 0; l < T.L; l++)
      for (int x = lane; x < T.w; x += 32)
        T.cin[l * T.S + T.HP + x] = gcode[T.d.off + (int64_t)l * T.Wp + x];
    for (int i = lane; i < T.L * kGmax; i += 32) {
      int l = i / kGmax, j = i - l * kGmax;
      if (T.has_up)
        T.cin[l * T.S + T.HP - kGmax + j] = strips[halo_up[T.d.strip] + l].tail_code[j];
      if (T.has_dn) T.cin[l * T.S + T.HP + T.w + j] = strips[halo_dn[T.d.strip] + l].head_code[j];
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void clear_codes(const TileCtx &T, uint8_t *c, int lane) {
  uint4 e = make_uint4(FULL, FULL, FULL, FULL);
  uint4 *c16 = reinterpret_cast<uint4 *>(c);
  for (int i = lane; i < T.nwords * 2; i += 32) c16[i] = e;
}

// valid range of lane l in the smem rows (R2)
__device__ __forceinline__ int row_hi(const TileCtx &T, int l) {
  return l * T.S + T.HP + T.w + (T.has_dn ? kGmax : 0);
}
__device__ __forceinline__ int row_lo(const TileCtx &T, int l) {
  return l * T.S + T.HP - (T.has_up ? kGmax : 0);
}

__device__ int lc_decide(const StepParams &P, const TileCtx &T, const uint8_t *c,
                         const uint32_t *bits, int q, int dir, uint32_t tt, int Vk) {
  const int l = lane_of(T, q);
  const int l2 = l + dir;
  if (l2 < 0 || l2 >= T.L) return -1;
  const int q2 = q + dir * T.S;
  const int x = T.d.a + (q - l * T.S - T.HP);
  return lc_rule(bits, q, q2, row_lo(T, l), row_hi(T, l), row_lo(T, l2), row_hi(T, l2), c[q],
                 l, l2, T.L, dir, T.d.n - 1 - x, tt, (T.d.flags & kPeriodic) != 0, Vk, P.D)
             ? q2
             : -1;
}

// lane change of all owned vehicles of (c, vout, bits) in place; returns
// the number of changes.  Decisions read the pre-change state only.
__device__ int lane_change(const StepParams &P, TileCtx &T, uint8_t *c, uint32_t *bits,
                           int tstep, int lane) {
  const int n = enumerate(T, bits, T.vpos, lane);
  const int dir = (tstep & 1) ? -1 : +1;  // R4
  const uint32_t tt = P.tt_link[T.d.link];
  const int Vk = P.vmax_link[T.d.link];
  for (int r = lane; r < n; r += 32) {
    int q2 = lc_decide(P, T, c, bits, T.vpos[r], dir, tt, Vk);
    T.dpos[r] = q2 < 0 ? 0xFFFFu : (uint16_t)q2;
  }
  __syncwarp();
  int cnt = 0;
  for (int r = lane; r < n; r += 32) {
    int q2 = T.dpos[r];
    if (q2 == 0xFFFF) continue;
    int q = T.vpos[r];
    c[q2] = c[q];
    T.vout[q2] = T.vout[q];
    c[q] = kEmpty;
    cnt++;
  }
  __syncwarp();
  build_bits(c, bits, T.nwords, lane);
  __syncwarp();
  return cnt;
}

// write the tile state (cout, vout, bout) back: codes, per-row vids,
// strips, node records (when the state is S1)
__device__ void write_back(const StepParams &P, TileCtx &T, bool node_recs, int lane) {
  if (!T.HP) {
    const int n16 = (T.L * T.Wp + 15) >> 4;
    uint4 *dst = reinterpret_cast<uint4 *>(P.code_out + T.d.off);
    const uint4 *src = reinterpret_cast<const uint4 *>(T.cout);
    for (int i = lane; i < n16; i += 32) __stcs(dst + i, src[i]);
  } else {
    for (int l = 0; l < T.L; l++)
      for (int x = lane; x < T.w; x += 32)
        P.code_out[T.d.off + (int64_t)l * T.Wp + x] = T.cout[l * T.S + T.HP + x];
  }
  const int n = enumerate(T, T.bout, T.vpos, lane);
  for (int r = lane; r < n; r += 32) {
    const int q = T.vpos[r];
    TS_CHK_NODE(T.vout[q] >= 0, 2048);
    TS_CHK_NODE((int)(T.cout[q] & 7u) <= (int)P.vmax_link[T.d.link], 4096);
    P.vid_out[vid_index(T, q, r)] = T.vout[q];
  }
  if (T.d.strip >= 0) {
    for (int i = lane; i < T.L * kGmax; i += 32) {
      int l = i / kGmax, j = i - l * kGmax;
      Strip *s = P.strip_out + T.d.strip + l;
      int ph = l * T.S + T.HP + j, pt = l * T.S + T.HP + T.w - kGmax + j;
      uint8_t ch = T.cout[ph], ct = T.cout[pt];
      int vh = ch < 0x80 ? T.vout[ph] : -1, vt = ct < 0x80 ? T.vout[pt] : -1;
      s->head_code[j] = ch;
      s->tail_code[j] = ct;
      s->head_vid[j] = vh;
      s->tail_vid[j] = vt;
      s->tail_pos[j] = vt >= 0 ? P.vpos[vt].p : -1;
    }
  }
  if (node_recs && !(T.d.flags & kPeriodic)) {
    for (int l = lane; l < T.L; l += 32) {
      if (T.d.flags & kLast) {
        const int pt0 = l * T.S + T.HP + T.w - kGmax;
        const uint32_t occ = __brev(win_at(T.bout, pt0)) >> 27;  // bit i = cell n-1-i
        uint64_t rec = (uint64_t)occ << 44;
        if (occ) {
          int i = __ffs(occ) - 1;
          int pf = pt0 + kGmax - 1 - i;
          rec |= (uint64_t)(uint32_t)T.vout[pf] | ((uint64_t)T.cout[pf] << 32) |
                 ((uint64_t)i << 40) | (1ull << 43);
        }
        P.tail_rec[P.nli[T.d.lane_gid + l]] = rec;
      }
      if (T.d.flags & kFirst)
        P.head_occ[P.nlo[T.d.lane_gid + l]] = (uint8_t)(win_at(T.bout, l * T.S + T.HP) & 31u);
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void place(TileCtx &T, int pos, uint8_t code, int vid) {
  T.cout[pos] = code;
  T.vout[pos] = vid;
}

// move one vehicle at smem position q (owned, or a ghost in the upstream
// halo) -- H4 + H5
__device__ __forceinline__ void move_one(const StepParams &P, TileCtx &T, Acc &acc, int q,
                                         int vid, bool ghost, int Vk, int64_t ghost_pos = -1) {
  const int l = lane_of(T, q);
  int x = T.d.a + (q - l * T.S - T.HP);
  const bool periodic = (T.d.flags & kPeriodic) != 0;
  if (periodic && x < 0) x += T.d.n;
  const int code = T.cin[q];
  const int v = code & 7, slot = code >> 3;
  // gap (PAPER.md:330-335 rule (ii)): nearest vehicle ahead within 5 cells
  const int lim = min(kGmax, row_hi(T, l) - q - 1);
  const uint32_t m = win_ahead(T.bin, q) & low_mask(lim);
  int g;
  if (m) g = __ffs(m) - 1;
  else if (lim == kGmax) g = kGmax;
  else if (slot == kSlotFinal) g = kGmax;  // R12: open end of the final link
  else g = min(kGmax, lim + (int)P.ext[P.nli[T.d.lane_gid + l]]);  // node grant (H3)
  const int v3 = nasch_v3(v, Vk, g, (uint32_t)P.t, (uint32_t)vid, P.k0, P.k1, P.p32);
  int y = x + v3;
  if (periodic && y >= T.d.n) y -= T.d.n;
  const int yl = y - T.d.a;
  if (yl >= 0 && yl < T.w) {
    place(T, l * T.S + T.HP + yl, (uint8_t)(v3 | (slot << 3)), vid);
    acc_place(acc, P.mode & kModeHash, vid, T.d.link, l, y, v3);
    // a migrant from the upstream strip brings its route position (the
    // vehicle state of another domain is not visible here)
    if (ghost) P.vpos[vid].p = ghost_pos;
  } else if (!periodic && y > T.d.n - 1 && !ghost) {
    if (slot == kSlotFinal) {  // exit to parking
      P.arr_time[vid] = P.t + 1;
      acc.arr++;
    }
    // else: node crossing; the node kernel placed it on the next link
  }
  if (!ghost) acc.work++;
}

// ------------------------------------------------------------- k_lc
__global__ void __launch_bounds__(256) k_lc(const StepParams P_) {
  const StepParams P = with_time(P_);
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long red[8 * 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  uint8_t *base = smem + warp * P.lay.bytes;
  Acc acc = {};
  TileCtx T;
  for (int ti = blockIdx.x * (blockDim.x >> 5) + warp; ti < P.ntiles; ti += nwarps_total) {
    tile_setup(T, P.tiles, ti, P.lay, base);
    load_codes(T, P.code_in, P.strip_in, P.halo_up, P.halo_dn, lane);
    build_bits(T.cin, T.bin, T.nwords, lane);
    __syncwarp();
    {
      const uint4 *s16 = reinterpret_cast<const uint4 *>(T.cin);
      uint4 *d16 = reinterpret_cast<uint4 *>(T.cout);
      for (int i = lane; i < T.nwords * 2; i += 32) d16[i] = s16[i];
    }
    const int n = enumerate(T, T.bin, T.vpos, lane);
    for (int r = lane; r < n; r += 32) T.vout[T.vpos[r]] = P.vid_in[vid_index(T, T.vpos[r], r)];
    __syncwarp();
    {
      const int dir = (P.t & 1) ? -1 : +1;
      const uint32_t tt = P.tt_link[T.d.link];
      const int Vk = P.vmax_link[T.d.link];
      for (int r = lane; r < n; r += 32) {
        int q2 = lc_decide(P, T, T.cin, T.bin, T.vpos[r], dir, tt, Vk);
        T.dpos[r] = q2 < 0 ? 0xFFFFu : (uint16_t)q2;
      }
      __syncwarp();
      for (int r = lane; r < n; r += 32) {
        int q2 = T.dpos[r];
        if (q2 == 0xFFFF) continue;
        int q = T.vpos[r];
        T.cout[q2] = T.cout[q];
        T.vout[q2] = T.vout[q];
        T.cout[q] = kEmpty;
        acc.lc++;
      }
      __syncwarp();
    }
    build_bits(T.cout, T.bout, T.nwords, lane);
    __syncwarp();
    write_back(P, T, true, lane);
  }
  flush_acc(P, acc, P.t + 1, red);
}

// ------------------------------------------------------------- k_step
__global__ void __launch_bounds__(256) k_step(const StepParams P_) {
  const StepParams P = with_time(P_);
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long red[8 * 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  uint8_t *base = smem + warp * P.lay.bytes;
  Acc acc = {};
  Acc acc_next = {};  // lane changes of step t+1 (fused)
  TileCtx T;
  const bool hash = (P.mode & kModeHash) != 0;
  for (int ti = blockIdx.x * (blockDim.x >> 5) + warp; ti < P.ntiles; ti += nwarps_total) {
    tile_setup(T, P.tiles, ti, P.lay, base);
    load_codes(T, P.code_in, P.strip_in, P.halo_up, P.halo_dn, lane);
    build_bits(T.cin, T.bin, T.nwords, lane);
    clear_codes(T, T.cout, lane);
    __syncwarp();
    const int Vk = P.vmax_link[T.d.link];
    const int n = enumerate(T, T.bin, T.vpos, lane);
    const uint32_t work0 = acc.work;
    if (P.mode & kModeMove) {
      for (int r = lane; r < n; r += 32) {
        const int q = T.vpos[r];
        move_one(P, T, acc, q, P.vid_in[vid_index(T, q, r)], false, Vk);
      }
      if (T.ghosts) {  // vehicles of the upstream strip that may enter this tile
        for (int i = lane; i < T.L * kGmax; i += 32) {
          int l = i / kGmax, j = i - l * kGmax;
          int q = l * T.S + T.HP - kGmax + j;
          if (occupied(T.bin, q)) {
            const Strip &hs = P.strip_in[P.halo_up[T.d.strip] + l];
            move_one(P, T, acc, q, hs.tail_vid[j], true, Vk, hs.tail_pos[j]);
          }
        }
      }
      // entrants granted by the node kernel (H3/H5): at most one per lane
      if ((T.d.flags & kFirst) && lane < T.L) {
        const int el = P.nlo[T.d.lane_gid + lane];
        uint64_t rec = P.entr[el];
        if ((uint32_t)(rec >> 43) == ((uint32_t)(P.t + 1) & 0x1FFFFFu) && (uint32_t)rec != kNoEntrant) {
          P.entr[el] = ~0ull;  // consumed (reset): the 21-bit time tag would match again 2^21 steps on
          int vid = (int)(uint32_t)rec;
          uint8_t code = (uint8_t)(rec >> 32);
          int y = (int)((rec >> 40) & 7);
          place(T, lane * T.S + T.HP + y, code, vid);
          acc_place(acc, hash, vid, T.d.link, lane, y, code & 7);
        }
      }
    } else {  // initial injection: state unchanged
      for (int r = lane; r < n; r += 32) {
        int q = T.vpos[r];
        int vid = P.vid_in[vid_index(T, q, r)];
        int l = lane_of(T, q);
        place(T, q, T.cin[q], vid);
        acc_place(acc, hash, vid, T.d.link, l, T.d.a + q - l * T.S - T.HP, T.cin[q] & 7);
      }
    }
    __syncwarp();
    if ((P.mode & kModeInject) && lane == 0) {
      inject_link(
          P, T.d.link, T.d.a, T.w, T.d.a == 0, [&](int x) { return T.cout[T.HP + x] == kEmpty; },
          [&](int x, uint8_t code, int vid) {
            place(T, T.HP + x, code, vid);
            acc.inj++;
            acc_place(acc, hash, vid, T.d.link, 0, T.d.a + x, 0);
          });
    }
    __syncwarp();
    if ((P.mode & kModeWork) && P.link_work) {
      uint32_t wk = acc.work - work0;
#pragma unroll
      for (int o = 16; o; o >>= 1) wk += __shfl_down_sync(FULL, wk, o);
      if (lane == 0 && wk) atomicAdd(P.link_work + T.d.link, (unsigned long long)wk);
    }
    build_bits(T.cout, T.bout, T.nwords, lane);
    __syncwarp();
    const bool lc_next = (P.mode & kModeLC) != 0;
    if (lc_next) acc_next.lc += lane_change(P, T, T.cout, T.bout, P.t + 1, lane);
    write_back(P, T, lc_next, lane);
  }
  flush_acc(P, acc, P.t + 1, red);
  if (P.mode & kModeLC) flush_acc(P, acc_next, P.t + 2, red);
}

// ------------------------------------------------------------- k_hash
__global__ void __launch_bounds__(256) k_hash(const StepParams P, unsigned long long *out) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  uint8_t *base = smem + warp * P.lay.bytes;
  uint64_t h = 0, cnt = 0;
  TileCtx T;
  for (int ti = blockIdx.x * (blockDim.x >> 5) + warp; ti < P.ntiles; ti += nwarps_total) {
    tile_setup(T, P.tiles, ti, P.lay, base);
    load_codes(T, P.code_in, P.strip_in, P.halo_up, P.halo_dn, lane);
    build_bits(T.cin, T.bin, T.nwords, lane);
    __syncwarp();
    const int n = enumerate(T, T.bin, T.vpos, lane);
    for (int r = lane; r < n; r += 32) {
      int q = T.vpos[r];
      int l = lane_of(T, q);
      h += vmix(P.vid_in[vid_index(T, q, r)], T.d.link, l, T.d.a + q - l * T.S - T.HP,
                T.cin[q] & 7);
      cnt++;
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    h += __shfl_down_sync(FULL, h, o);
    cnt += __shfl_down_sync(FULL, cnt, o);
  }
  if (lane == 0) {
    atomicAdd(out, (unsigned long long)h);
    atomicAdd(out + 1, (unsigned long long)cnt);
  }
}

// ====================================================================
// Intersections: O1 §Node (R8-R10).  Candidates are the
// front vehicles of the incoming lanes that want to pass the stop line
// (d < min(v+1, V)); majors first, minors only if the last G cells of every
// major lane are empty; one winner per target lane in (class, link, lane)
// order; the winner is granted the entry space E and, if its velocity takes
// it past the stop line, is written as the entrant of the target lane.
// ====================================================================
struct Cand {
  bool cand;
  int tgt, n2, d, v, vid;
  int tgt_row;  // row slot of the target lane (row kernel), or -1
};

// the lane's front vehicle (last kGmax cells) is on its final link: the row
// kernel reads the grant by row slot as the front's gap beyond the stop
// line, which for a final link is the open end (R12), kGmax -- so the row
// kernel needs no vid-list entry to take the front's gap
__device__ __forceinline__ bool front_final(uint64_t rec) {
  return ((rec >> 43) & 1) && (int)((rec >> 35) & 0x1F) == kSlotFinal;
}

// the front vehicle of an incoming lane: candidate to cross (d < min(v+1,
// V)) unless it is on its final link; its target lane (R8)
__device__ __forceinline__ Cand node_candidate(const NodeParams &P, uint64_t rec, int lane,
                                               int out_base, uint32_t tt, int vk) {
  Cand c{false, -1, 0, 0, 0, 0, -1};
  if (!((rec >> 43) & 1)) return c;
  const int code = (int)((rec >> 32) & 0xFF);
  c.d = (int)((rec >> 40) & 7);
  c.v = code & 7;
  const int slot = code >> 3;
  if (slot == kSlotFinal || !(c.d < min(c.v + 1, vk))) return c;
  const NodeOut o = P.nodeout[out_base + slot];
  const int tty = (tt >> (2 * slot)) & 3;
  const int l2 = tty == 0 ? min(lane, o.L - 1) : (tty == 2 ? 0 : o.L - 1);  // R8
  c.tgt = o.lgid + l2;
  c.tgt_row = o.row0 >= 0 ? o.row0 + l2 : -1;
  c.n2 = o.n;
  c.vid = (int)(uint32_t)rec;
  c.cand = true;
  return c;
}

// the winner's grant: returns ext; writes the entrant record if it crosses.
// head: occupancy of the first cells of the target lane.  The route
// position record (16 bytes per vehicle) is read only for a crossing.
__device__ __forceinline__ int node_grant(const NodeParams &P, const Cand &c, int vk, uint8_t head,
                                          uint32_t &crossings, bool pass = false) {
  const int E = min(ctz32((uint32_t)head | 0x20u), min(kGmax, c.n2));
  if (E == 0) return 0;
  const int v3 = nasch_v3(c.v, vk, min(kGmax, c.d + E), (uint32_t)P.t, (uint32_t)c.vid, P.k0,
                          P.k1, P.p32);
  if (v3 > c.d) {
    TS_CHK_NODE(v3 - c.d - 1 < E, 256);
    TS_CHK_NODE(v3 <= vk, 512);
    int nslot = 0;  // pass-through node of a ring: straight on, same route position
    if (!pass) {
      const VehPos q = P.vpos[c.vid];
      TS_CHK_NODE(q.p + 1 < q.e, 1024);
      nslot = (q.p + 2 < q.e) ? (int)P.rslot[q.p + 2] : kSlotFinal;
      P.vpos[c.vid].p = q.p + 1;
    }
    const int y2 = v3 - c.d - 1;
    const uint64_t rec = (uint64_t)(uint32_t)c.vid | ((uint64_t)(v3 | (nslot << 3)) << 32) |
                         ((uint64_t)y2 << 40) | ((uint64_t)((P.t + 1) & 0x1FFFFF) << 43);
    // a row-kernel lane reads its entrant by row slot, a general tile by
    // node-out-lane index: one record each (a scattered 8-byte store costs
    // a partial-sector read-modify-write in DRAM)
    if (c.tgt_row >= 0) P.entr_row[c.tgt_row] = rec;
    else P.entr[c.tgt] = rec;
    crossings += pass ? 0u : 1u;
  }
  return E;
}

__device__ __forceinline__ void node_flush(const NodeParams &P, uint32_t crossings,
                                           unsigned long long *red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) crossings += __shfl_down_sync(FULL, crossings, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = crossings;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += red[w];
    if (s) atomicAdd(P.stats + (size_t)((P.t + 1) & (kHist - 1)) * ST_N + ST_CROSS, s);
  }
}

// one thread per incoming lane; the lanes of a node are consecutive threads
// in priority order, so the winner of a target lane is the lowest eligible
// thread with that target.  Every warp resolves kNodeILP chunks at once
// stage by stage (records, out-slot table and target heads, grant), so their
// dependent loads overlap instead of running as one latency chain per
// chunk.
#ifndef TS_NODE_ILP
#define TS_NODE_ILP 1  // measured on 4a: 1 -> 31.5 us, 2 -> 35, 4 -> 39.6, 8 -> 49.6
#endif
constexpr int kNodeILP = TS_NODE_ILP;
// SIG: the domain has signalized nodes; WORK: load statistics requested
template <bool SIG, bool WORK>
__global__ void __launch_bounds__(256) k_node_warp(const NodeParams P_, const NodeWarpParams W) {
  const NodeParams P = with_time(P_);
  __shared__ unsigned long long red[8];
  const int lane = threadIdx.x & 31;
  const uint32_t gmask = (1u << P.G) - 1u;
  uint32_t crossings = 0;
  const int c0 = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * kNodeILP;
  NodeLane e[kNodeILP];
  uint64_t rec[kNodeILP];
  uint32_t sg[kNodeILP];
  int row[kNodeILP];
  bool act[kNodeILP];
#pragma unroll
  for (int k = 0; k < kNodeILP; k++) {  // stage 1: static lane data (before the wait)
    const int c = min(c0 + k, W.nchunks - 1), i = 32 * c + lane;  // node-lane index
    act[k] = c0 + k < W.nchunks;
    e[k] = W.lanes[i];
    sg[k] = SIG ? W.sig[i] : 0u;
    row[k] = W.nl_row[i];
  }
  // programmatic dependent launch: the records of S1 are the previous
  // kernel's output; once it is complete the next move kernel may start
  // its own prologue
  grid_dep_wait();
  grid_dep_launch();
#pragma unroll
  for (int k = 0; k < kNodeILP; k++)  // lane records of S1
    rec[k] = P.tail_rec[32 * min(c0 + k, W.nchunks - 1) + lane];
  Cand cd[kNodeILP];
  bool win[kNodeILP];
  uint8_t head[kNodeILP];
#pragma unroll
  for (int k = 0; k < kNodeILP; k++) {  // stage 2: candidates and winners
    const bool a = act[k] && e[k].lane_gid >= 0;
    if (!a) rec[k] = 0;
    const uint32_t nodemask = __match_any_sync(FULL, a ? (int)e[k].first : 64 + lane);
    const bool busy =
        (__ballot_sync(FULL, a && e[k].major && (((uint32_t)(rec[k] >> 44)) & gmask)) & nodemask) != 0u;
    cd[k] = Cand{false, -1, 0, 0, 0, 0, -1};
    if (a) cd[k] = node_candidate(P, rec[k], e[k].lane, e[k].out_base, e[k].tt, e[k].vk);
    // every candidate's target head, loaded before the winner is known (one
    // dependent load less on the chain; losers' loads are wasted; measured
    // -0.3 % window / -0.5 % steady per step)
    head[k] = cd[k].cand ? P.head_occ[cd[k].tgt] : (uint8_t)0;
    // signalized node (R23): red approaches have the virtual blocker, green
    // ones need no gap acceptance; otherwise priority + gap acceptance (R9)
    const bool eligible =
        cd[k].cand && ((SIG && (sg[k] >> 31)) ? sig_green(sg[k], P.t) : (e[k].major || !busy));
    const uint32_t grp = __match_any_sync(FULL, eligible ? cd[k].tgt : -1 - lane);
    win[k] = eligible && (__ffs(grp) - 1) == lane;
  }
#pragma unroll
  for (int k = 0; k < kNodeILP; k++) {  // stage 4: grants
    int ext = 0;
    const uint32_t cr0 = crossings;
    if (win[k]) ext = node_grant(P, cd[k], e[k].vk, head[k], crossings, (e[k].major & 2) != 0);
    if (act[k]) {
      P.ext[32 * (c0 + k) + lane] = (uint8_t)ext;
      if (row[k] >= 0) P.ext_row[row[k]] = (uint8_t)(front_final(rec[k]) ? kGmax : ext);
    }
    if (WORK) {  // load statistics: the node's lanes in range + its crossings
      const bool a = act[k] && e[k].lane_gid >= 0;
      const uint32_t nodemask = __match_any_sync(FULL, a ? (int)e[k].first : 64 + lane);
      const uint32_t wk = (uint32_t)((rec[k] >> 43) & 1) + (crossings - cr0);
      const uint32_t sum = __reduce_add_sync(nodemask, wk);
      if (a && (__ffs(nodemask) - 1) == lane && sum)
        atomicAdd(P.node_work + W.nl_node[32 * (c0 + k) + lane], (unsigned long long)sum);
    }
  }
  node_flush(P, crossings, red);
}

// general fallback: one thread per node (any in-degree)
__global__ void __launch_bounds__(128) k_node(const NodeParams P_) {
  const NodeParams P = with_time(P_);
  __shared__ unsigned long long red[4];
  const int ni = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t crossings = 0;
  if (ni < P.nnodes) {
    const int node = P.node_ids ? P.node_ids[ni] : ni;
    const uint32_t sg0 = P.node_sig ? P.node_sig[node] : 0u;  // phase-0 word (R23)
    const int a = P.in_off[node], b = P.in_off[node + 1];
    int maxcls = -2147483647;
    for (int i = a; i < b; i++) maxcls = max(maxcls, P.link_cls[P.in_list[i]]);
    const uint32_t gmask = (1u << P.G) - 1u;
    bool majorfree = true;
    for (int i = a; i < b; i++) {
      const int j = P.in_list[i];
      const int lg = P.link_lgid[j];
      for (int l = 0; l < P.link_lanes[j]; l++) {
        P.ext[lg + l] = 0;
        if (P.lane_row[lg + l] >= 0)
          P.ext_row[P.lane_row[lg + l]] = (uint8_t)(front_final(P.tail_rec[lg + l]) ? kGmax : 0);
        if (!(sg0 >> 31) && P.link_cls[j] == maxcls &&
            ((uint32_t)(P.tail_rec[lg + l] >> 44) & gmask))
          majorfree = false;
      }
    }
    const uint32_t cr0 = crossings;
    uint32_t in_range = 0;  // load statistics: lanes whose front vehicle is in range
    if (P.node_work)
      for (int i = a; i < b; i++) {
        const int j = P.in_list[i], lg = P.link_lgid[j];
        for (int l = 0; l < P.link_lanes[j]; l++) in_range += (uint32_t)((P.tail_rec[lg + l] >> 43) & 1);
      }
    constexpr int kMaxClaim = 128;  // target lanes taken (<= out-links x lanes)
    int claimed[kMaxClaim];
    int nclaimed = 0;
    for (int pass = 0; pass < 2; pass++) {
      if (pass == 1 && !majorfree) break;
      for (int i = a; i < b; i++) {
        const int j = P.in_list[i];
        if ((P.link_cls[j] == maxcls) != (pass == 0)) continue;
        const int lg = P.link_lgid[j];
        for (int l = 0; l < P.link_lanes[j]; l++) {
          const uint64_t rec = P.tail_rec[lg + l];
          const Cand cd = node_candidate(P, rec, l, P.out_off[node], P.tt_link[j], P.vmax_link[j]);
          if (!cd.cand) continue;
          if (sg0 >> 31) {  // signalized: phase 0 = maximal class, phase 1 = the rest
            const int c = (int)(sg0 & 1023u), g0 = (int)((sg0 >> 20) & 1023u);
            const int off = (int)((sg0 >> 10) & 1023u);
            const bool ph0 = P.link_cls[j] == maxcls;
            const uint32_t s1 = (1u << 31) | (uint32_t)c |
                                ((uint32_t)(((off - g0) % c + c) % c) << 10) |
                                ((uint32_t)(c - g0) << 20);
            if (!sig_green(ph0 ? sg0 : s1, P.t)) continue;
          }
          const int bit = cd.tgt;  // target lanes of a node are distinct global lanes
          bool taken = false;
          for (int q = 0; q < nclaimed; q++) taken |= claimed[q] == bit;
          if (taken) continue;
          if (nclaimed < kMaxClaim) claimed[nclaimed++] = bit;
          P.ext[lg + l] = (uint8_t)node_grant(P, cd, P.vmax_link[j], P.head_occ[cd.tgt],
                                              crossings);
          if (P.lane_row[lg + l] >= 0) P.ext_row[P.lane_row[lg + l]] = P.ext[lg + l];
        }
      }
    }
    if (P.node_work && in_range + (crossings - cr0))
      P.node_work[node] += (unsigned long long)(in_range + (crossings - cr0));
  }
  node_flush(P, crossings, red);
}

// ------------------------------------------------------- strip exchange
// dst[dslot ? dslot[j] : j] = src[sslot ? sslot[j] : j] for j < n, one
// 4-byte word per thread (pack: boundary strips -> send buffer; unpack:
// receive buffer -> mirror strips, H2/H7)
__global__ void __launch_bounds__(256) k_strip_copy(const Strip *src, const int32_t *sslot,
                                                    Strip *dst, const int32_t *dslot, int64_t n) {
  constexpr int kW = sizeof(Strip) / 4;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * kW) return;
  const int64_t j = i / kW;
  const int w = (int)(i - j * kW);
  const int64_t s = sslot ? sslot[j] : j, d = dslot ? dslot[j] : j;
  reinterpret_cast<uint32_t *>(dst + d)[w] = reinterpret_cast<const uint32_t *>(src + s)[w];
}

// direct delivery: one 4-byte word of one strip per thread
__global__ void __launch_bounds__(256) k_strip_direct(const DirectParams P) {
  constexpr int kW = sizeof(Strip) / 4;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.n * kW) return;
  const int64_t j = i / kW;
  const int w = (int)(i - j * kW);
  const int4 e = P.plan[j];
  reinterpret_cast<uint32_t *>(P.dst[e.z] + e.w)[w] =
      reinterpret_cast<const uint32_t *>(P.src[e.x] + e.y)[w];
}

// ------------------------------------------------------------ launchers
void launch_strip_direct(const DirectParams &p, void *stream) {
  if (p.n <= 0) return;
  const int64_t words = p.n * (int64_t)(sizeof(Strip) / 4);
  k_strip_direct<<<(unsigned)((words + 255) / 256), 256, 0, (cudaStream_t)stream>>>(p);
}
void launch_strip_copy(const Strip *src, const int32_t *sslot, Strip *dst, const int32_t *dslot,
                       int64_t n, void *stream) {
  if (n <= 0) return;
  const int64_t words = n * (int64_t)(sizeof(Strip) / 4);
  k_strip_copy<<<(unsigned)((words + 255) / 256), 256, 0, (cudaStream_t)stream>>>(src, sslot, dst,
                                                                                 dslot, n);
}
void launch_lc(const StepParams &p, int blocks, int threads, int smem, void *stream) {
  k_lc<<<blocks, threads, smem, (cudaStream_t)stream>>>(p);
}
void launch_step(const StepParams &p, int blocks, int threads, int smem, void *stream) {
  k_step<<<blocks, threads, smem, (cudaStream_t)stream>>>(p);
}
void launch_node(const NodeParams &p, void *stream) {
  if (p.nnodes <= 0) return;
  k_node<<<(p.nnodes + 127) / 128, 128, 0, (cudaStream_t)stream>>>(p);
}
__global__ void k_clock(int32_t *clock, unsigned long long *stats, int n, int advance) {
  if (advance) {
    if (threadIdx.x == 0) *clock += n;
    return;
  }
  const int t0 = *clock;
  for (int i = threadIdx.x; i < n * ST_N; i += blockDim.x)
    stats[(size_t)((t0 + 1 + i / ST_N) & (kHist - 1)) * ST_N + i % ST_N] = 0ull;
}
void launch_clock(int32_t *clock, unsigned long long *stats, int n, bool advance, void *stream) {
  k_clock<<<1, 256, 0, (cudaStream_t)stream>>>(clock, stats, n, advance ? 1 : 0);
}

void launch_node_warp(const NodeParams &p, const NodeWarpParams &w, void *stream, bool pdl) {
  if (w.nchunks <= 0) return;
  const int blocks = (w.nchunks + 8 * kNodeILP - 1) / (8 * kNodeILP);
  if (w.sig) {
    if (p.node_work) launch_pdl(k_node_warp<true, true>, blocks, 256, 0, stream, pdl, p, w);
    else launch_pdl(k_node_warp<true, false>, blocks, 256, 0, stream, pdl, p, w);
  } else {
    if (p.node_work) launch_pdl(k_node_warp<false, true>, blocks, 256, 0, stream, pdl, p, w);
    else launch_pdl(k_node_warp<false, false>, blocks, 256, 0, stream, pdl, p, w);
  }
}
void launch_hash(const StepParams &p, int blocks, int threads, int smem, void *stream,
                 unsigned long long *out) {
  k_hash<<<blocks, threads, smem, (cudaStream_t)stream>>>(p, out);
}

// The attribute is per function (process-wide), while every handle asks for
// its own size: only ever raise it, so no handle's launch falls below it.
cudaError_t set_smem_attrs(int bytes) {
  static int current[64] = {0};  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (bytes <= current[dev]) return cudaSuccess;
  current[dev] = bytes;
  cudaError_t e = cudaFuncSetAttribute(k_lc, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_hash, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int occupancy_blocks(int threads, int smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_step, threads, smem);
  return nb;
}

// the node checks' counters (bits, count) of the current device; reset
// zeroes them.  0, or -1 on a CUDA error; zeros in an unchecked build
int node_checks(unsigned int *v, int reset) {
#ifdef TS_CHECKED
  if (cudaMemcpyFromSymbol(v, g_ts_chk_node, 2 * sizeof(unsigned int)) != cudaSuccess) return -1;
  if (reset) {
    const unsigned int z[2] = {0u, 0u};
    if (cudaMemcpyToSymbol(g_ts_chk_node, z, sizeof z) != cudaSuccess) return -1;
  }
#else
  (void)reset;
  v[0] = v[1] = 0u;
#endif
  return 0;
}

}  // namespace tsim
