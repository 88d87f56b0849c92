// tsim_kernels.cu -- sm_100a kernels of the TRANSIMS CA time step
// (Nagel & Rickert, §3-§4; readings R1-R22 in DESIGN.md §3).
//
// State: one int8 code per lane-cell (0xFF empty, else velocity | out-slot
// << 3) and, per lane-row, the vids of its vehicles in cell order.  Gap
// queries use an occupancy bitmap (one bit per lane-cell): the 5-cell
// look-ahead / look-behind of PAPER.md:390-395 is a funnel-shifted 32-bit
// window and a ctz.
//
// Fast path (whole-link tiles, the HBM-bound configs):
//   k_rows       one warp per group of <= 32 lane-rows, one thread per row:
//                velocity update + move (H4/H5), node entrants, injection
//                (H6), and -- fused -- the lane change of step t+1 (H1)
//   k_node_warp  intersections (H3), one thread per incoming lane,
//                __match_any_sync picks one winner per target lane
// General path (tiles with 5-cell halos: long / periodic / split links):
//   k_lc, k_step one warp per tile, vehicles enumerated by rank
//   k_node       one thread per node
//   k_hash       state hash
#include <cuda_runtime.h>

#include "tsim_internal.h"

namespace tsim {

#define FULL 0xffffffffu

// ------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11) with the curand round and Weyl
// constants, counter (t, vid, 0, 0), key (k0, k1); only output word 0 is
// used (reading R3).  The zero counter words fold away in round 1.
__device__ __forceinline__ uint32_t philox_w0(uint32_t t, uint32_t vid, uint32_t k0,
                                              uint32_t k1) {
  uint32_t c0 = t, c1 = vid, c2 = 0u, c3 = 0u;
#pragma unroll
  for (int r = 0; r < 10; r++) {
    if (r) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  return c0;
}

// NaSch velocity update (PAPER.md:330-335 rules (i)-(iii); R15):
// accelerate, clamp to the gap, random slowdown (draw skipped when v2 = 0,
// which cannot change the result).
__device__ __forceinline__ int nasch_v3(int v, int Vk, int g, uint32_t t, uint32_t vid,
                                        uint32_t k0, uint32_t k1, uint64_t p32) {
  int v2 = min(min(v + 1, Vk), g);
  if (v2 > 0 && (uint64_t)philox_w0(t, vid, k0, k1) < p32) v2 -= 1;
  return v2;
}

// ---------------------------------------------------------- state hash
__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}
__device__ __forceinline__ uint64_t vmix(int vid, int link, int lane, int cell, int v) {
  uint64_t a = (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)link << 32);
  uint64_t b = (uint64_t)(uint32_t)cell | ((uint64_t)(uint32_t)lane << 32) |
               ((uint64_t)(uint32_t)v << 40);
  return fmix64(fmix64(a) + b * 0x9E3779B97F4A7C15ULL);
}

// ------------------------------------------------------------ bit helpers
// 4 code bytes -> 4 occupancy bits (occupied iff bit 7 clear)
__device__ __forceinline__ uint32_t occ4(uint32_t w) {
  return ((((~w) & 0x80808080u) >> 7) * 0x01020408u) >> 24;
}

// bits[0] and bits[nwords+1..] are zero pads so that windows never branch
__device__ __forceinline__ void build_bits(const uint8_t *c, uint32_t *bits, int nwords,
                                           int lane) {
  for (int j = lane; j < nwords; j += 32) {
    const uint4 *p = reinterpret_cast<const uint4 *>(c + 32 * j);
    uint4 a = p[0], b = p[1];
    bits[j + 1] = occ4(a.x) | occ4(a.y) << 4 | occ4(a.z) << 8 | occ4(a.w) << 12 |
                  occ4(b.x) << 16 | occ4(b.y) << 20 | occ4(b.z) << 24 | occ4(b.w) << 28;
  }
  if (lane == 0) {
    bits[0] = 0u;
    bits[nwords + 1] = 0u;
    bits[nwords + 2] = 0u;
  }
}

__device__ __forceinline__ int occupied(const uint32_t *bits, int q) {
  return (bits[(q >> 5) + 1] >> (q & 31)) & 1u;
}
__device__ __forceinline__ void set_bit(uint32_t *bits, int q) {
  atomicOr(bits + (q >> 5) + 1, 1u << (q & 31));
}
// bit i = position s+i
__device__ __forceinline__ uint32_t win_at(const uint32_t *bits, int s) {
  return __funnelshift_r(bits[(s >> 5) + 1], bits[(s >> 5) + 2], s & 31);
}
// bit i = position q+1+i
__device__ __forceinline__ uint32_t win_ahead(const uint32_t *bits, int q) {
  return win_at(bits, q + 1);
}
// bit i = position q-1-i
__device__ __forceinline__ uint32_t win_behind(const uint32_t *bits, int q) {
  return __brev(win_at(bits, q - 32));
}

__device__ __forceinline__ int ctz32(uint32_t m) { return m ? __ffs(m) - 1 : 32; }
__device__ __forceinline__ uint32_t low_mask(int n) {  // bits [0, n), n in [0, 32]
  return n >= 32 ? FULL : ((1u << n) - 1u);
}

__device__ __forceinline__ uint32_t range_mask(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 32);
  if (lo >= hi) return 0u;
  return low_mask(hi) & ~low_mask(lo);
}

// ------------------------------------------------------------- tile ctx
struct Acc {
  uint64_t hash, sumv;
  uint32_t active, arr, inj, lc, work;
};

__device__ __forceinline__ void acc_place(Acc &a, bool hash, int vid, int link, int l, int x,
                                          int v) {
  a.active++;
  a.sumv += v;
  if (hash) a.hash += vmix(vid, link, l, x, v);
}

__device__ void flush_acc(const StepParams &P, Acc &a, int slot_t, unsigned long long *smem_red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t h = a.hash, sv = a.sumv;
  uint32_t act = a.active, arr = a.arr, inj = a.inj, lc = a.lc;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    h += __shfl_down_sync(FULL, h, o);
    sv += __shfl_down_sync(FULL, sv, o);
    act += __shfl_down_sync(FULL, act, o);
    arr += __shfl_down_sync(FULL, arr, o);
    inj += __shfl_down_sync(FULL, inj, o);
    lc += __shfl_down_sync(FULL, lc, o);
  }
  if (lane == 0) {
    unsigned long long *r = smem_red + warp * 8;
    r[0] = h;
    r[1] = act;
    r[2] = arr;
    r[3] = inj;
    r[4] = lc;
    r[5] = sv;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    unsigned long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += smem_red[w * 8 + threadIdx.x];
    const int idx = threadIdx.x == 0 ? ST_HASH : threadIdx.x == 1 ? ST_ACTIVE
                  : threadIdx.x == 2 ? ST_ARR : threadIdx.x == 3 ? ST_INJ
                  : threadIdx.x == 4 ? ST_LC : ST_SUMV;
    unsigned long long *st = P.stats + (size_t)(slot_t & (kHist - 1)) * ST_N;
    if (s) atomicAdd(st + idx, s);
  }
  __syncthreads();
}

// ====================================================================
// General path: one warp per tile (halo tiles, split links, any layout)
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

// owned positions of word j
__device__ __forceinline__ uint32_t owned_mask(const TileCtx &T, int j) {
  // a word spans every row it intersects (rows can be as short as 12 cells)
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

// stage S codes of the tile (+ 5-cell halos from strips) into smem
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

// cells ahead / behind inside the lane's valid range (R2)
__device__ __forceinline__ int row_hi(const TileCtx &T, int l) {
  return l * T.S + T.HP + T.w + (T.has_dn ? kGmax : 0);
}
__device__ __forceinline__ int row_lo(const TileCtx &T, int l) {
  return l * T.S + T.HP - (T.has_up ? kGmax : 0);
}

// lane-change geometry shared by both paths: [lo, hi) is the valid range of
// the lane-row in the flat bitmap (positions below lo are before the link
// start and count as empty; the row ends at hi).
__device__ __forceinline__ int ahead_in(const uint32_t *bits, int q, int hi) {
  return min(min(ctz32(win_ahead(bits, q)), kGmax), hi - q - 1);
}
__device__ __forceinline__ int behind_in(const uint32_t *bits, int q, int lo) {
  uint32_t r = win_behind(bits, q);
  int nvalid = q - lo;
  if (nvalid < 32) r &= low_mask(nvalid);
  return min(ctz32(r), kGmax);
}

// O1 §LC decision (R4-R7).  q: position of the vehicle,
// q2 = q + dir*stride the target cell; lanes l (own) and l2 (target) with
// valid ranges [lo, hi) / [lo2, hi2); d = cells to the link end.
__device__ __forceinline__ bool lc_rule(const uint32_t *bits, int q, int q2, int lo, int hi,
                                        int lo2, int hi2, int code, int l, int l2, int L,
                                        int dir, int d, uint32_t tt, bool periodic, int Vk,
                                        int D) {
  if (occupied(bits, q2)) return false;
  const int v = code & 7, slot = code >> 3;
  int set = 0;  // 0 all lanes, 1 {0} (right turn), 2 {L-1} (left turn)
  if (slot != kSlotFinal && !periodic) {
    int tty = (tt >> (2 * slot)) & 3;
    set = tty == 0 ? 0 : (tty == 2 ? 1 : 2);
  }
  const bool own_ok = set == 0 || (set == 1 ? l == 0 : l == L - 1);
  if (!own_ok) {  // turn-motivated, only towards the allowed lane
    const bool toward = (set == 1 && dir < 0) || (set == 2 && dir > 0);
    if (!toward) return false;
    int rf = min(v + 1, Vk), rb = Vk;
    if (d < D) {  // R6: desperation over the last D cells
      rf = (rf * d) / D;
      rb = (rb * d) / D;
    }
    return ahead_in(bits, q2, hi2) >= rf && behind_in(bits, q2, lo2) >= rb;
  }
  const bool tgt_ok = set == 0 || (set == 1 ? l2 == 0 : l2 == L - 1);
  if (!tgt_ok) return false;
  const int g = ahead_in(bits, q, hi);  // R5: the other lane is faster
  return g < v + 1 && ahead_in(bits, q2, hi2) > g && behind_in(bits, q2, lo2) >= Vk;
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
      s->tail_cur[j] = vt >= 0 ? P.cursor[vt] : -1;
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
        P.tail_rec[T.d.lane_gid + l] = rec;
      }
      if (T.d.flags & kFirst)
        P.head_occ[T.d.lane_gid + l] = (uint8_t)(win_at(T.bout, l * T.S + T.HP) & 31u);
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
                                         int vid, bool ghost, int Vk) {
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
  else g = min(kGmax, lim + (int)P.ext[T.d.lane_gid + l]);  // node grant (H3)
  const int v3 = nasch_v3(v, Vk, g, (uint32_t)P.t, (uint32_t)vid, P.k0, P.k1, P.p32);
  int y = x + v3;
  if (periodic && y >= T.d.n) y -= T.d.n;
  const int yl = y - T.d.a;
  if (yl >= 0 && yl < T.w) {
    place(T, l * T.S + T.HP + yl, (uint8_t)(v3 | (slot << 3)), vid);
    acc_place(acc, P.mode & kModeHash, vid, T.d.link, l, y, v3);
  } else if (!periodic && y > T.d.n - 1 && !ghost) {
    if (slot == kSlotFinal) {  // exit to parking
      P.arr_time[vid] = P.t + 1;
      acc.arr++;
    }
    // else: node crossing; k_node placed it on the next link
  }
  if (!ghost) acc.work++;
}

// injection from parking (R13) by one thread: walks the
// link's pending list in (departure, vid) order; cell_free / place_fn act
// on lane 0 of the tile.
template <class FreeFn, class PlaceFn>
__device__ __forceinline__ void inject_link(const StepParams &P, int k, int a, int w, bool first,
                                            FreeFn cell_free, PlaceFn place_fn) {
  const int e = P.pend_off[k + 1];
  int h = P.pend_head[k];
  const int tn = P.t + 1;
  for (int i = h; i < e; i++) {
    const int vid = P.pend_list[i];
    if (P.dep[vid] > tn) break;
    if (P.inj_time[vid] <= P.t) continue;
    const int ec = P.entry[vid];
    if (ec < a || ec >= a + w) continue;
    if (!cell_free(ec - a)) continue;  // retry next step
    const int64_t ro = P.route_off[vid];
    const int slot0 = (P.route_off[vid + 1] - ro > 1) ? P.out_pos[P.route[ro + 1]] : kSlotFinal;
    P.inj_time[vid] = tn;
    place_fn(ec - a, (uint8_t)(slot0 << 3), vid);
  }
  if (first) {
    while (h < e && P.inj_time[P.pend_list[h]] <= tn) h++;
    P.pend_head[k] = h;
  }
}

// ------------------------------------------------------------- k_lc
__global__ void __launch_bounds__(256) k_lc(const StepParams P) {
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
__global__ void __launch_bounds__(256) k_step(const StepParams P) {
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
          if (occupied(T.bin, q))
            move_one(P, T, acc, q, P.strip_in[P.halo_up[T.d.strip] + l].tail_vid[j], true, Vk);
        }
      }
      // entrants granted by k_node (H3/H5): at most one per lane
      if ((T.d.flags & kFirst) && lane < T.L) {
        uint64_t rec = P.entr[T.d.lane_gid + lane];
        if ((uint32_t)(rec >> 43) == ((uint32_t)(P.t + 1) & 0x1FFFFFu)) {
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

// ====================================================================
// Fast path: k_rows -- one warp per group of whole-link tiles, one thread
// per lane-row.  All vehicles of a row are processed by its thread in cell
// order; the in-lane order is preserved by the move, so the row's vid list
// is streamed in and out with 128-bit accesses.
// ====================================================================
struct VidReader {  // sequential 128-bit reader of a row's vid list
  const int32_t *p;
  int i;
  uint4 buf;
  __device__ __forceinline__ int next() {
    if ((i & 3) == 0) buf = __ldg(reinterpret_cast<const uint4 *>(p + i));
    const int k = i & 3;
    i++;
    return k == 0 ? (int)buf.x : k == 1 ? (int)buf.y : k == 2 ? (int)buf.z : (int)buf.w;
  }
};

struct VidWriter {  // sequential 128-bit writer of a row's vid list
  int32_t *p;
  int j;
  uint4 buf;
  __device__ __forceinline__ void put(int v) {
    const int k = j & 3;
    if (k == 0) buf.x = v;
    else if (k == 1) buf.y = v;
    else if (k == 2) buf.z = v;
    else buf.w = v;
    j++;
    if (k == 3) __stcs(reinterpret_cast<uint4 *>(p + j - 4), buf);
  }
  __device__ __forceinline__ void flush() {
    const int k = j & 3, b = j & ~3;
    if (k > 0) p[b] = (int)buf.x;
    if (k > 1) p[b + 1] = (int)buf.y;
    if (k > 2) p[b + 2] = (int)buf.z;
  }
};

// bits of row cells [32*wj, 32*wj+32) (row starting at flat position s,
// w cells)
__device__ __forceinline__ uint32_t row_word(const uint32_t *bits, int s, int w, int wj) {
  return win_at(bits, s + 32 * wj) & low_mask(w - 32 * wj);
}

// vid of an entrant / injected vehicle of row `row` at cell x
__device__ __forceinline__ int special_vid(const int32_t *ent, const int32_t *injx,
                                           const int32_t *injv, int ninj, int row, int x) {
  if (ent[32 + row] == x) return ent[row];
  const int key = (row << 16) | x;
  for (int k = 0; k < ninj; k++)
    if (injx[k] == key) return injv[k];
  return -1;
}

__global__ void __launch_bounds__(128) k_rows(const StepParams P, const RowsParams R) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long red[4 * 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  const RowsLayout &Y = R.lay;
  uint8_t *base = smem + warp * Y.bytes;
  uint8_t *cin = base + Y.o_cin, *cout = base + Y.o_cout;
  uint32_t *bin = reinterpret_cast<uint32_t *>(base + Y.o_bin);
  uint32_t *bmid = reinterpret_cast<uint32_t *>(base + Y.o_bmid);
  uint32_t *bspec = reinterpret_cast<uint32_t *>(base + Y.o_bspec);
  uint32_t *blv = reinterpret_cast<uint32_t *>(base + Y.o_bleave);
  int32_t *ent = reinterpret_cast<int32_t *>(base + Y.o_ent);
  int32_t *injx = reinterpret_cast<int32_t *>(base + Y.o_injx);
  int32_t *injv = reinterpret_cast<int32_t *>(base + Y.o_injv);
  int32_t *misc = reinterpret_cast<int32_t *>(base + Y.o_misc);
  const bool hash = (P.mode & kModeHash) != 0;
  const bool lc_next = (P.mode & kModeLC) != 0;
  const int dir = ((P.t + 1) & 1) ? -1 : +1;  // R4, lane change of step t+1
  Acc acc = {};
  Acc acc_next = {};
  for (int g = blockIdx.x * (blockDim.x >> 5) + warp; g < R.ngroups; g += nwarps_total) {
    const GroupDesc G = R.groups[g];
    const int64_t off0 = P.tiles[G.t0].off;
    const int nw = (G.bytes + 31) >> 5;
    // ---- stage the group's codes, clear the work bitmaps
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
      ent[32 + lane] = -1;  // entrant cell per row
    }
    __syncwarp();
    build_bits(cin, bin, nw, lane);
    __syncwarp();
    // ---- this thread's row
    const bool active = lane < G.nrows;
    TileDesc d;
    int l = 0, s = 0, Wp = 4, Vk = 1, nrw = 0;
    if (active) {
      const int rm = R.rowmap[(size_t)g * 32 + lane];
      l = rm & 7;
      d = P.tiles[G.t0 + (rm >> 3)];
      Wp = row_pitch(d.w);
      s = (int)(d.off - off0) + l * Wp;
      Vk = P.vmax_link[d.link];
      nrw = (d.w + 31) >> 5;
    }
    const int64_t rbase = active ? d.off + (int64_t)l * Wp : 0;
    const uint32_t work0 = acc.work;
    // ---- velocity update + move (H4/H5)
    if (active && (P.mode & kModeMove)) {
      VidReader rd{P.vid_in + rbase, 0, make_uint4(0, 0, 0, 0)};
      for (int wj = 0; wj < nrw; wj++) {
        uint32_t m = row_word(bin, s, d.w, wj);
        while (m) {
          const int x = 32 * wj + __ffs(m) - 1;
          m &= m - 1u;
          const int q = s + x;
          const int code = cin[q];
          const int v = code & 7, slot = code >> 3;
          const int vid = rd.next();
          const int lim = min(kGmax, d.w - 1 - x);
          const uint32_t ma = win_ahead(bin, q) & low_mask(lim);
          int gp;
          if (ma) gp = __ffs(ma) - 1;
          else if (lim == kGmax || slot == kSlotFinal) gp = kGmax;  // R12 open end
          else gp = min(kGmax, lim + (int)P.ext[d.lane_gid + l]);   // node grant
          const int v3 = nasch_v3(v, Vk, gp, (uint32_t)P.t, (uint32_t)vid, P.k0, P.k1, P.p32);
          const int y = x + v3;
          if (y < d.w) {
            cout[s + y] = (uint8_t)(v3 | (slot << 3));
            set_bit(bmid, s + y);
            acc_place(acc, hash, vid, d.link, l, y, v3);
          } else if (slot == kSlotFinal) {  // exit to parking
            P.arr_time[vid] = P.t + 1;
            acc.arr++;
          }  // else: crossed the node; k_node_warp placed it
          acc.work++;
        }
      }
      // entrant granted by the node kernel
      if (d.flags & kFirst) {
        const uint64_t rec = P.entr[d.lane_gid + l];
        if ((uint32_t)(rec >> 43) == ((uint32_t)(P.t + 1) & 0x1FFFFFu)) {
          const int vid = (int)(uint32_t)rec;
          const uint8_t code = (uint8_t)(rec >> 32);
          const int y = (int)((rec >> 40) & 7);
          cout[s + y] = code;
          set_bit(bmid, s + y);
          set_bit(bspec, s + y);
          ent[lane] = vid;
          ent[32 + lane] = y;
          acc_place(acc, hash, vid, d.link, l, y, code & 7);
        }
      }
      if ((P.mode & kModeInject) && l == 0 && P.pend_off[d.link + 1] > P.pend_head[d.link]) {
        const int row = lane;
        inject_link(
            P, d.link, 0, d.w, true, [&](int x) { return cout[s + x] == kEmpty; },
            [&](int x, uint8_t code, int vid) {
              cout[s + x] = code;
              set_bit(bmid, s + x);
              set_bit(bspec, s + x);
              const int k = atomicAdd(misc, 1);
              injx[k] = (row << 16) | x;
              injv[k] = vid;
              acc.inj++;
              acc_place(acc, hash, vid, d.link, 0, x, 0);
            });
      }
    }
    __syncwarp();
    // ---- lane change of step t+1 on the post-move state (H1, fused)
    const int l2 = l + dir;
    if (active && lc_next && l2 >= 0 && l2 < d.L) {
      const uint32_t tt = P.tt_link[d.link];
      const int s2 = s + dir * Wp;
      int nch = 0;
      for (int wj = 0; wj < nrw; wj++) {
        uint32_t m = row_word(bmid, s, d.w, wj);
        while (m) {
          const int x = 32 * wj + __ffs(m) - 1;
          m &= m - 1u;
          if (lc_rule(bmid, s + x, s2 + x, s, s + d.w, s2, s2 + d.w, cout[s + x], l, l2, d.L, dir,
                      d.w - 1 - x, tt, false, Vk, P.D)) {
            set_bit(blv, s + x);
            nch++;
          }
        }
      }
      acc_next.lc += nch;
    }
    // final codes are assembled in cin
    for (int i = lane; i < 2 * nw; i += 32)
      reinterpret_cast<uint4 *>(cin)[i] = make_uint4(FULL, FULL, FULL, FULL);
    __syncwarp();
    // ---- final state of the row: own post-move vehicles that stay, plus
    // arrivals from the row l - dir; vid list streamed out in cell order
    if (active) {
      const int ls = l - dir;  // source row of arrivals (thread lane - dir)
      const bool has_src = lc_next && ls >= 0 && ls < d.L;
      const int ss = s - dir * Wp;
      VidReader rd{P.vid_in + rbase, 0, make_uint4(0, 0, 0, 0)};
      VidWriter wr{P.vid_out + rbase, 0, make_uint4(0, 0, 0, 0)};
      uint32_t tocc = 0, hocc = 0;
      int fx = -1, fvid = 0, fcode = 0;
      for (int wj = 0; wj < nrw; wj++) {
        const uint32_t mid = row_word(bmid, s, d.w, wj);
        const uint32_t lv = lc_next ? row_word(blv, s, d.w, wj) : 0u;
        const uint32_t arr = has_src ? row_word(blv, ss, d.w, wj) : 0u;
        const uint32_t sp = row_word(bspec, s, d.w, wj);
        uint32_t u = mid | arr;
        while (u) {
          const int b = __ffs(u) - 1;
          u &= u - 1u;
          const uint32_t bit = 1u << b;
          const int x = 32 * wj + b;
          int vid, code;
          if (mid & bit) {
            vid = (sp & bit) ? special_vid(ent, injx, injv, misc[0], lane, x) : rd.next();
            if (lv & bit) continue;  // changed to row l + dir
            code = cout[s + x];
          } else {  // arrived from row ls at the same cell
            code = cout[ss + x];
            if (occupied(bspec, ss + x)) {
              vid = special_vid(ent, injx, injv, misc[0], lane - dir, x);
            } else {  // rank among the source row's input-derived vehicles
              int idx = 0;
              for (int wk = 0; wk <= (x >> 5); wk++) {
                uint32_t mm = row_word(bmid, ss, d.w, wk) & ~row_word(bspec, ss, d.w, wk);
                if (wk == (x >> 5)) mm &= low_mask(x & 31);
                idx += __popc(mm);
              }
              vid = P.vid_in[d.off + (int64_t)ls * Wp + idx];
            }
          }
          wr.put(vid);
          cin[s + x] = (uint8_t)code;
          if (x >= d.w - kGmax) {
            tocc |= 1u << (d.w - 1 - x);
            fx = x;
            fvid = vid;
            fcode = code;
          }
          if (x < kGmax) hocc |= 1u << x;
        }
      }
      wr.flush();
      if (lc_next) {  // the output is S1(t+1): node records for k_node_warp
        if (d.flags & kLast) {
          uint64_t rec = (uint64_t)tocc << 44;
          if (fx >= 0)
            rec |= (uint64_t)(uint32_t)fvid | ((uint64_t)fcode << 32) |
                   ((uint64_t)(d.w - 1 - fx) << 40) | (1ull << 43);
          P.tail_rec[d.lane_gid + l] = rec;
        }
        if (d.flags & kFirst) P.head_occ[d.lane_gid + l] = (uint8_t)hocc;
      }
    }
    __syncwarp();
    {
      uint4 *dst = reinterpret_cast<uint4 *>(P.code_out + off0);
      const uint4 *src = reinterpret_cast<const uint4 *>(cin);
      for (int i = lane; i < (G.bytes >> 4); i += 32) __stcs(dst + i, src[i]);
    }
    __syncwarp();
    if ((P.mode & kModeWork) && P.link_work && active) {  // load statistics
      const uint32_t wk = acc.work - work0;
      if (wk) atomicAdd(P.link_work + d.link, (unsigned long long)wk);
    }
  }
  flush_acc(P, acc, P.t + 1, red);
  if (lc_next) flush_acc(P, acc_next, P.t + 2, red);
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

// ------------------------------------------------------------- nodes
// O1 §Node (R8-R10).  Candidates are the front vehicles
// of the incoming lanes that want to pass the stop line (d < min(v+1, V));
// majors first, minors only if the last G cells of every major lane are
// empty; one winner per target lane in (class, link, lane) order; the
// winner is granted the entry space E and, if its velocity takes it past
// the stop line, is written as the entrant of the target lane.
struct Cand {
  bool cand;
  int tgt, k2, l2, d, v, vid;
};

__device__ __forceinline__ Cand node_candidate(const NodeParams &P, uint64_t rec, int link,
                                               int lane, int node) {
  Cand c{false, -1, 0, 0, 0, 0, 0};
  if (!((rec >> 43) & 1)) return c;
  const int code = (int)((rec >> 32) & 0xFF);
  c.d = (int)((rec >> 40) & 7);
  c.v = code & 7;
  const int slot = code >> 3;
  if (slot == kSlotFinal || !(c.d < min(c.v + 1, (int)P.vmax_link[link]))) return c;
  c.k2 = P.out_list[P.out_off[node] + slot];
  const int tty = (P.tt_link[link] >> (2 * slot)) & 3;
  const int L2 = P.link_lanes[c.k2];
  c.l2 = tty == 0 ? min(lane, L2 - 1) : (tty == 2 ? 0 : L2 - 1);  // R8
  c.tgt = P.link_lgid[c.k2] + c.l2;
  c.vid = (int)(uint32_t)rec;
  c.cand = true;
  return c;
}

// the winner's grant: returns ext; writes the entrant record if it crosses
__device__ __forceinline__ int node_grant(const NodeParams &P, const Cand &c, int link,
                                          uint32_t &crossings) {
  const int E = min(ctz32((uint32_t)P.head_occ[c.tgt] | 0x20u), min(kGmax, P.link_ncell[c.k2]));
  if (E == 0) return 0;
  const int v3 = nasch_v3(c.v, P.vmax_link[link], min(kGmax, c.d + E), (uint32_t)P.t,
                          (uint32_t)c.vid, P.k0, P.k1, P.p32);
  if (v3 > c.d) {
    const int y2 = v3 - c.d - 1;
    const int r = P.cursor[c.vid];
    P.cursor[c.vid] = r + 1;
    const int64_t ro = P.route_off[c.vid];
    const int m = (int)(P.route_off[c.vid + 1] - ro);
    const int nslot = (r + 2 < m) ? P.out_pos[P.route[ro + r + 2]] : kSlotFinal;
    P.entr[c.tgt] = (uint64_t)(uint32_t)c.vid | ((uint64_t)(v3 | (nslot << 3)) << 32) |
                    ((uint64_t)y2 << 40) | ((uint64_t)((P.t + 1) & 0x1FFFFF) << 43);
    crossings++;
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
// thread with that target (__match_any_sync)
__global__ void __launch_bounds__(256) k_node_warp(const NodeParams P, const NodeWarpParams W) {
  __shared__ unsigned long long red[8];
  const int lane = threadIdx.x & 31;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  const uint32_t gmask = (1u << P.G) - 1u;
  uint32_t crossings = 0;
  for (int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); c < W.nchunks;
       c += nwarps_total) {
    const int a = W.chunk_off[c], n = W.chunk_off[c + 1] - a;
    const bool act = lane < n;
    NodeLane e{0, 0, -1 - lane, 0, 0};
    uint64_t rec = 0;
    if (act) {
      e = W.lanes[a + lane];
      rec = P.tail_rec[e.lane_gid];
    }
    const uint32_t nodemask = __match_any_sync(FULL, e.node);
    const bool busy = (__ballot_sync(FULL, act && e.major && (((uint32_t)(rec >> 44)) & gmask)) &
                       nodemask) != 0u;
    Cand cd{false, -1, 0, 0, 0, 0, 0};
    if (act) cd = node_candidate(P, rec, e.link, e.lane, e.node);
    const bool eligible = cd.cand && (e.major || !busy);
    const int key = eligible ? cd.tgt : -1 - lane;
    const uint32_t grp = __match_any_sync(FULL, key);
    int ext = 0;
    if (eligible && (__ffs(grp) - 1) == lane) ext = node_grant(P, cd, e.link, crossings);
    if (act) P.ext[e.lane_gid] = (uint8_t)ext;
  }
  node_flush(P, crossings, red);
}

// general fallback: one thread per node (any in-degree)
__global__ void __launch_bounds__(128) k_node(const NodeParams P) {
  __shared__ unsigned long long red[4];
  const int node = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t crossings = 0;
  if (node < P.nnodes) {
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
        if (P.link_cls[j] == maxcls && ((uint32_t)(P.tail_rec[lg + l] >> 44) & gmask))
          majorfree = false;
      }
    }
    uint32_t claimed[4] = {0u, 0u, 0u, 0u};  // (slot, lane) targets taken
    for (int pass = 0; pass < 2; pass++) {
      if (pass == 1 && !majorfree) break;
      for (int i = a; i < b; i++) {
        const int j = P.in_list[i];
        if ((P.link_cls[j] == maxcls) != (pass == 0)) continue;
        const int lg = P.link_lgid[j];
        for (int l = 0; l < P.link_lanes[j]; l++) {
          const uint64_t rec = P.tail_rec[lg + l];
          const Cand cd = node_candidate(P, rec, j, l, node);
          if (!cd.cand) continue;
          const int slot = (int)((rec >> 35) & 15);
          const int bit = slot * 8 + cd.l2;
          if (claimed[bit >> 5] & (1u << (bit & 31))) continue;
          claimed[bit >> 5] |= 1u << (bit & 31);
          P.ext[lg + l] = (uint8_t)node_grant(P, cd, j, crossings);
        }
      }
    }
  }
  node_flush(P, crossings, red);
}

// ------------------------------------------------------------ launchers
void launch_lc(const StepParams &p, int blocks, int threads, int smem, void *stream) {
  k_lc<<<blocks, threads, smem, (cudaStream_t)stream>>>(p);
}
void launch_step(const StepParams &p, int blocks, int threads, int smem, void *stream) {
  k_step<<<blocks, threads, smem, (cudaStream_t)stream>>>(p);
}
void launch_rows(const StepParams &p, const RowsParams &r, int blocks, int threads, int smem,
                 void *stream) {
  k_rows<<<blocks, threads, smem, (cudaStream_t)stream>>>(p, r);
}
void launch_node(const NodeParams &p, void *stream) {
  if (p.nnodes <= 0) return;
  k_node<<<(p.nnodes + 127) / 128, 128, 0, (cudaStream_t)stream>>>(p);
}
void launch_node_warp(const NodeParams &p, const NodeWarpParams &w, void *stream) {
  if (w.nchunks <= 0) return;
  const int blocks = (w.nchunks + 7) / 8;
  k_node_warp<<<blocks, 256, 0, (cudaStream_t)stream>>>(p, w);
}
void launch_hash(const StepParams &p, int blocks, int threads, int smem, void *stream,
                 unsigned long long *out) {
  k_hash<<<blocks, threads, smem, (cudaStream_t)stream>>>(p, out);
}

cudaError_t set_smem_attrs(int bytes) {
  cudaError_t e = cudaFuncSetAttribute(k_lc, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(k_hash, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}
cudaError_t set_rows_smem(int bytes) {
  return cudaFuncSetAttribute(k_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int occupancy_blocks(int threads, int smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_step, threads, smem);
  return nb;
}
int occupancy_rows(int threads, int smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows, threads, smem);
  return nb;
}

}  // namespace tsim
