// tsim_kernels.cu -- sm_100a kernels of the TRANSIMS CA time step
// (Nagel & Rickert, §3-§4; readings R1-R22 in DESIGN.md §3).
//
// Work unit = one tile (cells [a, a+w) of every lane of one link), owned by
// one warp.  The warp stages the tile's int8 cell codes in shared memory,
// builds an occupancy bitmap (one bit per lane-cell) and answers every gap
// query of the rules with a 32-bit funnel-shifted window of that bitmap:
// the 5-cell look-ahead / look-behind of PAPER.md:390-395 is a ctz / clz.
// Vehicles are enumerated by rank (prefix popcount), so the compact vid
// list of the tile is read and written fully coalesced, ~8 B per vehicle.
//
// Kernels:
//   k_lc    S(t)  -> S1(t)   lane change (H1), writes node records + strips
//   k_node  S1(t) -> ext/entrants   intersections (H3), one thread per node
//   k_step  S1(t) -> S(t+1)  velocity update + move (H4/H5), entrants,
//                            injection (H6); optionally fused lane change of
//                            step t+1 (-> S1(t+1)) when tiles are whole links
//   k_hash  S(t) -> state hash
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

// ------------------------------------------------------------ tile ctx
struct Acc {
  uint64_t hash, sumv;
  uint32_t active, arr, inj, lc, work;
};

struct TileCtx {
  TileDesc d;
  int S, HP, nwords, L, w;
  int has_up, has_dn, ghosts;
  uint8_t *cin, *cout;
  uint32_t *bin, *bout;
  int32_t *vout;
  uint16_t *vpos, *dpos;
};

__device__ __forceinline__ void tile_setup(TileCtx &T, const TileDesc *tiles, int ti,
                                           const WarpLayout &lay, uint8_t *base) {
  T.d = tiles[ti];
  T.L = T.d.L;
  T.w = T.d.w;
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
}

__device__ __forceinline__ int lane_of(const TileCtx &T, int p) {
  int l = 0;
  while (l + 1 < T.L && p >= (l + 1) * T.S) l++;
  return l;
}

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

// bit i = position q+1+i
__device__ __forceinline__ uint32_t win_ahead(const uint32_t *bits, int q) {
  int s = q + 1;
  return __funnelshift_r(bits[(s >> 5) + 1], bits[(s >> 5) + 2], s & 31);
}

// bit i = position q-1-i
__device__ __forceinline__ uint32_t win_behind(const uint32_t *bits, int q) {
  int s = q - 32;
  return __brev(__funnelshift_r(bits[(s >> 5) + 1], bits[(s >> 5) + 2], s & 31));
}

__device__ __forceinline__ int ctz32(uint32_t m) { return m ? __ffs(m) - 1 : 32; }

__device__ __forceinline__ uint32_t range_mask(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 32);
  if (lo >= hi) return 0u;
  uint32_t up = hi == 32 ? FULL : ((1u << hi) - 1u);
  return up & ~((1u << lo) - 1u);
}

// owned positions of word j
__device__ __forceinline__ uint32_t owned_mask(const TileCtx &T, int j) {
  int p0 = 32 * j;
  if (!T.HP) return range_mask(0, T.L * T.w - p0);
  int l = p0 / T.S;
  uint32_t m = 0u;
  for (int k = l; k <= l + 1 && k < T.L; k++)
    m |= range_mask(k * T.S + T.HP - p0, k * T.S + T.HP + T.w - p0);
  return m;
}

// rank -> position for the owned vehicles of `bits`; returns the count
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
  return total;
}

// stage S codes of the tile (+ 5-cell halos from strips) into smem
__device__ void load_codes(const TileCtx &T, const uint8_t *gcode, const Strip *strips,
                           const int32_t *halo_up, const int32_t *halo_dn, int lane) {
  const int nb = T.nwords * 32;
  if (!T.HP) {
    const int n16 = (T.L * T.w + 15) >> 4;
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
        T.cin[l * T.S + T.HP + x] = gcode[T.d.off + (int64_t)l * T.w + x];
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
__device__ __forceinline__ int ahead_lc(const TileCtx &T, const uint32_t *bits, int q, int l) {
  return min(min(ctz32(win_ahead(bits, q)), kGmax), row_hi(T, l) - q - 1);
}
__device__ __forceinline__ int behind_lc(const TileCtx &T, const uint32_t *bits, int q, int l) {
  uint32_t r = win_behind(bits, q);
  int nvalid = q - row_lo(T, l);  // below the link start counts as empty
  if (nvalid < 32) r &= (1u << nvalid) - 1u;
  return min(ctz32(r), kGmax);
}

// O1 §LC decision (R4-R7) of the vehicle at q on the
// state (c, bits); returns the target position or -1.
__device__ int lc_decide(const StepParams &P, const TileCtx &T, const uint8_t *c,
                         const uint32_t *bits, int q, int dir, uint32_t tt, int Vk) {
  const int l = lane_of(T, q);
  const int l2 = l + dir;
  if (l2 < 0 || l2 >= T.L) return -1;
  const int q2 = q + dir * T.S;
  if (occupied(bits, q2)) return -1;
  const int code = c[q];
  const int v = code & 7, slot = code >> 3;
  int set = 0;  // 0 all lanes, 1 {0} (right turn), 2 {L-1} (left turn)
  if (slot != kSlotFinal && !(T.d.flags & kPeriodic)) {
    int tty = (tt >> (2 * slot)) & 3;
    set = tty == 0 ? 0 : (tty == 2 ? 1 : 2);
  }
  auto in_set = [&](int ln) { return set == 0 || (set == 1 ? ln == 0 : ln == T.L - 1); };
  if (!in_set(l)) {
    const int toward = (set == 1 && dir < 0) || (set == 2 && dir > 0);
    if (!toward) return -1;
    const int x = T.d.a + (q - l * T.S - T.HP);
    const int d = T.d.n - 1 - x;
    int rf = min(v + 1, Vk), rb = Vk;
    if (d < P.D) {  // R6: desperation over the last D cells
      rf = (rf * d) / P.D;
      rb = (rb * d) / P.D;
    }
    if (ahead_lc(T, bits, q2, l2) >= rf && behind_lc(T, bits, q2, l2) >= rb) return q2;
    return -1;
  }
  if (!in_set(l2)) return -1;
  const int g = ahead_lc(T, bits, q, l);  // R5: the other lane is faster
  if (g < v + 1 && ahead_lc(T, bits, q2, l2) > g && behind_lc(T, bits, q2, l2) >= Vk) return q2;
  return -1;
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

// write the tile state (cout, vout, bout) back: codes, compact vids, strips,
// node records (when the state is S1)
__device__ void write_back(const StepParams &P, TileCtx &T, bool node_recs, int lane) {
  // codes
  if (!T.HP) {
    const int n16 = (T.L * T.w + 15) >> 4;
    uint4 *dst = reinterpret_cast<uint4 *>(P.code_out + T.d.off);
    const uint4 *src = reinterpret_cast<const uint4 *>(T.cout);
    for (int i = lane; i < n16; i += 32) __stcs(dst + i, src[i]);
  } else {
    for (int l = 0; l < T.L; l++)
      for (int x = lane; x < T.w; x += 32)
        P.code_out[T.d.off + (int64_t)l * T.w + x] = T.cout[l * T.S + T.HP + x];
  }
  // vids, coalesced by rank
  const int n = enumerate(T, T.bout, T.vpos, lane);
  for (int r = lane; r < n; r += 32) __stcs(P.vid_out + T.d.off + r, T.vout[T.vpos[r]]);
  // strips for the neighbours' halos
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
        uint32_t occ = 0;  // bit i = cell n-1-i
        for (int i = 0; i < kGmax; i++) occ |= (uint32_t)occupied(T.bout, pt0 + kGmax - 1 - i) << i;
        uint64_t rec = (uint64_t)occ << 44;
        if (occ) {
          int i = __ffs(occ) - 1;
          int pf = pt0 + kGmax - 1 - i;
          rec |= (uint64_t)(uint32_t)T.vout[pf] | ((uint64_t)T.cout[pf] << 32) |
                 ((uint64_t)i << 40) | (1ull << 43);
        }
        P.tail_rec[T.d.lane_gid + l] = rec;
      }
      if (T.d.flags & kFirst) {
        const int ph0 = l * T.S + T.HP;
        uint32_t occ = 0;
        for (int j = 0; j < kGmax; j++) occ |= (uint32_t)occupied(T.bout, ph0 + j) << j;
        P.head_occ[T.d.lane_gid + l] = (uint8_t)occ;
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void place(TileCtx &T, int pos, uint8_t code, int vid) {
  T.cout[pos] = code;
  T.vout[pos] = vid;
}

__device__ __forceinline__ void acc_place(Acc &a, bool hash, int vid, int link, int l, int x,
                                          int v) {
  a.active++;
  a.sumv += v;
  if (hash) a.hash += vmix(vid, link, l, x, v);
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
  const uint32_t m = win_ahead(T.bin, q) & ((1u << lim) - 1u);
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
    // cout = cin, vout from the compact list
    {
      const uint4 *s16 = reinterpret_cast<const uint4 *>(T.cin);
      uint4 *d16 = reinterpret_cast<uint4 *>(T.cout);
      for (int i = lane; i < T.nwords * 2; i += 32) d16[i] = s16[i];
    }
    const int n = enumerate(T, T.bin, T.vpos, lane);
    for (int r = lane; r < n; r += 32) T.vout[T.vpos[r]] = __ldcs(P.vid_in + T.d.off + r);
    __syncwarp();
    // decisions on S(t) (cin / bin), applied to cout
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
      for (int r = lane; r < n; r += 32)
        move_one(P, T, acc, T.vpos[r], __ldcs(P.vid_in + T.d.off + r), false, Vk);
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
        int vid = P.vid_in[T.d.off + r];
        int l = lane_of(T, q);
        place(T, q, T.cin[q], vid);
        acc_place(acc, hash, vid, T.d.link, l, T.d.a + q - l * T.S - T.HP, T.cin[q] & 7);
      }
    }
    __syncwarp();
    // injection from parking (R13): lane 0 walks the
    // link's pending list in (departure, vid) order
    if ((P.mode & kModeInject) && lane == 0) {
      const int k = T.d.link;
      const int e = P.pend_off[k + 1];
      int h = P.pend_head[k];
      const int tn = P.t + 1;
      for (int i = h; i < e; i++) {
        const int vid = P.pend_list[i];
        if (P.dep[vid] > tn) break;
        if (P.inj_time[vid] <= P.t) continue;
        const int ec = P.entry[vid];
        if (ec < T.d.a || ec >= T.d.a + T.w) continue;
        const int q = T.HP + (ec - T.d.a);
        if (T.cout[q] != kEmpty) continue;  // retry next step
        const int64_t ro = P.route_off[vid];
        const int slot0 = (P.route_off[vid + 1] - ro > 1) ? P.out_pos[P.route[ro + 1]] : kSlotFinal;
        place(T, q, (uint8_t)(slot0 << 3), vid);
        P.inj_time[vid] = tn;
        acc.inj++;
        acc_place(acc, hash, vid, k, 0, ec, 0);
      }
      if (T.d.a == 0) {
        while (h < e && P.inj_time[P.pend_list[h]] <= tn) h++;
        P.pend_head[k] = h;
      }
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
  if (P.mode & kModeLC) {
    __syncthreads();
    flush_acc(P, acc_next, P.t + 2, red);
  }
}

// ------------------------------------------------------------- k_node
// O1 §Node (R8-R10): one thread per node.  Candidates are
// the front vehicles of the incoming lanes that want to pass the stop line
// (d < min(v+1, V)); majors first, minors only if the last G cells of every
// major lane are empty; one winner per target lane in (class, link, lane)
// order; the winner is granted the entry space E and, if its velocity takes
// it past the stop line, is written as the entrant of the target lane.
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
      if (P.link_cls[j] != maxcls) {
        for (int l = 0; l < P.link_lanes[j]; l++) P.ext[lg + l] = 0;
        continue;
      }
      for (int l = 0; l < P.link_lanes[j]; l++) {
        P.ext[lg + l] = 0;
        if ((uint32_t)(P.tail_rec[lg + l] >> 44) & gmask) majorfree = false;
      }
    }
    uint32_t claimed[4] = {0u, 0u, 0u, 0u};  // (slot, lane) targets taken
    const int ob = P.out_off[node];
    for (int pass = 0; pass < 2; pass++) {
      if (pass == 1 && !majorfree) break;
      for (int i = a; i < b; i++) {
        const int j = P.in_list[i];
        if ((P.link_cls[j] == maxcls) != (pass == 0)) continue;
        const int lg = P.link_lgid[j];
        const int Vj = P.vmax_link[j];
        const uint32_t tt = P.tt_link[j];
        for (int l = 0; l < P.link_lanes[j]; l++) {
          const uint64_t rec = P.tail_rec[lg + l];
          if (!((rec >> 43) & 1)) continue;
          const int code = (int)((rec >> 32) & 0xFF);
          const int d = (int)((rec >> 40) & 7);
          const int v = code & 7, slot = code >> 3;
          if (slot == kSlotFinal || !(d < min(v + 1, Vj))) continue;
          const int k2 = P.out_list[ob + slot];
          const int tty = (tt >> (2 * slot)) & 3;
          const int L2 = P.link_lanes[k2];
          const int l2 = tty == 0 ? min(l, L2 - 1) : (tty == 2 ? 0 : L2 - 1);  // R8
          const int bit = slot * 8 + l2;
          if (claimed[bit >> 5] & (1u << (bit & 31))) continue;
          claimed[bit >> 5] |= 1u << (bit & 31);
          const int lg2 = P.link_lgid[k2];
          const int E = min(ctz32((uint32_t)P.head_occ[lg2 + l2] | 0x20u), min(kGmax, P.link_ncell[k2]));
          P.ext[lg + l] = (uint8_t)E;
          if (E == 0) continue;
          const int vid = (int)(uint32_t)rec;
          const int v3 = nasch_v3(v, Vj, min(kGmax, d + E), (uint32_t)P.t, (uint32_t)vid, P.k0,
                                  P.k1, P.p32);
          if (v3 <= d) continue;  // stays on its link this step
          const int y2 = v3 - d - 1;
          const int r = P.cursor[vid];
          P.cursor[vid] = r + 1;
          const int64_t ro = P.route_off[vid];
          const int m = (int)(P.route_off[vid + 1] - ro);
          const int nslot = (r + 2 < m) ? P.out_pos[P.route[ro + r + 2]] : kSlotFinal;
          const uint64_t ent = (uint64_t)(uint32_t)vid | ((uint64_t)(v3 | (nslot << 3)) << 32) |
                               ((uint64_t)y2 << 40) | ((uint64_t)((P.t + 1) & 0x1FFFFF) << 43);
          P.entr[lg2 + l2] = ent;
          crossings++;
        }
      }
    }
  }
  // block reduction of the crossing count
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
      h += vmix(P.vid_in[T.d.off + r], T.d.link, l, T.d.a + q - l * T.S - T.HP, T.cin[q] & 7);
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

// ------------------------------------------------------------ launchers
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

int occupancy_blocks(int threads, int smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_step, threads, smem);
  return nb;
}

}  // namespace tsim
