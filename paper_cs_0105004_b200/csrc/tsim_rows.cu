// tsim_rows.cu -- bit-sliced fast path of the TRANSIMS CA step on sm_100a.
//
// k_rows: one warp per group of consecutive whole-link tiles (<= 32
// lane-rows).  The state of a tile is six bit-planes over its lane-cells
// (occupancy O, velocity bits V0..V2, allowed-lane class A0/A1) plus, per
// lane-row, the list of its vehicles in cell order (entries vid | out-slot
// << 27).  One lane handles one 32-cell word at a time, so the rules become
// boolean algebra on 32 cells at once.
//
// Velocity update and move (readings R2, R3, R12, R15):
//   F_k  = cells x+1..x+k empty and inside the row          (gap >= k)
//   T_k  = min(v+1, V) >= k                                 (acceleration)
//   U_k  = T_k & F_k                      (v2 >= k; thermometer code)
//   B    = Philox slowdown draw of every vehicle with v2 >= 1  (R3)
//   W_k  = (U_k & ~B) | (U_{k+1} & B)                      (v3 >= k)
//   D_k  = W_k & ~W_{k+1}                 (vehicles that move exactly k)
//   O'   = OR_k D_k << k, velocity and class bits carried the same way.
// Lane change of the next step (R4-R7), on S(t+1):
//   G_k / TG_k = own / target-lane gap >= k, BK_k = target back gap >= k,
//   E_k = v+1 >= k; the speed rule (R5) and the turn rule (R6, outside the
//   last D cells) are AND/OR of those masks; inside the last D cells the
//   turn rule's scaled thresholds are evaluated per candidate.  The moves
//   are a shift of the LV plane by one row (+-w bits).
// Per-vehicle work: the Philox draws (enumerated across the warp, 32 per
// warp step), row fronts at the stop line (node grant H3, exit R12),
// entrants and injection (H6), and the vid lists of rows whose vehicle set
// changed other than at the ends (lane changes, injection): those are
// rebuilt by rank arithmetic, in-lane order being preserved by every move.
#include "tsim_device.cuh"

namespace tsim {

// bits [0, n) for any n
static __device__ __forceinline__ uint32_t lowm(int n) {
  return n <= 0 ? 0u : (n >= 32 ? FULL : ((1u << n) - 1u));
}

// rank of group-flat bit position q in a plane with per-word prefixes wp
static __device__ __forceinline__ int flat_rank(const uint32_t *bits, const uint16_t *wp, int q) {
  return wp[q >> 5] + __popc(bits[(q >> 5) + 1] & low_mask(q & 31));
}
// same for (b1 & ~b2)
static __device__ __forceinline__ int flat_rank2(const uint32_t *b1, const uint32_t *b2,
                                                 const uint16_t *wp, int q) {
  const int j = (q >> 5) + 1;
  return wp[q >> 5] + __popc(b1[j] & ~b2[j] & low_mask(q & 31));
}

// position of the set bit of rank k (0-based) in m: five popcount halvings
static __device__ __forceinline__ int select_in_word(uint32_t m, int k) {
  int pos = 0, c = __popc(m & 0xFFFFu);
  if (k >= c) { k -= c; pos = 16; m >>= 16; }
  c = __popc(m & 0xFFu);
  if (k >= c) { k -= c; pos += 8; m >>= 8; }
  c = __popc(m & 0xFu);
  if (k >= c) { k -= c; pos += 4; m >>= 4; }
  c = __popc(m & 0x3u);
  if (k >= c) { k -= c; pos += 2; m >>= 2; }
  return pos + (k >= (int)(m & 1u) ? 1 : 0);
}

// Calls f(q) for every set bit q of the group plane `bits` (words 0..nw-1),
// 32 bits per warp step, load-balanced across the words: per chunk of 32
// words (one per lane) an exclusive scan of the counts; per step, the lanes
// whose bit range meets the 32-slot window post themselves in own[] at
// their first slot, and slot i belongs to the last poster at or before i.
template <class F>
static __device__ __forceinline__ void for_each_bit(const uint32_t *bits, int nw, int lane,
                                                    uint8_t *own, F &&f) {
  for (int j0 = 0; j0 < nw; j0 += 32) {
    const uint32_t m = j0 + lane < nw ? bits[j0 + lane + 1] : 0u;
    const int c = __popc(m);
    int s = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    const int T = __shfl_sync(FULL, s, 31);
    s -= c;
    for (int b = 0; b < T; b += 32) {
      const bool part = c > 0 && s < b + 32 && s + c > b;
      const int pos = max(s - b, 0);
      if (part) own[pos] = (uint8_t)lane;
      const uint32_t posted = __reduce_or_sync(FULL, part ? (1u << pos) : 0u);
      __syncwarp();
      const int src = own[31 - __clz(posted & lowm(lane + 1))];
      const uint32_t sm = __shfl_sync(FULL, m, src);
      const int ss = __shfl_sync(FULL, s, src);
      __syncwarp();
      if (b + lane < T) f(32 * (j0 + src) + select_in_word(sm, b + lane - ss));
    }
  }
}

// warp scan over the words of (b1 & ~b2) (b2 may be null): wp[j] = bits
// before word j, wp[nw] = total.  Returns the total.
static __device__ __forceinline__ int scan_words(const uint32_t *b1, const uint32_t *b2, int nw,
                                                 uint16_t *wp, int lane) {
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
    if (j < nw) wp[j] = (uint16_t)(total + sc - c);
    total += __shfl_sync(FULL, sc, 31);
  }
  if (lane == 0) wp[nw] = (uint16_t)total;
  __syncwarp();
  return total;
}

static __device__ __forceinline__ bool row_any(const uint32_t *bits, int s, int w) {
  uint32_t a = 0u;
  for (int x0 = 0; x0 < w; x0 += 32) a |= win_at(bits, s + x0) & low_mask(w - x0);
  return a != 0u;
}

static __device__ __forceinline__ int get3(const uint32_t *v0, const uint32_t *v1,
                                           const uint32_t *v2, int q) {
  return occupied(v0, q) | (occupied(v1, q) << 1) | (occupied(v2, q) << 2);
}

// list entry of an entrant / injected vehicle of row `row` at cell x
static __device__ __forceinline__ uint32_t special_entry(const int32_t *ent, const int32_t *injx,
                                                         const int32_t *injv, int ninj, int row,
                                                         int x) {
  if (ent[32 + row] == x) return (uint32_t)ent[row];
  const int key = (row << 16) | x;
  for (int k = 0; k < ninj; k++)
    if (injx[k] == key) return (uint32_t)injv[k];
  return 0xFFFFFFFFu;
}

struct RowsSmem {
  uint32_t *pl;  // planes, stride PS; plane p = pl + p*PS (pad word first)
  int PS;
  uint16_t *wp_in, *wp_mid, *wp_fin, *wdesc;
  uint8_t *wrow, *own;
  int32_t *t_wbase, *t_w, *t_lv, *t_lg, *t_link, *t_vrel, *t_row0, *t_pw;
  int32_t *r_tile, *r_l, *r_gs, *r_w, *r_lg, *r_vrel, *r_r0, *r_m0, *r_f0, *r_nin, *r_nfin,
      *r_front;
  int32_t *ent, *injx, *injv, *misc;
  __device__ __forceinline__ uint32_t *P(int p) const { return pl + p * PS; }
  // row holding group-flat bit q: the row of the word's first bit plus the
  // row starts inside the word up to q
  __device__ __forceinline__ int row_of(int q) const {
    const int j = q >> 5;
    return wrow[j] + __popc(P(PL_RS)[j + 1] & lowm((q & 31) + 1) & ~1u);
  }
};

// D_k (vehicles of word j moving exactly k cells, k = 0..5) and the
// vehicles that leave their row (row fronts passing the stop line)
static __device__ __forceinline__ void move_masks(const RowsSmem &S, int j, uint32_t D[6],
                                                  uint32_t &lr) {
  const int q = j + 1;
  const uint32_t O = S.P(PL_O)[q], B = S.P(PL_B)[q];
  uint32_t U[6];
  U[0] = S.P(PL_U1)[q];
  U[1] = S.P(PL_U2)[q];
  U[2] = S.P(PL_U3)[q];
  U[3] = S.P(PL_U4)[q];
  U[4] = S.P(PL_U5)[q];
  U[5] = 0u;
  uint32_t W[6];
#pragma unroll
  for (int k = 0; k < 5; k++) W[k] = (U[k] & ~B) | (U[k + 1] & B);  // v3 >= k+1
  W[5] = 0u;
  D[0] = O & ~W[0];
#pragma unroll
  for (int k = 1; k < 6; k++) D[k] = W[k - 1] & ~W[k];
  // a move of k cells that passes a row end leaves the row
  const uint32_t RE = S.P(PL_RE)[q], REn = S.P(PL_RE)[q + 1];
  uint32_t cr = 0u;
  lr = 0u;
#pragma unroll
  for (int k = 1; k < 6; k++) {
    cr |= __funnelshift_r(RE, REn, k - 1);
    lr |= D[k] & cr;
    D[k] &= ~cr;
  }
}

// cells of tile word jj (tile rows of w cells, L lanes) whose lane l has
// l + dir in [0, L)
static __device__ __forceinline__ uint32_t lane_ok_mask(int jj, int w, int L, int dir) {
  const int p0 = 32 * jj;
  return dir > 0 ? lowm((L - 1) * w - p0) : (lowm(L * w - p0) & ~lowm(w - p0));
}

__global__ void __launch_bounds__(128) k_rows(const StepParams P, const RowsParams R) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ unsigned long long red[4 * 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps_total = gridDim.x * (blockDim.x >> 5);
  const RowsLayout &Y = R.lay;
  uint8_t *base = smem + warp * Y.bytes;
  RowsSmem S;
  S.pl = reinterpret_cast<uint32_t *>(base + Y.o_planes);
  S.PS = Y.PS;
  S.wp_in = reinterpret_cast<uint16_t *>(base + Y.o_wp);
  S.wp_mid = S.wp_in + (Y.NG + 4);
  S.wp_fin = S.wp_in + 2 * (Y.NG + 4);
  S.wdesc = reinterpret_cast<uint16_t *>(base + Y.o_wdesc);
  S.wrow = base + Y.o_wrow;
  S.own = base + Y.o_own;
  int32_t *tt = reinterpret_cast<int32_t *>(base + Y.o_tiles);
  S.t_wbase = tt;
  S.t_w = tt + 32;
  S.t_lv = tt + 64;  // L | Vk << 4 | nwt << 8
  S.t_lg = tt + 96;
  S.t_link = tt + 128;
  S.t_vrel = tt + 160;
  S.t_row0 = tt + 192;
  S.t_pw = tt + 224;
  int32_t *rt = reinterpret_cast<int32_t *>(base + Y.o_rows);
  S.r_tile = rt;
  S.r_l = rt + 32;
  S.r_gs = rt + 64;  // group-flat bit of the row start
  S.r_w = rt + 96;
  S.r_lg = rt + 128;
  S.r_vrel = rt + 160;  // vid list of the row, relative to the group's first tile
  S.r_r0 = rt + 192;
  S.r_m0 = rt + 224;
  S.r_f0 = rt + 256;
  S.r_nin = rt + 288;
  S.r_nfin = rt + 320;
  S.r_front = rt + 352;
  S.ent = reinterpret_cast<int32_t *>(base + Y.o_ent);
  S.injx = reinterpret_cast<int32_t *>(base + Y.o_injx);
  S.injv = reinterpret_cast<int32_t *>(base + Y.o_injv);
  S.misc = reinterpret_cast<int32_t *>(base + Y.o_misc);
  const bool do_move = (P.mode & kModeMove) != 0;
  const bool hash = (P.mode & kModeHash) != 0;
  const bool lc = (P.mode & kModeLC) != 0;
  const int lct = do_move ? P.t + 1 : P.t;  // time of the lane-change sub-step
  const int dir = (lct & 1) ? -1 : +1;      // R4
  Acc acc = {};
  Acc acc_next = {};
  if (lane < PL_NUM) S.P(lane)[0] = 0u;  // front pad words, never written

  for (int g = blockIdx.x * (blockDim.x >> 5) + warp; g < R.ngroups; g += nwarps_total) {
    const GroupDesc G = R.groups[g];
    const int64_t off0 = P.tiles[G.t0].off;
    const int nw = G.nwg;
    // ---- tile table (lane = tile)
    {
      int nwt = 0, L = 0;
      if (lane < G.ntiles) {
        const TileDesc d = P.tiles[G.t0 + lane];
        nwt = tile_words(d.w, d.L);
        L = d.L;
        S.t_w[lane] = d.w;
        S.t_lv[lane] = d.L | (P.vmax_link[d.link] << 4) | (nwt << 8);
        S.t_lg[lane] = d.lane_gid;
        S.t_link[lane] = d.link;
        S.t_vrel[lane] = (int)(d.off - off0);
        S.t_pw[lane] = R.pw[G.t0 + lane];
      }
      int sw = nwt, sl = L;  // inclusive scans of words and rows
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(FULL, sw, o), b = __shfl_up_sync(FULL, sl, o);
        if (lane >= o) {
          sw += a;
          sl += b;
        }
      }
      if (lane < G.ntiles) {
        S.t_wbase[lane] = sw - nwt;
        S.t_row0[lane] = sl - L;
      }
    }
    __syncwarp();
    // ---- stage the input planes (word -> tile by binary search), zero the
    //      planes that are built bit by bit and the back pad words
    for (int j = lane; j < nw + 3; j += 32) {
      const int q = j + 1;
      if (j < nw) {
        int lo = 0, hi = G.ntiles - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (S.t_wbase[mid] <= j) lo = mid;
          else hi = mid - 1;
        }
        const int jj = j - S.t_wbase[lo];
        S.wdesc[j] = (uint16_t)((lo << 8) | jj);
        const int nwt = S.t_lv[lo] >> 8;
        const uint32_t *src = R.planes_in + S.t_pw[lo] + jj;
        uint32_t in[kStatePlanes];
#pragma unroll
        for (int p = 0; p < kStatePlanes; p++) in[p] = __ldcs(src + p * nwt);
#pragma unroll
        for (int p = 0; p < kStatePlanes; p++) S.P(p)[q] = in[p];
        S.P(PL_B)[q] = 0u;
        S.P(PL_RE)[q] = 0u;
        S.P(PL_RS)[q] = 0u;
        S.P(PL_ZN)[q] = 0u;
      } else {
#pragma unroll
        for (int p = 0; p < PL_NUM; p++) S.P(p)[q] = 0u;
      }
    }
    if (lane == 0) S.misc[0] = 0;
    S.ent[32 + lane] = -1;
    __syncwarp();
    // ---- row table (lane = row) and the static row planes
    const bool active = lane < G.nrows;
    int tl = 0, l = 0, gs = 0, w = 0, Wp = 4, Vk = 1, L = 1;
    if (active) {
      const int rm = R.rowmap[(size_t)g * 32 + lane];
      tl = rm >> 3;
      l = rm & 7;
      w = S.t_w[tl];
      Wp = row_pitch(w);
      L = S.t_lv[tl] & 15;
      Vk = (S.t_lv[tl] >> 4) & 15;
      gs = 32 * S.t_wbase[tl] + l * w;
      S.r_tile[lane] = tl;
      S.r_l[lane] = l;
      S.r_gs[lane] = gs;
      S.r_w[lane] = w;
      S.r_lg[lane] = S.t_lg[tl] + l;
      S.r_vrel[lane] = S.t_vrel[tl] + l * Wp;
      set_bit(S.P(PL_RE), gs + w - 1);
      set_bit(S.P(PL_RS), gs);
      for (int a = gs + max(w - P.D, 0), b = gs + w; a < b;) {  // desperation zone (R6)
        const int wi = a >> 5, hi = min(b, 32 * wi + 32);
        atomicOr(S.P(PL_ZN) + wi + 1, lowm(hi - 32 * wi) & ~lowm(a - 32 * wi));
        a = hi;
      }
      for (int j = (gs + 31) >> 5; 32 * j < gs + w; j++) S.wrow[j] = (uint8_t)lane;
    }
    const int lg = active ? S.t_lg[tl] + l : 0;
    const int link = active ? S.t_link[tl] : 0;
    const int32_t *vin_row = P.vid_in + off0 + (active ? S.t_vrel[tl] + l * Wp : 0);
    const int nb = min(w, kGmax);  // cells of the stop-line window
    __syncwarp();
    scan_words(S.P(PL_O), nullptr, nw, S.wp_in, lane);
    int nin = 0;
    if (active) {
      const int r0 = flat_rank(S.P(PL_O), S.wp_in, gs);
      nin = flat_rank(S.P(PL_O), S.wp_in, gs + w) - r0;
      S.r_r0[lane] = r0;
      S.r_nin[lane] = nin;
      if ((P.mode & kModeWork) && P.link_work && nin)
        atomicAdd(P.link_work + link, (unsigned long long)nin);
      acc.work += nin;
    }
    __syncwarp();
    if (do_move) {
      // ---- 1a. thermometer codes, one 32-cell word per lane
      for (int j = lane; j < nw; j += 32) {
        const int q = j + 1;
        const uint32_t O = S.P(PL_O)[q], On = S.P(PL_O)[q + 1];
        const uint32_t RE = S.P(PL_RE)[q], REn = S.P(PL_RE)[q + 1];
        const uint32_t V0 = S.P(PL_V0)[q], V1 = S.P(PL_V1)[q], V2 = S.P(PL_V2)[q];
        const int vk = (S.t_lv[S.wdesc[j] >> 8] >> 4) & 15;
        // gap >= k: cells x+1..x+k empty, none past the row end
        uint32_t F = ~__funnelshift_r(O, On, 1) & ~RE;
        uint32_t T = O;  // min(v+1, V) >= 1
        S.P(PL_U1)[q] = T & F;
        F &= ~__funnelshift_r(O, On, 2) & ~__funnelshift_r(RE, REn, 1);
        T = vk >= 2 ? (O & (V0 | V1 | V2)) : 0u;  // v >= 1
        S.P(PL_U2)[q] = T & F;
        F &= ~__funnelshift_r(O, On, 3) & ~__funnelshift_r(RE, REn, 2);
        T = vk >= 3 ? (V1 | V2) : 0u;  // v >= 2
        S.P(PL_U3)[q] = T & F;
        F &= ~__funnelshift_r(O, On, 4) & ~__funnelshift_r(RE, REn, 3);
        T = vk >= 4 ? (V2 | (V1 & V0)) : 0u;  // v >= 3
        S.P(PL_U4)[q] = T & F;
        F &= ~__funnelshift_r(O, On, 5) & ~__funnelshift_r(RE, REn, 4);
        T = vk >= 5 ? V2 : 0u;  // v >= 4
        S.P(PL_U5)[q] = T & F;
      }
      __syncwarp();
      // ---- 1b. the row front near the stop line: open end of the final
      //          link (R12) or entry space granted by the node (H3)
      if (active) {
        const uint32_t m = win_at(S.P(PL_O), gs + w - nb) & low_mask(nb);
        if (m) {
          const int xf = w - nb + 31 - __clz(m);
          const int d = w - 1 - xf;
          const uint32_t e = (uint32_t)__ldg(vin_row + nin - 1);
          const int slot = (int)(e >> kSlotShift);
          const int gp = slot == kSlotFinal ? kGmax : min(kGmax, d + (int)P.ext[lg]);
          if (gp > d) {
            const int q = gs + xf;
            const int v = get3(S.P(PL_V0), S.P(PL_V1), S.P(PL_V2), q);
            const int v2 = min(min(v + 1, Vk), gp);
            for (int k = d + 1; k <= v2; k++) set_bit(S.P(PL_U1 + k - 1), q);
          }
        }
      }
      __syncwarp();
      // ---- 1c. Philox slowdown draws (R3), 32 vehicles per warp step
      for_each_bit(S.P(PL_U1), nw, lane, S.own, [&](int q) {
        const int row = S.row_of(q);
        const int rank = flat_rank(S.P(PL_O), S.wp_in, q) - S.r_r0[row];
        const uint32_t e = (uint32_t)P.vid_in[off0 + S.r_vrel[row] + rank];
        if ((uint64_t)philox_w0((uint32_t)P.t, e & kVidMask, P.k0, P.k1) < P.p32)
          set_bit(S.P(PL_B), q);
      });
      __syncwarp();
      // ---- 1d. hop: O' = OR_k D_k << k, velocity and class bits likewise
      for (int j = lane; j < nw; j += 32) {
        uint32_t Dj[6], Dp[6], lrj, lrp;
        move_masks(S, j, Dj, lrj);
        if (j > 0) move_masks(S, j - 1, Dp, lrp);
        else {
#pragma unroll
          for (int k = 0; k < 6; k++) Dp[k] = 0u;
        }
        uint32_t sh[6];
        sh[0] = Dj[0];
#pragma unroll
        for (int k = 1; k < 6; k++) sh[k] = __funnelshift_l(Dp[k], Dj[k], k);
        const int q = j + 1;
        const uint32_t OO = sh[0] | sh[1] | sh[2] | sh[3] | sh[4] | sh[5];
        S.P(PL_OO)[q] = OO;
        S.P(PL_OV0)[q] = sh[1] | sh[3] | sh[5];
        S.P(PL_OV1)[q] = sh[2] | sh[3];
        S.P(PL_OV2)[q] = sh[4] | sh[5];
        const uint32_t A0 = S.P(PL_A0)[q], A1 = S.P(PL_A1)[q];
        const uint32_t A0p = S.P(PL_A0)[q - 1], A1p = S.P(PL_A1)[q - 1];
        uint32_t oa0 = Dj[0] & A0, oa1 = Dj[0] & A1;
#pragma unroll
        for (int k = 1; k < 6; k++) {
          oa0 |= __funnelshift_l(Dp[k] & A0p, Dj[k] & A0, k);
          oa1 |= __funnelshift_l(Dp[k] & A1p, Dj[k] & A1, k);
        }
        S.P(PL_OA0)[q] = oa0;
        S.P(PL_OA1)[q] = oa1;
        S.P(PL_LR)[q] = lrj;
        acc.active += __popc(OO);
        acc.sumv += __popc(sh[1]) + 2 * __popc(sh[2]) + 3 * __popc(sh[3]) + 4 * __popc(sh[4]) +
                    5 * __popc(sh[5]);
      }
    } else {  // no move (initial injection / lane change only)
      for (int j = lane; j < nw; j += 32) {
        const int q = j + 1;
        S.P(PL_OO)[q] = S.P(PL_O)[q];
        S.P(PL_OV0)[q] = S.P(PL_V0)[q];
        S.P(PL_OV1)[q] = S.P(PL_V1)[q];
        S.P(PL_OV2)[q] = S.P(PL_V2)[q];
        S.P(PL_OA0)[q] = S.P(PL_A0)[q];
        S.P(PL_OA1)[q] = S.P(PL_A1)[q];
        if (P.mode & kModeInject) acc.active += __popc(S.P(PL_O)[q]);
      }
    }
    __syncwarp();
    for (int j = lane; j < nw; j += 32) S.P(PL_SP)[j + 1] = 0u;  // U1 storage becomes SP
    __syncwarp();
    // ---- 1e. row events: exits, entrant, injection
    bool has_ent = false, injected = false;
    if (active && do_move) {
      const uint32_t m = win_at(S.P(PL_LR), gs + w - nb) & low_mask(nb);  // the front left
      if (m) {
        const uint32_t e = (uint32_t)__ldg(vin_row + nin - 1);
        if ((int)(e >> kSlotShift) == kSlotFinal) {  // exit to parking
          P.arr_time[e & kVidMask] = P.t + 1;
          acc.arr++;
        }  // else: crossed the node; k_node_warp placed it on the next link
      }
      const uint64_t rec = P.entr[lg];  // entrant granted by the node kernel
      if ((uint32_t)(rec >> 43) == ((uint32_t)(P.t + 1) & 0x1FFFFFu)) {
        const int evid = (int)(uint32_t)rec;
        const int code = (int)((rec >> 32) & 0xFF);
        const int y = (int)((rec >> 40) & 7);
        const int q = gs + y;
        set_bit(S.P(PL_OO), q);
        if (code & 1) set_bit(S.P(PL_OV0), q);
        if (code & 2) set_bit(S.P(PL_OV1), q);
        if (code & 4) set_bit(S.P(PL_OV2), q);
        set_bit(S.P(PL_SP), q);
        const int cls = lane_class(code >> 3, P.tt_link[link]);
        if (cls & 1) set_bit(S.P(PL_OA0), q);
        if (cls & 2) set_bit(S.P(PL_OA1), q);
        S.ent[lane] = evid | ((code >> 3) << kSlotShift);
        S.ent[32 + lane] = y;
        has_ent = true;
        acc.active++;
        acc.sumv += code & 7;
      }
    }
    if (active && (P.mode & kModeInject) && l == 0 && P.pend_off[link + 1] > P.pend_head[link]) {
      const int row = lane;
      inject_link(
          P, link, 0, w, true, [&](int x) { return !occupied(S.P(PL_OO), gs + x); },
          [&](int x, uint8_t code, int ivid) {
            const int q = gs + x;
            set_bit(S.P(PL_OO), q);
            set_bit(S.P(PL_SP), q);
            const int cls = lane_class(code >> 3, P.tt_link[link]);
            if (cls & 1) set_bit(S.P(PL_OA0), q);
            if (cls & 2) set_bit(S.P(PL_OA1), q);
            const int k = atomicAdd(S.misc, 1);
            S.injx[k] = (row << 16) | x;
            S.injv[k] = ivid | ((code >> 3) << kSlotShift);
            injected = true;
            acc.inj++;
            acc.active++;
          });
    }
    __syncwarp();
    // rank of input-derived vehicles (for vid lookups of S(t+1))
    scan_words(S.P(PL_OO), S.P(PL_SP), nw, S.wp_mid, lane);
    if (active) S.r_m0[lane] = flat_rank2(S.P(PL_OO), S.P(PL_SP), S.wp_mid, gs);
    __syncwarp();
    // entry (vid | slot) of the vehicle of S(t+1) at group-flat position q
    auto entry_at = [&](int row, int q) -> uint32_t {
      const int x = q - S.r_gs[row];
      if (occupied(S.P(PL_SP), q)) return special_entry(S.ent, S.injx, S.injv, S.misc[0], row, x);
      return (uint32_t)P.vid_in[off0 + S.r_vrel[row] + flat_rank2(S.P(PL_OO), S.P(PL_SP),
                                                                   S.wp_mid, q) - S.r_m0[row]];
    };
    if (hash) {  // state hash of S(t+1) (tests)
      for_each_bit(S.P(PL_OO), nw, lane, S.own, [&](int q) {
        const int row = S.row_of(q);
        const uint32_t e = entry_at(row, q);
        acc.hash += vmix((int)(e & kVidMask), S.t_link[S.r_tile[row]], S.r_l[row], q - S.r_gs[row],
                         get3(S.P(PL_OV0), S.P(PL_OV1), S.P(PL_OV2), q));
      });
      __syncwarp();
    }
    const uint32_t *OO = S.P(PL_OO);
    // ---- 2. lane change on S(t+1) (fused) or S(t) (lane change only):
    //         LV = vehicles that move to lane l + dir
    if (lc) {
      for (int j = lane; j < nw; j += 32) {
        const int q = j + 1;
        const uint32_t O = OO[q];
        uint32_t lv = 0u;
        const int wd = S.wdesc[j], t = wd >> 8, jj = wd & 255;
        const int tw = S.t_w[t], tlv = S.t_lv[t], tL = tlv & 15, vk = (tlv >> 4) & 15;
        uint32_t cand = O & lane_ok_mask(jj, tw, tL, dir);
        const int tb = 32 * j + dir * tw;  // target cell of bit 0
        const int lo_s = -32, hi_s = 32 * (nw + 1);
        uint32_t T0 = 0u;
        if (cand) {
          T0 = win_at(OO, min(max(tb, lo_s), hi_s));
          cand &= ~T0;
        }
        if (cand) {
          const uint32_t Tn = win_at(OO, min(max(tb + 32, lo_s), hi_s));
          const uint32_t Tp = win_at(OO, min(max(tb - 32, lo_s), hi_s));
          const uint32_t On = OO[q + 1];
          const uint32_t RE = S.P(PL_RE)[q], REn = S.P(PL_RE)[q + 1];
          const uint32_t RSc = S.P(PL_RS)[q], RSp = S.P(PL_RS)[q - 1];
          // gaps ahead in the own and target lanes (stop at the row end, R2)
          uint32_t G[6], TG[6];
          G[0] = FULL;
          TG[0] = FULL;
#pragma unroll
          for (int k = 1; k <= 5; k++) {
            const uint32_t e = __funnelshift_r(RE, REn, k - 1);
            G[k] = G[k - 1] & ~(__funnelshift_r(O, On, k) | e);
            TG[k] = TG[k - 1] & ~(__funnelshift_r(T0, Tn, k) | e);
          }
          // gap behind in the target lane (before the row start = empty)
          uint32_t before = RSc, BK = FULL, BKv = FULL;
#pragma unroll
          for (int k = 1; k <= 5; k++) {
            BK &= ~__funnelshift_l(Tp, T0, k) | before;
            if (k == vk) BKv = BK;
            before |= __funnelshift_l(RSp, RSc, k);
          }
          const uint32_t V0 = S.P(PL_OV0)[q], V1 = S.P(PL_OV1)[q], V2 = S.P(PL_OV2)[q];
          const uint32_t A0 = S.P(PL_OA0)[q], A1 = S.P(PL_OA1)[q];
          // E_k = (v + 1 >= k)
          const uint32_t E2 = V0 | V1 | V2, E3 = V1 | V2, E4 = V2 | (V1 & V0), E5 = V2,
                         E6 = V2 & V0;
          // speed-motivated (R5): own gap < v+1, target gap ahead > own gap,
          // target gap behind >= V; only for vehicles free to use any lane
          const uint32_t geq = G[1] & (~E2 | G[2]) & (~E3 | G[3]) & (~E4 | G[4]) &
                               (~E5 | G[5]) & ~E6;
          const uint32_t tgt = TG[1] & (~G[1] | TG[2]) & (~G[2] | TG[3]) & (~G[3] | TG[4]) &
                               (~G[4] | TG[5]) & ~G[5];
          lv = cand & ~A0 & ~A1 & ~geq & tgt & BKv;
          // turn-motivated (R6, R7): towards the allowed lane
          const uint32_t turn = cand & (dir < 0 ? (A0 & ~A1) : (A1 & ~A0));
          if (turn) {
            const uint32_t ZN = S.P(PL_ZN)[q];
            // ahead >= min(v+1, V), behind >= V outside the last D cells
            uint32_t req = TG[1];
            if (vk >= 2) req &= ~E2 | TG[2];
            if (vk >= 3) req &= ~E3 | TG[3];
            if (vk >= 4) req &= ~E4 | TG[4];
            if (vk >= 5) req &= ~E5 | TG[5];
            lv |= turn & ~ZN & req & BKv;
            uint32_t zc = turn & ZN;  // scaled thresholds: per candidate
            while (zc) {
              const int x = __ffs(zc) - 1;
              zc &= zc - 1u;
              const int qq = 32 * j + x;
              const int row = S.row_of(qq);
              const int rgs = S.r_gs[row], rl = S.r_l[row];
              const int v = (int)((V0 >> x) & 1u) | (int)(((V1 >> x) & 1u) << 1) |
                            (int)(((V2 >> x) & 1u) << 2);
              const int set = (int)((A0 >> x) & 1u) | (int)(((A1 >> x) & 1u) << 1);
              const int gs2 = rgs + dir * tw;
              if (lc_rule_set(OO, qq, qq + dir * tw, rgs, rgs + tw, gs2, gs2 + tw, v, set, rl,
                              rl + dir, tL, dir, rgs + tw - 1 - qq, vk, P.D))
                lv |= 1u << x;
            }
          }
        }
        S.P(PL_LV)[q] = lv;
        acc_next.lc += __popc(lv);
      }
      __syncwarp();
    }
    // ---- 3. apply the lane changes; final planes to smem and HBM
    for (int j = lane; j < nw; j += 32) {
      const int q = j + 1;
      const int wd = S.wdesc[j], t = wd >> 8, jj = wd & 255;
      const int nwt = S.t_lv[t] >> 8;
      uint32_t f = OO[q], fv0 = S.P(PL_OV0)[q], fv1 = S.P(PL_OV1)[q], fv2 = S.P(PL_OV2)[q],
               fa0 = S.P(PL_OA0)[q], fa1 = S.P(PL_OA1)[q];
      if (lc) {
        const int tw = S.t_w[t], tL = S.t_lv[t] & 15;
        const uint32_t lv = S.P(PL_LV)[q];
        uint32_t lvs = 0u;  // arrivals from lane l - dir
        const uint32_t sv = lane_ok_mask(jj, tw, tL, -dir);
        const int sb = min(max(32 * j - dir * tw, -32), 32 * (nw + 1));
        if (sv) lvs = win_at(S.P(PL_LV), sb) & sv;
        if (lv | lvs) {
          f = (f & ~lv) | lvs;
          fv0 = (fv0 & ~lv) | (win_at(S.P(PL_OV0), sb) & lvs);
          fv1 = (fv1 & ~lv) | (win_at(S.P(PL_OV1), sb) & lvs);
          fv2 = (fv2 & ~lv) | (win_at(S.P(PL_OV2), sb) & lvs);
          fa0 = (fa0 & ~lv) | (win_at(S.P(PL_OA0), sb) & lvs);
          fa1 = (fa1 & ~lv) | (win_at(S.P(PL_OA1), sb) & lvs);
        }
        S.P(PL_CH)[q] = lv | lvs;
      }
      S.P(PL_FIN)[q] = f;
      S.P(PL_FV0)[q] = fv0;
      S.P(PL_FV1)[q] = fv1;
      S.P(PL_FV2)[q] = fv2;
      S.P(PL_WORK)[q] = 0u;
      uint32_t *dst = R.planes_out + S.t_pw[t] + jj;
      __stcs(dst, f);
      __stcs(dst + nwt, fv0);
      __stcs(dst + 2 * nwt, fv1);
      __stcs(dst + 3 * nwt, fv2);
      __stcs(dst + 4 * nwt, fa0);
      __stcs(dst + 5 * nwt, fa1);
    }
    __syncwarp();
    // ---- 4. vid lists of the final state
    scan_words(S.P(PL_FIN), nullptr, nw, S.wp_fin, lane);
    bool rebuild = false;
    if (active) {
      const int f0 = flat_rank(S.P(PL_FIN), S.wp_fin, gs);
      const int nfin = flat_rank(S.P(PL_FIN), S.wp_fin, gs + w) - f0;
      S.r_f0[lane] = f0;
      S.r_nfin[lane] = nfin;
      const bool ch_lc = lc && row_any(S.P(PL_CH), gs, w);
      const uint4 *src = reinterpret_cast<const uint4 *>(vin_row);
      uint4 *dst = reinterpret_cast<uint4 *>(P.vid_out + off0 + S.r_vrel[lane]);
      if (!ch_lc && !injected && !has_ent) {
        // input vehicles minus an exit at the front: a prefix of the input list
        uint4 bufv = make_uint4(0, 0, 0, 0);
        for (int i = 0; i < nfin; i += 4) {
          bufv = __ldg(src + (i >> 2));
          __stcs(dst + (i >> 2), bufv);
        }
        const int k = (nfin - 1) & 3;
        S.r_front[lane] = (int)(k == 0 ? bufv.x : k == 1 ? bufv.y : k == 2 ? bufv.z : bufv.w);
      } else if (!ch_lc && !injected) {
        // the entrant lands behind every vehicle of the row: the list shifts by one
        uint32_t prev = (uint32_t)S.ent[lane];
        uint4 o = make_uint4(prev, 0, 0, 0);
        for (int i = 0; i < nfin; i += 4) {
          const uint4 a = __ldg(src + (i >> 2));
          o = make_uint4(prev, a.x, a.y, a.z);
          prev = a.w;
          __stcs(dst + (i >> 2), o);
        }
        const int k = (nfin - 1) & 3;
        S.r_front[lane] = (int)(k == 0 ? o.x : k == 1 ? o.y : k == 2 ? o.z : o.w);
      } else {
        rebuild = true;
        for (int a = gs, b = gs + w; a < b;) {  // mark the row's cells
          const int wi = a >> 5, hi = min(b, 32 * wi + 32);
          atomicOr(S.P(PL_WORK) + wi + 1, lowm(hi - 32 * wi) & ~lowm(a - 32 * wi));
          a = hi;
        }
      }
    }
    if (__ballot_sync(FULL, rebuild)) {
      __syncwarp();
      for (int j = lane; j < nw; j += 32) S.P(PL_WORK)[j + 1] &= S.P(PL_FIN)[j + 1];
      __syncwarp();
      for_each_bit(S.P(PL_WORK), nw, lane, S.own, [&](int q) {
        const int row = S.row_of(q);
        const int jo = flat_rank(S.P(PL_FIN), S.wp_fin, q) - S.r_f0[row];  // output slot
        const uint32_t e = occupied(OO, q) ? entry_at(row, q)  // own vehicle
                                           : entry_at(row - dir, q - dir * S.r_w[row]);  // arrived
        P.vid_out[off0 + S.r_vrel[row] + jo] = (int)e;
        if (jo == S.r_nfin[row] - 1) S.r_front[row] = (int)e;  // front vehicle
      });
    }
    __syncwarp();
    if (active && lc) {  // the output is S1: node records for k_node_warp
      const uint32_t fin = (win_at(S.P(PL_FIN), gs + w - nb) & low_mask(nb)) << (kGmax - nb);
      // bit i = cell w-5+i
      uint64_t rec = (uint64_t)(__brev(fin) >> 27) << 44;  // bit i = cell n-1-i
      if (fin) {
        const int xf = w - kGmax + 31 - __clz(fin);
        const uint32_t e = (uint32_t)S.r_front[lane];
        const int code = get3(S.P(PL_FV0), S.P(PL_FV1), S.P(PL_FV2), gs + xf) |
                         ((int)(e >> kSlotShift) << 3);
        rec |= (uint64_t)(e & kVidMask) | ((uint64_t)code << 32) |
               ((uint64_t)(w - 1 - xf) << 40) | (1ull << 43);
      }
      P.tail_rec[lg] = rec;
      P.head_occ[lg] = (uint8_t)(win_at(S.P(PL_FIN), gs) & low_mask(nb));
    }
    __syncwarp();
  }
  flush_acc(P, acc, P.t + 1, red);
  if (lc) flush_acc(P, acc_next, lct + 1, red);
}

// state hash of the row-mode state S(t) (one thread per lane-row)
__global__ void __launch_bounds__(128) k_rows_hash(const StepParams P, const RowsParams R,
                                                   unsigned long long *out) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t h = 0, cnt = 0;
  // rows are enumerated through the tiles: gid = tile * 8 + lane of tile
  const int ti = gid >> 3, l = gid & 7;
  if (ti < P.ntiles) {
    const TileDesc d = P.tiles[ti];
    if (l < d.L) {
      const int nwt = tile_words(d.w, d.L);
      const uint32_t *pl = R.planes_in + R.pw[ti];
      const int32_t *vl = P.vid_in + d.off + (int64_t)l * row_pitch(d.w);
      int k = 0;
      for (int x = 0; x < d.w; x++) {
        const int b = l * d.w + x;
        if (!((pl[b >> 5] >> (b & 31)) & 1u)) continue;
        const int v = (int)((pl[nwt + (b >> 5)] >> (b & 31)) & 1u) |
                      (int)(((pl[2 * nwt + (b >> 5)] >> (b & 31)) & 1u) << 1) |
                      (int)(((pl[3 * nwt + (b >> 5)] >> (b & 31)) & 1u) << 2);
        const uint32_t e = (uint32_t)vl[k++];
        h += vmix((int)(e & kVidMask), d.link, l, d.a + x, v);
        cnt++;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    h += __shfl_down_sync(FULL, h, o);
    cnt += __shfl_down_sync(FULL, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, (unsigned long long)h);
    atomicAdd(out + 1, (unsigned long long)cnt);
  }
}

void launch_rows(const StepParams &p, const RowsParams &r, int blocks, int threads, int smem,
                 void *stream) {
  k_rows<<<blocks, threads, smem, (cudaStream_t)stream>>>(p, r);
}
void launch_rows_hash(const StepParams &p, const RowsParams &r, void *stream,
                      unsigned long long *out) {
  const int n = p.ntiles * 8;
  k_rows_hash<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(p, r, out);
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
