// tsim_rows.cu -- register-resident bit-sliced fast path of the TRANSIMS CA
// step on sm_100a (Nagel & Rickert, §3; readings R1-R22 in
// DESIGN.md §3).
//
// k_rows: one THREAD per lane-row of a whole link of <= kRowMaxCells cells;
// the lanes of a link sit on consecutive threads of one warp, so the
// sideways look of the lane change is a warp shuffle.  A row's state lives
// in registers as six bit-planes of kRowWords words (occupancy O, velocity
// bits V0..V2, allowed-lane class A0/A1), loaded and stored as coalesced
// 128-byte lines (group-interleaved layout, tsim_internal.h); the rules
// become boolean algebra on 32 cells at a time with funnel shifts between
// the words of the row.  No shared memory and no warp barriers on the main
// path.
//
// Velocity update and move (R2, R3, R12, R15):
//   F_k  = cells x+1..x+k empty and inside the row          (gap >= k)
//   T_k  = min(v+1, V) >= k                                 (acceleration)
//   U_k  = T_k & F_k                      (v2 >= k; thermometer code)
//   B    = Philox slowdown draw of every vehicle with v2 >= 1  (R3)
//   W_k  = (U_k & ~B) | (U_{k+1} & B)                      (v3 >= k)
//   D_k  = W_k & ~W_{k+1}                 (vehicles that move exactly k)
//   O'   = OR_k D_k << k, velocity and class bits carried the same way.
// The row front near the stop line takes its gap from the node grant
// (H3, ext) or the open end of its final link (R12).
// Lane change of the next step (R4-R7), on S(t+1):
//   G_k / TG_k = own / target-lane gap >= k, BK_k = target back gap >= k,
//   E_k = v+1 >= k; the speed rule (R5) and the turn rule (R6, outside the
//   last D cells) are AND/OR of those masks; inside the last D cells the
//   turn rule's scaled thresholds are evaluated per candidate.
// Vid lists: every final vehicle is written to its rank in the final
// occupancy of its row (prefix popcount), so no list is written twice and
// rows whose vehicle set only lost its front or gained a back entrant are
// plain (shifted) vector copies.
#include "tsim_device.cuh"
#include "../../include/tsim.h"

// ---- checked build (-DTS_CHECKED; tests and tools only, never the bench):
// invariants of the row kernel's state, counted per device instead of
// asserted, read back by ts_debug_checks (include/tsim.h).  Bits:
//   1  the group's vid-block count differs from its occupancy planes
//   2  an input vehicle in a cell past its row end
//   4  a lane-change arrival onto a cell its own row keeps (a cell
//      written twice: "occupied by exactly one car")
//   8  a final vehicle past its row end, 16 a final velocity above the
//      link's vmax, 32 a group's output block larger
//      than its cells, 64 a vid-list entry scattered to a cell of the
//      final occupancy that is empty (a mis-ranked list), 128 the
//      self-test (every group of every launch while armed)
#ifdef TS_CHECKED
__device__ unsigned int g_ts_chk[4] = {0u, 0xFFFFFFFFu, 0u, 0u};
#define TS_CHK(cond, bit, grp)                          \
  do {                                                  \
    if (!(cond)) {                                      \
      atomicOr(&g_ts_chk[0], (unsigned)(bit));          \
      atomicMin(&g_ts_chk[1], (unsigned)(grp));         \
      atomicAdd(&g_ts_chk[2], 1u);                      \
    }                                                   \
  } while (0)
#else
#define TS_CHK(cond, bit, grp) ((void)0)
#endif

namespace tsim {

namespace {
constexpr int NW = kRowWords;

// bits [0, n) for any n
__device__ __forceinline__ uint32_t lowm(int n) {
  return n <= 0 ? 0u : (n >= 32 ? FULL : ((1u << n) - 1u));
}

// bit x of o = bit x+k of the row x (k in 1..31); cells past the last word
// read as `fill`
__device__ __forceinline__ void shr(uint32_t (&o)[NW], const uint32_t (&x)[NW], int k,
                                    uint32_t fill) {
#pragma unroll
  for (int i = 0; i < NW; i++) o[i] = __funnelshift_r(x[i], i + 1 < NW ? x[i + 1] : fill, k);
}
// bit x of o = bit x-k of the row x (k in 1..31); cells before 0 read as 0
__device__ __forceinline__ void shl(uint32_t (&o)[NW], const uint32_t (&x)[NW], int k) {
#pragma unroll
  for (int i = 0; i < NW; i++) o[i] = __funnelshift_l(i > 0 ? x[i - 1] : 0u, x[i], k);
}

__device__ __forceinline__ int popc_row(const uint32_t (&x)[NW]) {
  int c = 0;
#pragma unroll
  for (int i = 0; i < NW; i++) c += __popc(x[i]);
  return c;
}
__device__ __forceinline__ bool any_row(const uint32_t (&x)[NW]) {
  uint32_t a = 0u;
#pragma unroll
  for (int i = 0; i < NW; i++) a |= x[i];
  return a != 0u;
}
// one-hot mask of cell c inside word i (no dynamic register indexing: the
// compiler would otherwise move the row to local memory)
__device__ __forceinline__ uint32_t onehot(int i, int c) {
  const unsigned d = (unsigned)(c - 32 * i);
  return d < 32u ? (1u << d) : 0u;
}
// word i of the row (arithmetic select: no dynamic register indexing)
__device__ __forceinline__ uint32_t pick(const uint32_t (&x)[NW], int i) {
  uint32_t r = 0u;
#pragma unroll
  for (int k = 0; k < NW; k++) r |= x[k] & (0u - (uint32_t)(k == i));
  return r;
}
// bits [s, s + 32) of the row, s >= 0
__device__ __forceinline__ uint32_t win_row(const uint32_t (&x)[NW], int s) {
  return __funnelshift_r(pick(x, s >> 5), pick(x, (s >> 5) + 1), s & 31);
}
__device__ __forceinline__ int bit_row(const uint32_t (&x)[NW], int c) {
  uint32_t b = 0u;
#pragma unroll
  for (int i = 0; i < NW; i++) b |= x[i] & onehot(i, c);
  return b != 0u;
}
__device__ __forceinline__ void set_row(uint32_t (&x)[NW], int c) {
#pragma unroll
  for (int i = 0; i < NW; i++) x[i] |= onehot(i, c);
}
// highest set cell, -1 if none
__device__ __forceinline__ int top_row(const uint32_t (&x)[NW]) {
  int t = -1;
#pragma unroll
  for (int i = 0; i < NW; i++)
    if (x[i]) t = 32 * i + 31 - __clz(x[i]);
  return t;
}
// cells [a, b) of the row
__device__ __forceinline__ uint32_t range_w(int i, int a, int b) {
  return lowm(b - 32 * i) & ~lowm(a - 32 * i);
}
__device__ __forceinline__ uint32_t shfl_w(uint32_t v, int src) { return __shfl_sync(FULL, v, src); }

// exclusive warp prefix sum; *total = warp sum
__device__ __forceinline__ int warp_scan(int v, int lane, int *total) {
  int s = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(FULL, s, o);
    if (lane >= o) s += y;
  }
  *total = __shfl_sync(FULL, s, 31);
  return s - v;
}
// one-lane bulk (TMA) store of n entries of shared memory to global memory;
// both 16-byte aligned, the byte count rounded up to 16 (the destination
// block has room: group capacities are multiples of 4 entries)
__device__ __forceinline__ void bulk_store(int32_t *gdst, const int32_t *src, int n) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(src);
  const uint32_t bytes = (uint32_t)((n + 3) & ~3) * 4u;
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(sa),
               "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// TMA bulk load of a vid block into shared memory, completion on an
// mbarrier (one per warp): lane 0 arms the barrier with the byte count and
// issues the copy; every lane waits on the barrier's phase
__device__ __forceinline__ void mbar_init(uint64_t *bar) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(int32_t *sdst, const int32_t *gsrc, int n, uint64_t *bar) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sdst);
  const uint32_t ba = (uint32_t)__cvta_generic_to_shared(bar);
  const uint32_t bytes = (uint32_t)((n + 3) & ~3) * 4u;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(ba), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa),
      "l"(gsrc), "r"(bytes), "r"(ba)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t ba = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}" ::"r"(ba),
      "r"(parity)
      : "memory");
}

// bitwise OR into a shared-memory word (no return value)
__device__ __forceinline__ void red_or_shared(uint32_t saddr, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(saddr), "r"(v) : "memory");
}
// the bulk stores of this thread have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
}  // namespace

struct RowWords {
  uint32_t w[kRowWords];
};

// state hash contribution of one row of S(t+1) before its lane change
// (test instrument; kept out of line)
static __device__ __noinline__ uint64_t hash_row(RowWords oo, RowWords v0, RowWords v1,
                                                 RowWords v2, RowWords inj, int ent_y,
                                                 uint32_t ent_e, const int32_t *vin,
                                                 const int32_t *scratch, int link, int l, int a) {
  uint64_t h = 0;
  int k = 0;
  for (int c = 0; c < kRowMaxCells; c++) {
    const int i = c >> 5, x = c & 31;
    if (!((oo.w[i] >> x) & 1u)) continue;
    uint32_t e;
    if (c == ent_y) e = ent_e;
    else if ((inj.w[i] >> x) & 1u) e = (uint32_t)scratch[c];
    else e = (uint32_t)vin[k++];
    const int v = (int)((v0.w[i] >> x) & 1u) | (int)(((v1.w[i] >> x) & 1u) << 1) |
                  (int)(((v2.w[i] >> x) & 1u) << 2);
    h += vmix((int)(e & kVidMask), link, l, a + c, v);
  }
  return h;
}

// Turn-motivated lane change inside the last D cells (R6): the accepted
// gaps shrink with the distance d to the link end, (floor(min(v+1,V) d/D),
// floor(V d/D)); evaluated per candidate (rare, kept out of line).  zc:
// candidates of the word starting at cell c0; tg1..tg5: target-lane gap
// ahead >= k; tp, t0: target-lane occupancy of the previous / this word.
static __device__ __noinline__ uint32_t zone_lc(uint32_t zc, int c0, int w, int vk, uint32_t Dmul,
                                                uint32_t v0, uint32_t v1, uint32_t v2,
                                                uint32_t tg1, uint32_t tg2, uint32_t tg3,
                                                uint32_t tg4, uint32_t tg5, uint32_t tp,
                                                uint32_t t0) {
  uint32_t lv = 0u;
  while (zc) {
    const int x = __ffs(zc) - 1;
    zc &= zc - 1u;
    const int d = w - 1 - (c0 + x);
    const int v = (int)((v0 >> x) & 1u) | (int)(((v1 >> x) & 1u) << 1) | (int)(((v2 >> x) & 1u) << 2);
    // floor(x / D) = umulhi(x, ceil(2^32 / D)) for x < 2^32 / D (x <= 5 d < 5 D)
    const int rf = (int)__umulhi((uint32_t)(min(v + 1, vk) * d), Dmul),
              rb = (int)__umulhi((uint32_t)(vk * d), Dmul);
    // ahead >= rf: tg_rf at x; behind >= rb: target cells x-1..x-rb empty,
    // cells before the row start count as empty
    const uint32_t tg = rf <= 0 ? FULL : rf == 1 ? tg1 : rf == 2 ? tg2 : rf == 3 ? tg3
                      : rf == 4 ? tg4 : tg5;
    bool ok = (tg >> x) & 1u;
    if (rb > 0) {
      const uint32_t behind = __funnelshift_lc(tp, t0, 32 - x);  // bit j: cell c0+x-32+j
      const uint32_t need = ((1u << rb) - 1u) << (32 - rb);       // cells x-rb..x-1
      const int c = c0 + x;
      const uint32_t valid = c >= 32 ? FULL : (c == 0 ? 0u : ~((1u << (32 - c)) - 1u));
      if (behind & need & valid) ok = false;
    }
    if (ok) lv |= 1u << x;
  }
  return lv;
}

#ifndef TS_ROWS_INJ_TMPL
#define TS_ROWS_INJ_TMPL 1  // injection as a template mode bit (else a runtime test)
#endif
// The slowdown draws of a group whose vid block is not staged (more vehicles
// than the staging capacity; rare): the mover list in chunks of the
// capacity, vids from global memory; brake bits into bw[row * NW + word]
static __device__ __noinline__ void draws_unstaged(RowWords U1, RowWords O, int lane, int in_off,
                                                   int moff, int mtot, int cap, int32_t *mlist,
                                                   uint32_t *bw, const int32_t *vbase, uint32_t t,
                                                   uint32_t k0, uint32_t k1, uint64_t p32) {
  for (int base = 0; base < mtot; base += cap) {
    int j = moff - base, rb = in_off;
#pragma unroll 1
    for (int i = 0; i < kRowWords; i++) {
      uint32_t m = U1.w[i];
      const uint32_t o = O.w[i];
      while (m) {
        const int x = __ffs(m) - 1;
        m &= m - 1u;
        if (j >= 0 && j < cap)
          mlist[j] = ((rb + __popc(o & ((1u << x) - 1u))) << 12) | (lane << 7) | (32 * i + x);
        j++;
      }
      rb += __popc(o);
    }
    __syncwarp();
    const int n = min(mtot - base, cap);
    for (int jj = lane; jj < n; jj += 32) {
      const uint32_t me = (uint32_t)mlist[jj];
      const uint32_t e = (uint32_t)vbase[me >> 12];
      if ((uint64_t)philox_w0(t, e & kVidMask, k0, k1) < p32)
        atomicOr(bw + ((me >> 5) & 127u), 1u << (me & 31u));
    }
    __syncwarp();
  }
}

// Vid lists of the final state (the group's output block): rows whose
// vehicle set only lost its front or gained a back entrant are (shifted)
// prefix copies of their input list; rows whose set changed inside (lane
// changes, injections) scatter every vehicle of S(t+1) before the lane
// change to its rank in the final occupancy of its row (own, or l + dir),
// 32 at a time across the warp from the rows' masks published in aux.
// ibase / obase: the group's input / output block (shared memory when
// staged, else global); inj_scratch: the group's injection scratch.
template <int NWT>
__device__ __forceinline__ void vid_lists(const int32_t *ibase, int32_t *obase, int32_t *aux,
                                          const uint32_t (&OO)[NWT], const uint32_t (&FO)[NWT],
                                          const uint32_t (&LV)[NWT], const uint32_t (&INJ)[NWT],
                                          int nfin, int in_off, int out_off, bool has_ent, int ent_y,
                                          uint32_t ent_e, bool changed, bool ginj, int dir,
                                          int lane, const int32_t *inj_scratch) {
  constexpr int NW = NWT;
  const int32_t *vin = ibase + in_off;
  int32_t *vout = obase + out_off;
  if (!changed && nfin > 0) {
    // input vehicles minus an exit at the front (a prefix of the input
    // list), shifted by one when the entrant lands behind every vehicle
    const int sh = has_ent ? 1 : 0;
    if (has_ent) vout[0] = (int32_t)ent_e;
    int i = sh;
    for (; i + 4 <= nfin; i += 4) {
      const int32_t a0 = vin[i - sh], a1 = vin[i + 1 - sh], a2 = vin[i + 2 - sh],
                    a3 = vin[i + 3 - sh];
      vout[i] = a0;
      vout[i + 1] = a1;
      vout[i + 2] = a2;
      vout[i + 3] = a3;
    }
    for (; i < nfin; i++) vout[i] = vin[i - sh];
  }
  if (const uint32_t gmask = __ballot_sync(FULL, changed)) {
    // rows whose vehicle set changed inside (lane changes, injections):
    // every vehicle of S(t+1) before the lane change goes to its rank in
    // the final occupancy of its row (own, or l + dir).  The vehicles of
    // all such rows are processed 32 at a time across the warp from the
    // rows' masks published in shared memory.
    uint32_t *rOO = reinterpret_cast<uint32_t *>(aux), *rFO = rOO + 32 * NW,
             *rLV = rFO + 32 * NW, *rIN = rLV + 32 * NW;
    int32_t *mInOff = aux + 4 * 32 * NW, *mOutOff = mInOff + 32, *mEnt = mOutOff + 32,
            *mEntE = mEnt + 32, *mItem = mEntE + 32;  // mItem: 33 entries
    // per row: popcount prefixes of the OO / FO words (bytes 1..3: words 0,
    // 0-1, 0-2), so an item finds its word and its rank without loops
    uint32_t *pOO = reinterpret_cast<uint32_t *>(mItem + 36), *pFO = pOO + 32;
    {
      uint32_t po = 0u, pf = 0u;
      int so = 0, sf = 0;
#pragma unroll
      for (int i = 0; i < NW; i++) {
        rOO[lane * NW + i] = OO[i];
        rFO[lane * NW + i] = FO[i];
        rLV[lane * NW + i] = LV[i];
        if (ginj) rIN[lane * NW + i] = INJ[i];
        if (i > 0) {
          po |= (uint32_t)so << (8 * i);
          pf |= (uint32_t)sf << (8 * i);
        }
        so += __popc(OO[i]);
        sf += __popc(FO[i]);
      }
      pOO[lane] = po;
      pFO[lane] = pf;
    }
    mInOff[lane] = in_off;
    mOutOff[lane] = out_off;
    mEnt[lane] = ent_y;
    mEntE[lane] = (int32_t)ent_e;
    int itot;
    const int ioff = warp_scan(changed ? popc_row(OO) : 0, lane, &itot);
    mItem[lane] = ioff;
    if (lane == 0) mItem[32] = itot;
    __syncwarp();
    for (int J = lane; J < itot; J += 32) {
      // the row of item J: the last row whose first item is <= J
      int r0 = 0;
#pragma unroll
      for (int st = 16; st; st >>= 1)
        if (mItem[r0 + st] <= J) r0 += st;
      const int rr = J - mItem[r0];  // rank of the vehicle in the row's OO
      // the word holding set bit number rr, and the rank inside it
      const uint32_t po = pOO[r0];
      const int p1 = (int)((po >> 8) & 0xFF), p2 = (int)((po >> 16) & 0xFF), p3 = (int)(po >> 24);
      const int wi = (rr >= p1) + (rr >= p2) + (rr >= p3);
      uint32_t wsel = rOO[r0 * NW + wi];
      int c = 32 * wi, k2 = rr - (int)((po >> (8 * wi)) & 0xFF);
      {  // select bit k2 of wsel by popcount halving
        uint32_t m = wsel;
        int pos = 0, cnt = __popc(m & 0xFFFFu);
        if (k2 >= cnt) { k2 -= cnt; pos = 16; m >>= 16; }
        cnt = __popc(m & 0xFFu);
        if (k2 >= cnt) { k2 -= cnt; pos += 8; m >>= 8; }
        cnt = __popc(m & 0xFu);
        if (k2 >= cnt) { k2 -= cnt; pos += 4; m >>= 4; }
        cnt = __popc(m & 0x3u);
        if (k2 >= cnt) { k2 -= cnt; pos += 2; m >>= 2; }
        c += pos + (k2 >= (int)(m & 1u) ? 1 : 0);
      }
      const int ci = c >> 5;
      const uint32_t bit = 1u << (c & 31), lowb = bit - 1u;
      const uint32_t inj_w = ginj ? rIN[r0 * NW + ci] : 0u;
      uint32_t e;
      if (c == mEnt[r0]) {
        e = (uint32_t)mEntE[r0];
      } else if (inj_w & bit) {
        e = (uint32_t)inj_scratch[(size_t)r0 * kRowMaxCells + c];
      } else {
        int ninj = 0;
        if (ginj) {
          ninj = __popc(inj_w & lowb);
          for (int i = 0; i < ci; i++) ninj += __popc(rIN[r0 * NW + i]);
        }
        const int me = (mEnt[r0] >= 0 && mEnt[r0] < c) ? 1 : 0;
        e = (uint32_t)ibase[mInOff[r0] + rr - me - ninj];
      }
      const int dst = (rLV[r0 * NW + ci] & bit) ? r0 + dir : r0;
      const int rank = __popc(rFO[dst * NW + ci] & lowb) + (int)((pFO[dst] >> (8 * ci)) & 0xFF);
      TS_CHK(rFO[dst * NW + ci] & bit, 64, 0xFFFFFFF0u);
      obase[mOutOff[dst] + rank] = (int32_t)e;
    }
  }
}

// The vid lists of a staged group without injections (the common case),
// lane-change rows by (row, word) items: every lane-change row publishes its masks, prefix
// counts and offsets; then the warp takes the items (row, word) 32 at a
// time and each lane writes the vehicles of its word of S(t+1) (before the
// lane change) to their ranks in the final occupancy -- of their own row,
// or of l + dir for a leaver.  The per-row data is loaded once per item,
// not per vehicle, and the words of one round carry similar numbers of
// vehicles (unlike whole rows).  (It replaced a per-vehicle cell table +
// warp scatter: k_rows -3.3 % in the driver's window, -1.1 % at steady
// state.)
template <int NWT>
__device__ __forceinline__ void vid_lists_rw(const int32_t *ibase, int32_t *obase, int32_t *aux,
                                             const uint32_t (&OO)[NWT], const uint32_t (&FO)[NWT],
                                             const uint32_t (&LV)[NWT], int nfin, int in_off,
                                             int out_off, bool has_ent, int ent_y, uint32_t ent_e,
                                             bool changed, int dir, int lane) {
  constexpr int NW = NWT;
  const int32_t *vin = ibase + in_off;
  int32_t *vout = obase + out_off;
  if (!changed && nfin > 0) {  // (shifted) prefix copy, as in vid_lists
    const int sh = has_ent ? 1 : 0;
    if (has_ent) vout[0] = (int32_t)ent_e;
    int i = sh;
    for (; i + 4 <= nfin; i += 4) {
      const int32_t a0 = vin[i - sh], a1 = vin[i + 1 - sh], a2 = vin[i + 2 - sh],
                    a3 = vin[i + 3 - sh];
      vout[i] = a0;
      vout[i + 1] = a1;
      vout[i + 2] = a2;
      vout[i + 3] = a3;
    }
    for (; i < nfin; i++) vout[i] = vin[i - sh];
  }
  const uint32_t cm = __ballot_sync(FULL, changed);
  if (cm == 0u) return;  // warp-uniform
  // aux: rOO, rFO, rLV (32 x NW each), then per row: pOO, pFO (byte i =
  // count of words before i), mIn (input index of its rank-0 vehicle: the
  // entrant, if any, counts as rank 0 and is not in the input), mOut, mEnt,
  // and the list of the lane-change rows
  uint32_t *rOO = reinterpret_cast<uint32_t *>(aux), *rFO = rOO + 32 * NW, *rLV = rFO + 32 * NW;
  uint32_t *pOO = rLV + 32 * NW, *pFO = pOO + 32;
  int32_t *mIn = reinterpret_cast<int32_t *>(pFO + 32), *mOut = mIn + 32, *mEnt = mOut + 32,
          *rlist = mEnt + 32;
  {
    uint32_t po = 0u, pf = 0u;
    int so = 0, sf = 0;
#pragma unroll
    for (int i = 0; i < NW; i++) {
      rFO[lane * NW + i] = FO[i];
      if (changed) {
        rOO[lane * NW + i] = OO[i];
        rLV[lane * NW + i] = LV[i];
      }
      if (i > 0) {
        po |= (uint32_t)so << (8 * i);
        pf |= (uint32_t)sf << (8 * i);
      }
      so += __popc(OO[i]);
      sf += __popc(FO[i]);
    }
    pOO[lane] = po;
    pFO[lane] = pf;
  }
  mIn[lane] = in_off - (ent_y >= 0 ? 1 : 0);
  mOut[lane] = out_off;
  mEnt[lane] = ent_y >= 0 ? (int32_t)ent_e : -1;
  if (changed) rlist[__popc(cm & ((1u << lane) - 1u))] = lane;
  __syncwarp();
  const int nitems = __popc(cm) * NW;
  for (int J = lane; J < nitems; J += 32) {
    const int r = rlist[J / NW], i = J % NW;
    uint32_t m = rOO[r * NW + i];
    if (!m) continue;
    const uint32_t lvw = rLV[r * NW + i], fo = rFO[r * NW + i];
    int k = (int)((pOO[r] >> (8 * i)) & 0xFFu);  // rank in the row's OO of the word's first vehicle
    const int in0 = mIn[r], ent = mEnt[r];
    const int of = mOut[r] + (int)((pFO[r] >> (8 * i)) & 0xFFu);
    int ot = 0;
    uint32_t fot = 0u;
    if (lvw) {  // the target row of its leavers
      const int r2 = r + dir;
      fot = rFO[r2 * NW + i];
      ot = mOut[r2] + (int)((pFO[r2] >> (8 * i)) & 0xFFu);
    }
    do {
      const uint32_t bit = m & (0u - m), lowb = bit - 1u;
      m ^= bit;
      const uint32_t e = (k == 0 && ent != -1) ? (uint32_t)ent : (uint32_t)ibase[in0 + k];
      k++;
      const int dst = (lvw & bit) ? ot + __popc(fot & lowb) : of + __popc(fo & lowb);
      TS_CHK(((lvw & bit) ? fot : fo) & bit, 64, 0xFFFFFFF0u);
      obase[dst] = (int32_t)e;
    } while (m);
  }
}

// the same out of line, for groups whose blocks are not staged (rare)
static __device__ __noinline__ void vid_lists_global(const int32_t *ibase, int32_t *obase,
                                                     int32_t *aux, RowWords OO, RowWords FO,
                                                     RowWords LV, RowWords INJ, int nfin,
                                                     int in_off, int out_off, bool has_ent,
                                                     int ent_y, uint32_t ent_e, bool changed,
                                                     bool ginj, int dir, int lane,
                                                     const int32_t *inj_scratch) {
  vid_lists(ibase, obase, aux, OO.w, FO.w, LV.w, INJ.w, nfin, in_off, out_off, has_ent, ent_y,
            ent_e, changed, ginj, dir, lane, inj_scratch);
}

#ifndef TS_ROWS_DRAW2
#define TS_ROWS_DRAW2 1  // two Philox chains per lane in the draw loop
#endif
#ifndef TS_ROWS_WARP_FLUSH
#define TS_ROWS_WARP_FLUSH 1  // counters flushed per warp (no block barrier at the end)
#endif
#ifndef TS_ROWS_MINB
#define TS_ROWS_MINB (512 / TS_ROWS_TPB)  // resident blocks per SM: 128 registers (96 measured 2.5% slower)
#endif
// MODE = the uniform mode bits kModeMove | kModeLC | kModeHash of the launch
// (specialised so the hot fused instantiation carries no dead paths)
template <int MODE>
__global__ void __launch_bounds__(TS_ROWS_TPB, TS_ROWS_MINB) k_rows(const StepParams P_, const RowsParams R) {
  const StepParams P = with_time(P_);
  __shared__ unsigned long long red[(TS_ROWS_TPB / 32) * 8];
  __shared__ uint64_t vbar[TS_ROWS_TPB / 32];   // per warp: vid block arrival
  extern __shared__ __align__(16) int32_t stage[];  // per warp: vid block in, vid block out
  const int lane = threadIdx.x & 31;
  int32_t *s_in = stage + (threadIdx.x >> 5) * rows_stage_words(R.cap);
  int32_t *s_out = s_in + R.cap;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  constexpr bool do_move = (MODE & kModeMove) != 0;
  constexpr bool hash = (MODE & kModeHash) != 0;
  constexpr bool lc = (MODE & kModeLC) != 0;
  constexpr bool halo = (MODE & kModeHalo) != 0;  // ring segment rows
  constexpr bool inject = (MODE & kModeInject) != 0;  // injection from parking (pending trips)
  const int lct = do_move ? P.t + 1 : P.t;  // time of the lane-change sub-step
  const int dir = (lct & 1) ? -1 : +1;      // R4
  Acc acc = {};
  Acc acc_next = {};
  bool dep_done = false;  // programmatic dependent launch: node output not yet awaited
  grid_dep_launch();      // the next node kernel may start its prologue

  // groups are handed out dynamically (one atomic per warp and group): no
  // warp idles while another still has a queue of groups (a static
  // round-robin assignment measured 6-11 % slower: the groups' work varies).
  // Every warp's first group is its warp index (no atomic at the start,
  // where all warps would queue on the one counter); later groups come from
  // the counter, offset by the warp count; the next group is fetched one
  // iteration ahead
  auto grab = [&]() {
    int g = 0;
    if (lane == 0) g = (int)(atomicAdd(R.gctr, 1ull) - R.gbase) + (TS_ROWS_FIRST_STATIC ? nwarps : 0);
    return __shfl_sync(FULL, g, 0);
  };
  uint64_t *bar = &vbar[threadIdx.x >> 5];
  uint32_t bar_phase = 0;
  if (lane == 0) mbar_init(bar);
  __syncwarp();
#if TS_ROWS_FIRST_STATIC
  int g_next = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
#else
  int g_next = grab();
#endif
  // the next group's vid-block offset and vehicle count, loaded one
  // iteration ahead (the bulk copy of its block needs them first)
  int voff_n = 0, tot_n = 0;
  if (g_next < R.ngroups) {
    voff_n = R.gvoff[g_next];
    tot_n = R.gcnt_in[g_next];
  }
  // the next group's planes are loaded into registers once this group's
  // input planes are dead (after the hop), so they are in flight while this
  // group changes lanes and builds its vid lists (measured: k_rows -2.8 %
  // in the driver's window, -4.3 % at steady state; a shared-memory prefetch
  // buffer measured 3-4 % slower: it cost occupancy)
  uint32_t nP[kStatePlanes][NW];
  auto load_planes = [&](int gg) {
    const uint32_t *pin = R.planes_in + group_plane_base(gg) + lane;
#pragma unroll
    for (int q = 0; q < kStatePlanes; q++)
#pragma unroll
      for (int i = 0; i < NW; i++) nP[q][i] = __ldcs(pin + (q * NW + i) * 32);
  };
  if (g_next < R.ngroups) load_planes(g_next);
  // the packed descriptor word (w, l, L, vk) of the next group is loaded
  // with its planes (-1.7 % / -2.2 %; its node grants and entrants loaded
  // there too measured +1.2 %)
  uint32_t n_dw = 0u;
  if (g_next < R.ngroups) n_dw = reinterpret_cast<const uint32_t *>(R.rows + (size_t)g_next * 32 + lane)[3];
  for (;;) {
    const int g = g_next;
    if (g >= R.ngroups) break;
    g_next = grab();
    if (lane == 0) bulk_wait_read();  // the previous group's output block
    uint32_t O[NW], V0[NW], V1[NW], V2[NW], A0[NW], A1[NW];
#pragma unroll
    for (int i = 0; i < NW; i++) {
      O[i] = nP[0][i];
      V0[i] = nP[1][i];
      V1[i] = nP[2][i];
      V2[i] = nP[3][i];
      A0[i] = nP[4][i];
      A1[i] = nP[5][i];
    }
    __syncwarp();  // the previous group's staged blocks are free
    const RowDesc rd = R.rows[(size_t)g * 32 + lane];
    const uint32_t dw = n_dw;  // RowDesc bytes 12..15: w, l, L, vk
    const int w = (int)(dw & 0xFF), l = (int)((dw >> 8) & 0xFF), L = (int)((dw >> 16) & 0xFF),
              link = rd.link, lg = rd.lg, vk = (int)(dw >> 24);
    const int voff = voff_n;
    // the group's vid block (its vehicle count was written with it) is
    // staged in shared memory when it fits, loaded together with the planes
    const int tot_in = tot_n;
    const bool staged = tot_in <= R.cap;
    const bool tma_in = staged && tot_in > 0;
    if (tma_in && lane == 0) {  // the previous group's generic reads of s_in come first
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(s_in, R.vid_in + voff, tot_in, bar);
    }
    // per-row gathers of this step, issued early: node grant, entrant,
    // pending trips
    const bool do_move0 = do_move && w > 0;
    if (!dep_done) {  // the node grants / entrants are the previous kernel's output
      grid_dep_wait();
      dep_done = true;
    }
    // node grant and entrant by row slot (no dependence on the descriptor)
    const int ext_raw = do_move ? (int)P.ext_row[(size_t)g * 32 + lane] : 0;
    const uint64_t ent_raw = do_move ? P.entr_row[(size_t)g * 32 + lane] : 0ull;
    const int ext_lg = do_move0 ? ext_raw : 0;
    const uint64_t ent_rec = do_move0 ? ent_raw : 0ull;
    const bool may_inject = (TS_ROWS_INJ_TMPL ? inject : (P.mode & kModeInject) != 0) && w > 0 && l == 0 &&
                            P.pend_off[link + 1] > P.pend_head[link];
    uint32_t VAL[NW];
#pragma unroll
    for (int i = 0; i < NW; i++) VAL[i] = lowm(w - 32 * i);
    const int nin = popc_row(O);
    int tot_chk;
    const int in_off = warp_scan(nin, lane, &tot_chk);
    TS_CHK(tot_chk == tot_in, 1, g);
    TS_CHK(g_ts_chk[3] == 0u, 128, g);  // self-test armed by ts_debug_checks(out, 2)
#ifdef TS_CHECKED
    for (int i = 0; i < NW; i++) TS_CHK((O[i] & ~VAL[i]) == 0u, 2, g);
#endif
    auto vid_wait = [&]() {
      if (tma_in) {
        mbar_wait(bar, bar_phase);
        bar_phase ^= 1u;
      }
      __syncwarp();
    };
    // a move launch waits for the block only before its draws (the front's
    // gap comes from the grant, not from its list entry): the bulk copy
    // overlaps the thermometer code and the mover list (-0.8 % / -1 %)
    if (!do_move) vid_wait();
    const int32_t *vin = (staged ? (const int32_t *)s_in : R.vid_in + voff) + in_off;
    acc.work += nin;
    if ((P.mode & kModeWork) && P.link_work && nin)
      atomicAdd(P.link_work + link, (unsigned long long)nin);

    // S(t+1) before its lane change: OO (occupancy), OV0..2, OA0/1
    uint32_t OO[NW], OV0[NW], OV1[NW], OV2[NW], OA0[NW], OA1[NW];
    bool has_ent = false;
    int ent_y = -1;
    uint32_t ent_e = 0u;
    uint32_t efront = 0u;
    if (do_move) {
      // front vehicle inside the last 5 cells: its list entry (out-slot)
      const int xf = top_row(O);
      const int nb = min(w, kGmax);
      const bool front_zone = xf >= w - nb && xf >= 0;
      // ---- thermometer codes U_k = (v2 >= k), word by word; cells past the
      //      row end count as occupied.  The row front near the stop line
      //      takes its gap from the node grant (H3) or the open end of its
      //      final link (R12): fv2 = its v2 when that lets it go past d.
      uint32_t Oext[NW];
#pragma unroll
      for (int i = 0; i < NW; i++) Oext[i] = O[i] | ~VAL[i];
      int fd = 99, fv2 = 0;
      if (front_zone) {
        const int d = w - 1 - xf;
        // (the node kernel grants kGmax to a front on its final link, R12)
        const int gp = min(kGmax, d + ext_lg);
        if (gp > d) {
          const int v = bit_row(V0, xf) | (bit_row(V1, xf) << 1) | (bit_row(V2, xf) << 2);
          fd = d;
          fv2 = min(min(v + 1, vk), gp);
        }
      }
      const int xw = xf >> 5;  // the front's word and bit
      const uint32_t xbit = 1u << (xf & 31);
      // U_k of word i (k = 1..5)
      auto thermo = [&](int i, uint32_t (&u)[5]) {
        const uint32_t o0 = Oext[i], o1 = i + 1 < NW ? Oext[i + 1] : FULL;
        uint32_t f = FULL;
#pragma unroll
        for (int k = 1; k <= 5; k++) {
          f &= ~__funnelshift_r(o0, o1, k);
          uint32_t T;
          if (k == 1) T = O[i];
          else if (k == 2) T = vk >= 2 ? (V0[i] | V1[i] | V2[i]) : 0u;  // v >= 1
          else if (k == 3) T = vk >= 3 ? (V1[i] | V2[i]) : 0u;          // v >= 2
          else if (k == 4) T = vk >= 4 ? (V2[i] | (V1[i] & V0[i])) : 0u;  // v >= 3
          else T = vk >= 5 ? V2[i] : 0u;                                  // v >= 4
          u[k - 1] = T & f;
          if (i == xw && k > fd && k <= fv2) u[k - 1] |= xbit;
        }
      };
      uint32_t U1[NW];  // movers: v2 >= 1
#pragma unroll
      for (int i = 0; i < NW; i++) {
        const uint32_t o1 = i + 1 < NW ? Oext[i + 1] : FULL;
        U1[i] = O[i] & ~__funnelshift_r(Oext[i], o1, 1);
        if (i == xw && fd == 0 && fv2 >= 1) U1[i] |= xbit;
      }
      // ---- Philox slowdown draws (R3) of the vehicles with v2 >= 1, 32 at a
      //      time across the warp: each row lists the block offsets of its
      //      movers, the warp draws for the whole list (full lanes), each row
      //      takes its brake bits back in order
      uint32_t Bm[NW];
      {
        int mtot;
        const int mc = popc_row(U1);
        const int moff = warp_scan(mc, lane, &mtot);
        // mover list entries: block offset << 12 | row slot << 7 | cell
        int32_t *mlist = s_out;  // free until the output phase
        uint32_t *bw = reinterpret_cast<uint32_t *>(s_out + R.cap);
#pragma unroll
        for (int i = 0; i < NW; i++) bw[lane * NW + i] = 0u;  // this row's brake bits
        // brake iff u < p32, i.e. u <= p32 - 1 (p32 in [1, 2^32]; p32 = 0 draws nothing)
        const uint32_t p32m1 = (uint32_t)(P.p32 - 1);
        if (staged) {  // mtot <= tot_in <= cap: the whole list fits
          int j = moff, rb = in_off;
#pragma unroll
          for (int i = 0; i < NW; i++) {
            uint32_t m = U1[i];
            const uint32_t o = O[i];
            const int b = (rb << 12) | (lane << 7) | (32 * i);
            while (m) {
              const uint32_t lsb = m & (0u - m), below = lsb - 1u;
              m ^= lsb;
              mlist[j++] = b + (__popc(o & below) << 12) + __popc(below);
            }
            rb += __popc(o);
          }
          vid_wait();  // the vid block has arrived (includes the warp barrier)
          // the draws: the vid from the staged block; brake bit by a shared-
          // memory reduction at word (row slot * NW + word) = (entry >> 5) & 127
          const uint32_t bw_s = (uint32_t)__cvta_generic_to_shared(bw);
          // the Philox round keys: launch parameters, read by the rounds as
          // uniform (constant-bank) operands -- no per-lane registers (copying
          // them into registers measured 1.5 % slower in the window)
          uint32_t rk[20];
#pragma unroll
          for (int r = 0; r < 20; r++) rk[r] = P_.rk[r];
          if (P.p32 != 0) {
#if TS_ROWS_DRAW2
            // two independent Philox chains per lane and iteration
            int jj = lane;
            for (; jj + 32 < mtot; jj += 64) {
              const uint32_t me0 = (uint32_t)mlist[jj], me1 = (uint32_t)mlist[jj + 32];
              const uint32_t e0 = (uint32_t)s_in[me0 >> 12], e1 = (uint32_t)s_in[me1 >> 12];
              const uint32_t b0 = philox_w0_rk((uint32_t)P.t, e0 & kVidMask, rk) <= p32m1 ? 1u : 0u;
              const uint32_t b1 = philox_w0_rk((uint32_t)P.t, e1 & kVidMask, rk) <= p32m1 ? 1u : 0u;
              red_or_shared(bw_s + (((me0 >> 5) & 127u) << 2), b0 << (me0 & 31u));
              red_or_shared(bw_s + (((me1 >> 5) & 127u) << 2), b1 << (me1 & 31u));
            }
            for (; jj < mtot; jj += 32) {
#else
            for (int jj = lane; jj < mtot; jj += 32) {
#endif
              const uint32_t me = (uint32_t)mlist[jj];
              const uint32_t e = (uint32_t)s_in[me >> 12];
              // no branch: every lane ORs its brake bit, or 0 (measured faster
              // than a divergent reduction of the ~20 % that brake)
              const uint32_t brk = philox_w0_rk((uint32_t)P.t, e & kVidMask, rk) <= p32m1 ? 1u : 0u;
              red_or_shared(bw_s + (((me >> 5) & 127u) << 2), brk << (me & 31u));
            }
          }
          __syncwarp();
        } else {  // a group larger than the staging (rare): out of line
          vid_wait();
          RowWords u1w, ow;
#pragma unroll
          for (int i = 0; i < NW; i++) {
            u1w.w[i] = U1[i];
            ow.w[i] = O[i];
          }
          draws_unstaged(u1w, ow, lane, in_off, moff, mtot, R.cap, mlist, bw, R.vid_in + voff,
                         (uint32_t)P.t, P.k0, P.k1, P.p32);
        }
#pragma unroll
        for (int i = 0; i < NW; i++) Bm[i] = bw[lane * NW + i];
        __syncwarp();
      }
      if (front_zone) efront = (uint32_t)vin[nin - 1];  // for an exit (below)
      // ---- hop, word by word: D_k = vehicles moving exactly k (v3 = k);
      //      those passing the row end leave it (LR); O' = OR_k D_k << k with
      //      the velocity and class bits carried along
      uint32_t LR = 0u, Dp[6], DpA0[6], DpA1[6];
#pragma unroll
      for (int k = 0; k < 6; k++) Dp[k] = DpA0[k] = DpA1[k] = 0u;
#pragma unroll
      for (int i = 0; i < NW; i++) {
        uint32_t u[5];
        thermo(i, u);
        const uint32_t b = Bm[i];
        uint32_t W[6];
#pragma unroll
        for (int k = 1; k <= 5; k++)
          W[k - 1] = (u[k - 1] & ~b) | ((k < 5 ? u[k] : 0u) & b);  // v3 >= k
        W[5] = 0u;
        const uint32_t D0 = O[i] & ~W[0];
        uint32_t oo = D0, ov0 = 0u, ov1 = 0u, ov2 = 0u, oa0 = D0 & A0[i], oa1 = D0 & A1[i];
        const uint32_t val1 = i + 1 < NW ? VAL[i + 1] : 0u;
#pragma unroll
        for (int k = 1; k <= 5; k++) {
          const uint32_t stay = __funnelshift_r(VAL[i], val1, k);  // x + k inside the row
          const uint32_t dk0 = W[k - 1] & ~W[k];
          LR |= dk0 & ~stay;
          const uint32_t dk = dk0 & stay, da0 = dk & A0[i], da1 = dk & A1[i];
          const uint32_t sh = __funnelshift_l(Dp[k], dk, k);
          oo |= sh;
          if (k & 1) ov0 |= sh;
          if (k & 2) ov1 |= sh;
          if (k & 4) ov2 |= sh;
          oa0 |= __funnelshift_l(DpA0[k], da0, k);
          oa1 |= __funnelshift_l(DpA1[k], da1, k);
          Dp[k] = dk;
          DpA0[k] = da0;
          DpA1[k] = da1;
        }
        OO[i] = oo;
        OV0[i] = ov0;
        OV1[i] = ov1;
        OV2[i] = ov2;
        OA0[i] = oa0;
        OA1[i] = oa1;
      }
      // ---- the front left the row: exit to parking or
      //      node crossing (the node kernel placed it on the next link)
      if (LR) {
        if ((int)(efront >> kSlotShift) == kSlotFinal) {
          P.arr_time[efront & kVidMask] = P.t + 1;
          acc.arr++;
        }
      }
      // ---- entrant granted by the node kernel (H3/H5), behind every vehicle
      if (w > 0) {
        const uint64_t rec = ent_rec;
        if ((uint32_t)(rec >> 43) == ((uint32_t)(P.t + 1) & 0x1FFFFFu) && (uint32_t)rec != kNoEntrant) {
          const int code = (int)((rec >> 32) & 0xFF);
          ent_y = (int)((rec >> 40) & 7);
          set_row(OO, ent_y);
          if (code & 1) set_row(OV0, ent_y);
          if (code & 2) set_row(OV1, ent_y);
          if (code & 4) set_row(OV2, ent_y);
          const int cls = lane_class(code >> 3, P.tt_link[link]);
          if (cls & 1) set_row(OA0, ent_y);
          if (cls & 2) set_row(OA1, ent_y);
          ent_e = (uint32_t)rec | ((uint32_t)(code >> 3) << kSlotShift);
          has_ent = true;
          // consumed (reset): the 21-bit time tag would match again 2^21 steps on
          P.entr_row[(size_t)g * 32 + lane] = ~0ull;
        }
      }
    } else {  // no move: initial injection / lane change only
#pragma unroll
      for (int i = 0; i < NW; i++) {
        OO[i] = O[i];
        OV0[i] = V0[i];
        OV1[i] = V1[i];
        OV2[i] = V2[i];
        OA0[i] = A0[i];
        OA1[i] = A1[i];
      }
    }
    if (g_next < R.ngroups) {
      load_planes(g_next);  // this group's input planes are dead
      n_dw = reinterpret_cast<const uint32_t *>(R.rows + (size_t)g_next * 32 + lane)[3];
    }
    if (g_next < R.ngroups) {  // the next group's block offset and count (see above)
      voff_n = R.gvoff[g_next];
      tot_n = R.gcnt_in[g_next];
    }
    // ---- injection from parking (H6, R13): lane 0 of links with pending trips
    uint32_t INJ[NW];
#pragma unroll
    for (int i = 0; i < NW; i++) INJ[i] = 0u;
    bool injected = false;
    if (may_inject) {
      int32_t *scratch = R.inj_scratch + ((size_t)g * 32 + lane) * kRowMaxCells;
      inject_link(
          P, link, 0, w, true, [&](int x) { return !bit_row(OO, x); },
          [&](int x, uint8_t code, int ivid) {
            set_row(OO, x);
            set_row(INJ, x);
            const int cls = lane_class(code >> 3, P.tt_link[link]);
            if (cls & 1) set_row(OA0, x);
            if (cls & 2) set_row(OA1, x);
            scratch[x] = ivid | ((code >> 3) << kSlotShift);
            injected = true;
            acc.inj++;
          });
    }
    if (do_move || !lc) acc.active += popc_row(OO);
    if (do_move) acc.sumv += popc_row(OV0) + 2 * popc_row(OV1) + 4 * popc_row(OV2);

    // ---- lane change on S(t+1) (fused) or S(t) (lane change only):
    //      LV = vehicles that move to lane l + dir, AR = arrivals from l - dir
    uint32_t LV[NW], AR[NW];
#pragma unroll
    for (int i = 0; i < NW; i++) {
      LV[i] = 0u;
      AR[i] = 0u;
    }
    const bool has_tgt = w > 0 && l + dir >= 0 && l + dir < L;
    const bool has_src = w > 0 && l - dir >= 0 && l - dir < L;
    if (lc) {
      uint32_t T0[NW];
#pragma unroll
      for (int i = 0; i < NW; i++) T0[i] = shfl_w(OO[i], lane + dir);
      // ring segment rows (kModeHalo): the lane change looks across the
      // cuts -- the next segment's first cells ahead, the previous
      // segment's last cells behind (S(t), the launch's input)
      uint32_t hx = 0u, hp = 0u;
      if (halo && w > 0) {
        const int slot = g * 32 + lane;
        const int ns = R.ring_next[slot], pq = R.ring_prev[slot];
        hx = R.planes_in[group_plane_base(ns >> 5) + (ns & 31)];  // occupancy word 0
        const int ps = pq & 0xFFFFFF, pw = (int)((uint32_t)pq >> 24), kq = pw >> 5, sq = pw & 31;
        const uint32_t *pb = R.planes_in + group_plane_base(ps >> 5) + (ps & 31);
        hp = kq == 0 ? pb[0] << (32 - sq)
                     : (sq == 0 ? pb[(kq - 1) * 32] : __funnelshift_r(pb[(kq - 1) * 32], pb[kq * 32], sq));
      }
      const uint32_t thx = shfl_w(hx, lane + dir), thp = shfl_w(hp, lane + dir);
      // cells 32 i .. 32 i + 31 of a row, those past its end from the next segment
      auto ext_word = [&](const uint32_t (&X)[NW], uint32_t nx, int i) -> uint32_t {
        const int o = 32 * i - w;
        const uint32_t nxt = o >= 0 ? (o < 32 ? nx >> o : 0u) : (o > -32 ? nx << (-o) : 0u);
        if (i >= NW) return nxt;
        return (X[i] & VAL[i]) | (nxt & ~VAL[i]);
      };
      uint32_t cand[NW];
      bool anyc = false;
#pragma unroll
      for (int i = 0; i < NW; i++) {
        cand[i] = has_tgt ? (OO[i] & ~T0[i]) : 0u;
        anyc |= cand[i] != 0u;
      }
      if (anyc) {
        const int zs = P.D >= w ? 0 : w - P.D;  // desperation zone: last D cells (R6)
#pragma unroll
        for (int i = 0; i < NW; i++) {
          // word i: gaps ahead in the own and target lanes (stop at the row
          // end, R2); gap behind in the target lane (before the row start =
          // empty).  G_k / TG_k / BK_k = gap >= k.
          const uint32_t o0 = halo ? ext_word(OO, hx, i) : OO[i] | ~VAL[i],
                         o1 = halo ? ext_word(OO, hx, i + 1)
                                   : (i + 1 < NW ? (OO[i + 1] | ~VAL[i + 1]) : FULL);
          const uint32_t t0 = halo ? ext_word(T0, thx, i) : T0[i] | ~VAL[i],
                         t1 = halo ? ext_word(T0, thx, i + 1)
                                   : (i + 1 < NW ? (T0[i + 1] | ~VAL[i + 1]) : FULL);
          const uint32_t tp = i > 0 ? T0[i - 1] : (halo ? thp : 0u);
          uint32_t G[6], TG[6], BK = FULL, BKv = FULL;
          G[0] = TG[0] = FULL;
#pragma unroll
          for (int k = 1; k <= 5; k++) {
            G[k] = G[k - 1] & ~__funnelshift_r(o0, o1, k);
            TG[k] = TG[k - 1] & ~__funnelshift_r(t0, t1, k);
            BK &= ~__funnelshift_l(tp, T0[i], k);
            if (k == vk) BKv = BK;
          }
          // E_k = (v + 1 >= k)
          const uint32_t E2 = OV0[i] | OV1[i] | OV2[i], E3 = OV1[i] | OV2[i],
                         E4 = OV2[i] | (OV1[i] & OV0[i]), E5 = OV2[i], E6 = OV2[i] & OV0[i];
          // speed-motivated (R5): own gap < v+1, target gap ahead > own gap,
          // target gap behind >= V; only for vehicles free to use any lane
          const uint32_t geq =
              G[1] & (~E2 | G[2]) & (~E3 | G[3]) & (~E4 | G[4]) & (~E5 | G[5]) & ~E6;
          const uint32_t tgt = TG[1] & (~G[1] | TG[2]) & (~G[2] | TG[3]) & (~G[3] | TG[4]) &
                               (~G[4] | TG[5]) & ~G[5];
          uint32_t lv = cand[i] & ~OA0[i] & ~OA1[i] & ~geq & tgt & BKv;
          // turn-motivated (R6, R7): towards the allowed lane
          const uint32_t turn =
              cand[i] & (dir < 0 ? (OA0[i] & ~OA1[i]) : (OA1[i] & ~OA0[i]));
          if (turn) {
            const uint32_t ZN = range_w(i, zs, w);
            // ahead >= min(v+1, V), behind >= V outside the last D cells
            uint32_t req = TG[1];
            if (vk >= 2) req &= ~E2 | TG[2];
            if (vk >= 3) req &= ~E3 | TG[3];
            if (vk >= 4) req &= ~E4 | TG[4];
            if (vk >= 5) req &= ~E5 | TG[5];
            lv |= turn & ~ZN & req & BKv;
            const uint32_t zc = turn & ZN;  // scaled thresholds (R6): per candidate
            if (zc)
              lv |= zone_lc(zc, 32 * i, w, vk, P.Dmul, OV0[i], OV1[i], OV2[i], TG[1], TG[2], TG[3],
                            TG[4], TG[5], tp, T0[i]);
          }
          LV[i] = lv;
        }
      }
#pragma unroll
      for (int i = 0; i < NW; i++) AR[i] = shfl_w(LV[i], lane - dir);
      if (!has_src) {
#pragma unroll
        for (int i = 0; i < NW; i++) AR[i] = 0u;
      }
      acc_next.lc += popc_row(LV);
    }
    // ---- apply the lane changes word by word; final planes to HBM
    uint32_t FO[NW], FV0[NW], FV1[NW], FV2[NW];
    {
      uint32_t *pout = R.planes_out + group_plane_base(g) + lane;
#pragma unroll
      for (int i = 0; i < NW; i++) {
        const uint32_t keep = ~LV[i], ar = AR[i];
        uint32_t fa0 = OA0[i], fa1 = OA1[i];
        FO[i] = (OO[i] & keep) | ar;
        FV0[i] = OV0[i];
        FV1[i] = OV1[i];
        FV2[i] = OV2[i];
        if (lc) {  // arrivals carry their velocity and class bits from lane l - dir
          FV0[i] = (FV0[i] & keep) | (shfl_w(OV0[i], lane - dir) & ar);
          FV1[i] = (FV1[i] & keep) | (shfl_w(OV1[i], lane - dir) & ar);
          FV2[i] = (FV2[i] & keep) | (shfl_w(OV2[i], lane - dir) & ar);
          fa0 = (fa0 & keep) | (shfl_w(OA0[i], lane - dir) & ar);
          fa1 = (fa1 & keep) | (shfl_w(OA1[i], lane - dir) & ar);
        }
        __stcs(pout + (0 * NW + i) * 32, FO[i]);
        __stcs(pout + (1 * NW + i) * 32, FV0[i]);
        __stcs(pout + (2 * NW + i) * 32, FV1[i]);
        __stcs(pout + (3 * NW + i) * 32, FV2[i]);
        __stcs(pout + (4 * NW + i) * 32, fa0);
        __stcs(pout + (5 * NW + i) * 32, fa1);
#ifdef TS_CHECKED
        TS_CHK(((OO[i] & keep) & ar) == 0u, 4, g);
        TS_CHK((FO[i] & ~VAL[i]) == 0u, 8, g);
        for (uint32_t m = FO[i]; m; m &= m - 1u) {
          const int x = __ffs(m) - 1;
          const int v = (int)((FV0[i] >> x) & 1u) | (int)(((FV1[i] >> x) & 1u) << 1) |
                        (int)(((FV2[i] >> x) & 1u) << 2);
          TS_CHK(v <= vk, 16, g);
        }
#endif
      }
    }

    // ---- vid lists of the final state: the group's output block, staged
    //      in shared memory when it fits, written back with coalesced stores
    const int nfin = popc_row(FO);
    int tot_out;
    const int out_off = warp_scan(nfin, lane, &tot_out);
    const bool ostaged = tot_out <= R.cap;
#ifdef TS_CHECKED
    {
      int wsum;
      (void)warp_scan(w, lane, &wsum);
      TS_CHK(tot_out <= wsum, 32, g);
    }
#endif
    int32_t *obase = ostaged ? s_out : R.vid_out + voff;
    int32_t *vout = obase + out_off;
    const bool moved_lc = any_row(LV) || any_row(AR);
    // the state hash (tests) is taken below for every row, so hashed runs
    // take exactly the vid-list paths of the unhashed (benchmarked) runs
    const bool changed = moved_lc || injected;
    const bool ginj = inject && __any_sync(FULL, injected);
    const int32_t *scr = R.inj_scratch + (size_t)g * 32 * kRowMaxCells;
    if (staged && ostaged && !ginj) {  // shared-memory blocks (the common case)
      vid_lists_rw(s_in, s_out, s_out + R.cap, OO, FO, LV, nfin, in_off, out_off, has_ent, ent_y,
                   ent_e, changed, dir, lane);
    } else {
      RowWords oo, fo, lv, inj;
#pragma unroll
      for (int i = 0; i < NW; i++) {
        oo.w[i] = OO[i];
        fo.w[i] = FO[i];
        lv.w[i] = LV[i];
        inj.w[i] = INJ[i];
      }
      vid_lists_global(staged ? (const int32_t *)s_in : R.vid_in + voff, obase, s_out + R.cap, oo,
                       fo, lv, inj, nfin, in_off, out_off, has_ent, ent_y, ent_e, changed, ginj,
                       dir, lane, scr);
    }
    if (hash && (do_move || !lc) && w > 0) {  // hash of S(t+1) before its lane change (tests)
      RowWords oo, v0, v1, v2, inj;
#pragma unroll
      for (int i = 0; i < NW; i++) {
        oo.w[i] = OO[i];
        v0.w[i] = OV0[i];
        v1.w[i] = OV1[i];
        v2.w[i] = OV2[i];
        inj.w[i] = INJ[i];
      }
      acc.hash += hash_row(oo, v0, v1, v2, inj, ent_y, ent_e, vin,
                           R.inj_scratch + ((size_t)g * 32 + lane) * kRowMaxCells, link, l,
                           R.row_a ? R.row_a[g * 32 + lane] : 0);
    }
    // the output block's shared-memory writes become visible to the bulk copy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const uint32_t efin = nfin > 0 ? (uint32_t)vout[nfin - 1] : 0u;  // final front vehicle
    if (ostaged && lane == 0 && tot_out > 0) bulk_store(R.vid_out + voff, s_out, tot_out);
    if (lane == 0) R.gcnt_out[g] = tot_out;
    // ---- node records of the output S1 (read by k_node_warp, H3)
    if (lc && w > 0) {
      const int nb = min(w, kGmax);
      const int xf = top_row(FO);
      // bit j = cell n-1-j of the last nb cells
      const uint32_t occ = __brev(win_row(FO, w - nb) & lowm(nb)) >> (32 - nb);
      uint64_t rec = (uint64_t)occ << 44;
      if (occ) {
        const int xi = xf >> 5, xb = xf & 31;
        const int code = (int)((pick(FV0, xi) >> xb) & 1u) | (int)(((pick(FV1, xi) >> xb) & 1u) << 1) |
                         (int)(((pick(FV2, xi) >> xb) & 1u) << 2) | ((int)(efin >> kSlotShift) << 3);
        rec |= (uint64_t)(efin & kVidMask) | ((uint64_t)code << 32) |
               ((uint64_t)(w - 1 - xf) << 40) | (1ull << 43);
      }
      P.tail_rec[rd.nli] = rec;
      P.head_occ[lg] = (uint8_t)(FO[0] & lowm(nb));
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#if TS_ROWS_WARP_FLUSH
  flush_acc_warp(P, acc, P.t + 1);
  if (lc) flush_acc_warp(P, acc_next, lct + 1);
  (void)red;
#else
  flush_acc(P, acc, P.t + 1, red);
  if (lc) flush_acc(P, acc_next, lct + 1, red);
#endif
}

// state hash of the row-mode state S(t) (one thread per lane-row)
__global__ void __launch_bounds__(128) k_rows_hash(const RowsParams R, unsigned long long *out) {
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  const int g = gid >> 5, lane = gid & 31;
  uint64_t h = 0, cnt = 0;
  const bool act = g < R.ngroups;
  const uint32_t *pl = R.planes_in + group_plane_base(act ? g : 0) + lane;
  int n = 0;
  if (act)
    for (int i = 0; i < NW; i++) n += __popc(pl[i * 32]);
  int tot;
  const int off = warp_scan(n, lane, &tot);
  if (act) {
    const RowDesc rd = R.rows[gid];
    const int32_t *vl = R.vid_in + R.gvoff[g] + off;
    int k = 0;
    for (int i = 0; i < NW; i++) {
      uint32_t m = pl[i * 32];
      while (m) {
        const int x = __ffs(m) - 1;
        m &= m - 1u;
        const int v = (int)((pl[(NW + i) * 32] >> x) & 1u) |
                      (int)(((pl[(2 * NW + i) * 32] >> x) & 1u) << 1) |
                      (int)(((pl[(3 * NW + i) * 32] >> x) & 1u) << 2);
        const uint32_t e = (uint32_t)vl[k++];
        h += vmix((int)(e & kVidMask), rd.link, rd.l, (R.row_a ? R.row_a[gid] : 0) + 32 * i + x, v);
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

// the mode bits that select an instantiation (injection only while trips
// are pending, so the hot instantiation of a fully placed network carries
// no injection code)
constexpr int kRowsModeMask = kModeMove | kModeLC | kModeHash | kModeHalo | (TS_ROWS_INJ_TMPL ? kModeInject : 0);
#define TS_ROWS_CASES(X)                                                                       \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15) X(36) X(44)
void launch_rows(const StepParams &p, const RowsParams &r, int blocks, int threads, int smem,
                 void *stream, bool pdl) {
  switch (p.mode & kRowsModeMask) {
#define TS_ROWS_CASE(m) \
  case m: launch_pdl(k_rows<m>, blocks, threads, smem, stream, pdl, p, r); break;
    TS_ROWS_CASES(TS_ROWS_CASE)
#undef TS_ROWS_CASE
  }
}
void launch_rows_hash(const StepParams &p, const RowsParams &r, void *stream,
                      unsigned long long *out) {
  (void)p;
  const int n = r.ngroups * 32;
  k_rows_hash<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(r, out);
}
cudaError_t set_rows_smem(int bytes) {  // only ever raised (see set_smem_attrs)
  static int current[64] = {0};  // per device
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (bytes <= current[dev]) return cudaSuccess;
  current[dev] = bytes;
  cudaError_t e = cudaSuccess;
#define TS_ROWS_ATTR(m) \
  if (cudaError_t x = cudaFuncSetAttribute(k_rows<m>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)) e = x;
  TS_ROWS_CASES(TS_ROWS_ATTR)
#undef TS_ROWS_ATTR
  return e;
}
int occupancy_rows(int threads, int smem) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_rows<kModeMove | kModeLC>, threads, smem);
  return nb;
}

}  // namespace tsim

namespace tsim {
int node_checks(unsigned int *v, int reset);  // csrc/tsim_kernels.cu
}

// Read (and optionally reset) the checked build's invariant counters of the
// current device (include/tsim.h): the row kernel's and the node kernels'.
extern "C" int ts_debug_checks(uint32_t *out, int32_t reset) {
  if (!out) return TS_EINVAL;
#ifdef TS_CHECKED
  unsigned int v[4], vn[2];
  if (cudaMemcpyFromSymbol(v, g_ts_chk, sizeof v) != cudaSuccess) return TS_EINTERNAL;
  if (tsim::node_checks(vn, reset != 0) != 0) return TS_EINTERNAL;
  out[0] = 1u;
  out[1] = v[0] | vn[0];
  out[2] = v[1];
  out[3] = v[2] + vn[1];
  if (reset) {  // 2: zero and arm the self-test, 1: zero and disarm
    const unsigned int z[4] = {0u, 0xFFFFFFFFu, 0u, reset == 2 ? 1u : 0u};
    if (cudaMemcpyToSymbol(g_ts_chk, z, sizeof z) != cudaSuccess) return TS_EINTERNAL;
  }
#else
  (void)reset;
  out[0] = 0u;
  out[1] = 0u;
  out[2] = 0xFFFFFFFFu;
  out[3] = 0u;
#endif
  return TS_OK;
}
