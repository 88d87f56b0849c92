// tsim_device.cuh -- device helpers shared by the sm_100a kernels of the
// TRANSIMS CA step (Nagel & Rickert, §3-§4; readings R1-R22 in
// DESIGN.md §3): Philox slowdown, the NaSch velocity rule, the lane-change
// rule on occupancy bitmaps, injection, per-CTA statistics.
#pragma once
#include <cuda_runtime.h>

#include "tsim_internal.h"

namespace tsim {

#define FULL 0xffffffffu

// ------------------------------------------- programmatic dependent launch
// griddepcontrol (sm_90+): a kernel launched with programmatic stream
// serialisation may start while its predecessor finishes; it must wait
// before reading the predecessor's output.  Both are no-ops otherwise.
static __device__ __forceinline__ void grid_dep_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
static __device__ __forceinline__ void grid_dep_launch() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// launch with the programmatic-serialisation attribute when pdl is set
template <typename... KArgs, typename... Args>
static inline cudaError_t launch_pdl(void (*kern)(KArgs...), int blocks, int threads, int smem,
                                     void *stream, bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(blocks);
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// ------------------------------------------------------ step time
// Kernels replayed from a CUDA graph read the step time from the device
// clock (tdev); the captured t is the offset within the graph.
template <typename Params>
static __device__ __forceinline__ Params with_time(const Params &p) {
  Params q = p;
  if (p.tdev) q.t += *p.tdev;
  return q;
}

// ------------------------------------------------------------- Philox
// Philox4x32-10 (Salmon et al., SC'11) with the curand round and Weyl
// constants, counter (t, vid, 0, 0), key (k0, k1); only output word 0 is
// used (reading R3).  The zero counter words fold away in round 1.
static __device__ __forceinline__ uint32_t philox_w0(uint32_t t, uint32_t vid, uint32_t k0,
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

// The same with the key schedule precomputed per launch (rk[2 r] / rk[2 r
// + 1] = round-r keys, kernel parameters): the round keys are operands from
// the constant bank instead of per-draw additions in registers.
static __device__ __forceinline__ uint32_t philox_w0_rk(uint32_t t, uint32_t vid,
                                                        const uint32_t (&rk)[20]) {
  uint32_t c0 = t, c1 = vid, c2 = 0u, c3 = 0u;
#pragma unroll
  for (int r = 0; r < 10; r++) {
    const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    const uint32_t n0 = hi1 ^ c1 ^ rk[2 * r], n2 = hi0 ^ c3 ^ rk[2 * r + 1];
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
static __device__ __forceinline__ int nasch_v3(int v, int Vk, int g, uint32_t t, uint32_t vid,
                                               uint32_t k0, uint32_t k1, uint64_t p32) {
  int v2 = min(min(v + 1, Vk), g);
  if (v2 > 0 && (uint64_t)philox_w0(t, vid, k0, k1) < p32) v2 -= 1;
  return v2;
}

// ---------------------------------------------------------- state hash
static __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}
static __device__ __forceinline__ uint64_t vmix(int vid, int link, int lane, int cell, int v) {
  uint64_t a = (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)link << 32);
  uint64_t b = (uint64_t)(uint32_t)cell | ((uint64_t)(uint32_t)lane << 32) |
               ((uint64_t)(uint32_t)v << 40);
  return fmix64(fmix64(a) + b * 0x9E3779B97F4A7C15ULL);
}

// ------------------------------------------------------------ bitmaps
// Flat occupancy bitmaps: bit p of position p is bits[(p >> 5) + 1]; word 0
// and the last two words are zero pads so that windows never branch.

// 4 code bytes -> 4 occupancy bits (occupied iff bit 7 clear)
static __device__ __forceinline__ uint32_t occ4(uint32_t w) {
  return ((((~w) & 0x80808080u) >> 7) * 0x01020408u) >> 24;
}

static __device__ __forceinline__ void build_bits(const uint8_t *c, uint32_t *bits, int nwords,
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

static __device__ __forceinline__ int occupied(const uint32_t *bits, int q) {
  return (bits[(q >> 5) + 1] >> (q & 31)) & 1u;
}
static __device__ __forceinline__ void set_bit(uint32_t *bits, int q) {
  atomicOr(bits + (q >> 5) + 1, 1u << (q & 31));
}
// bit i = position s+i
static __device__ __forceinline__ uint32_t win_at(const uint32_t *bits, int s) {
  return __funnelshift_r(bits[(s >> 5) + 1], bits[(s >> 5) + 2], s & 31);
}
// bit i = position q+1+i
static __device__ __forceinline__ uint32_t win_ahead(const uint32_t *bits, int q) {
  return win_at(bits, q + 1);
}
// bit i = position q-1-i
static __device__ __forceinline__ uint32_t win_behind(const uint32_t *bits, int q) {
  return __brev(win_at(bits, q - 32));
}

static __device__ __forceinline__ int ctz32(uint32_t m) { return m ? __ffs(m) - 1 : 32; }
static __device__ __forceinline__ uint32_t low_mask(int n) {  // bits [0, n), n in [0, 32]
  return n >= 32 ? FULL : ((1u << n) - 1u);
}
static __device__ __forceinline__ uint32_t range_mask(int lo, int hi) {
  lo = max(lo, 0);
  hi = min(hi, 32);
  if (lo >= hi) return 0u;
  return low_mask(hi) & ~low_mask(lo);
}

// ------------------------------------------------------- lane change
// Gaps on the flat bitmap for a lane-row whose valid range is [lo, hi):
// positions below lo are before the link start and count as empty (R2),
// the row ends at hi.
static __device__ __forceinline__ int ahead_in(const uint32_t *bits, int q, int hi) {
  return min(min(ctz32(win_ahead(bits, q)), kGmax), hi - q - 1);
}
static __device__ __forceinline__ int behind_in(const uint32_t *bits, int q, int lo) {
  uint32_t r = win_behind(bits, q);
  int nvalid = q - lo;
  if (nvalid < 32) r &= low_mask(nvalid);
  return min(ctz32(r), kGmax);
}

// O1 §LC decision (R4-R7).  q: position of the vehicle,
// q2 = its cell in the target lane; lanes l (own) and l2 (target) with valid
// ranges [lo, hi) / [lo2, hi2); d = cells to the link end.  Cheap rejections
// first: target occupied, then (speed-motivated) own gap >= v+1.
// allowed-lane class of a vehicle (R7): 0 all lanes (straight on or final
// link), 1 {0} (right turn), 2 {L-1} (left turn); tt = turn types of the
// link's out-slots (2 bits each: 0 T, 1 L, 2 R)
static __device__ __forceinline__ int lane_class(int slot, uint32_t tt) {
  if (slot == kSlotFinal) return 0;
  const int tty = (tt >> (2 * slot)) & 3;
  return tty == 0 ? 0 : (tty == 2 ? 1 : 2);
}

static __device__ __forceinline__ bool lc_rule_set(const uint32_t *bits, int q, int q2, int lo,
                                                   int hi, int lo2, int hi2, int v, int set, int l,
                                                   int l2, int L, int dir, int d, int Vk, int D);

static __device__ __forceinline__ bool lc_rule(const uint32_t *bits, int q, int q2, int lo,
                                               int hi, int lo2, int hi2, int code, int l, int l2,
                                               int L, int dir, int d, uint32_t tt, bool periodic,
                                               int Vk, int D) {
  const int set = periodic ? 0 : lane_class(code >> 3, tt);
  return lc_rule_set(bits, q, q2, lo, hi, lo2, hi2, code & 7, set, l, l2, L, dir, d, Vk, D);
}

static __device__ __forceinline__ bool lc_rule_set(const uint32_t *bits, int q, int q2, int lo,
                                                   int hi, int lo2, int hi2, int v, int set, int l,
                                                   int l2, int L, int dir, int d, int Vk, int D) {
  if (occupied(bits, q2)) return false;
  const bool own_ok = set == 0 || (set == 1 ? l == 0 : l == L - 1);
  if (own_ok) {
    // speed-motivated (R5): own gap < v+1, target gap larger, back gap >= V
    const bool tgt_ok = set == 0 || (set == 1 ? l2 == 0 : l2 == L - 1);
    if (!tgt_ok) return false;
    const int g = ahead_in(bits, q, hi);
    if (g >= v + 1) return false;
    return ahead_in(bits, q2, hi2) > g && behind_in(bits, q2, lo2) >= Vk;
  }
  // turn-motivated, only towards the allowed lane; desperation (R6)
  const bool toward = (set == 1 && dir < 0) || (set == 2 && dir > 0);
  if (!toward) return false;
  int rf = min(v + 1, Vk), rb = Vk;
  if (d < D) {
    rf = (rf * d) / D;
    rb = (rb * d) / D;
  }
  return ahead_in(bits, q2, hi2) >= rf && behind_in(bits, q2, lo2) >= rb;
}

// ------------------------------------------------------------ counters
struct Acc {
  uint64_t hash, sumv;
  uint32_t active, arr, inj, lc, work;
};

static __device__ __forceinline__ void acc_place(Acc &a, bool hash, int vid, int link, int l,
                                                 int x, int v) {
  a.active++;
  a.sumv += v;
  if (hash) a.hash += vmix(vid, link, l, x, v);
}

// warp reduction of the counters into the stats slot of time slot_t (no
// block barrier: a warp that finishes early exits)
static __device__ void flush_acc_warp(const StepParams &P, Acc &a, int slot_t) {
  const int lane = threadIdx.x & 31;
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
    unsigned long long *st = P.stats + (size_t)(slot_t & (kHist - 1)) * ST_N;
    if (h) atomicAdd(st + ST_HASH, (unsigned long long)h);
    if (act) atomicAdd(st + ST_ACTIVE, (unsigned long long)act);
    if (arr) atomicAdd(st + ST_ARR, (unsigned long long)arr);
    if (inj) atomicAdd(st + ST_INJ, (unsigned long long)inj);
    if (lc) atomicAdd(st + ST_LC, (unsigned long long)lc);
    if (sv) atomicAdd(st + ST_SUMV, (unsigned long long)sv);
  }
}

// block reduction of the counters into the stats slot of time slot_t
static __device__ void flush_acc(const StepParams &P, Acc &a, int slot_t,
                                 unsigned long long *smem_red) {
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

// ------------------------------------------------------------ parking
// Injection from parking (R13) by one thread: walks the
// link's pending list in (departure, vid) order; the first vehicle to find
// its entry cell (lane 0) empty takes it with v = 0, the others retry.
template <class FreeFn, class PlaceFn>
static __device__ __forceinline__ void inject_link(const StepParams &P, int k, int a, int w,
                                                   bool first, FreeFn cell_free,
                                                   PlaceFn place_fn) {
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
    const VehPos q = P.vpos[vid];
    const int slot0 = (q.e - q.p > 1) ? (int)P.rslot[q.p + 1] : kSlotFinal;
    P.inj_time[vid] = tn;
    place_fn(ec - a, (uint8_t)(slot0 << 3), vid);
  }
  if (first) {
    while (h < e && P.inj_time[P.pend_list[h]] <= tn) h++;
    P.pend_head[k] = h;
  }
}

}  // namespace tsim
