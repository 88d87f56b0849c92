// tsim_internal.h -- device layout shared by the host driver (tsim_api.cu)
// and the sm_100a kernels (tsim_kernels.cu).  See DESIGN.md §6 for the
// layout rationale.
#pragma once
#include <cstdint>

namespace tsim {

constexpr int kGmax = 5;          // interaction range, PAPER.md:390-395 (R2)
constexpr int kSlotFinal = 15;    // code slot: vehicle is on its final link
constexpr uint8_t kEmpty = 0xFF;  // empty lane-cell code
constexpr int kHist = 4096;       // per-step stats ring buffer
constexpr int kHaloPad = 16;      // smem pad on both sides of a halo tile row
constexpr int kMaxLanes = 8;

// Cell code (one byte per lane-cell): 0xFF empty, else bits 0-2 velocity
// (0..5) and bits 3-6 the out-slot of the vehicle's next route link at the
// link's downstream node (15 = final link).  Occupied iff bit 7 is clear.

// Tile flags
constexpr uint8_t kFirst = 1;     // tile starts at cell 0 of a non-periodic link
constexpr uint8_t kLast = 2;      // tile ends at the end of a non-periodic link
constexpr uint8_t kPeriodic = 4;  // tile of the periodic (ring) link
constexpr uint8_t kHalo = 8;      // tile reads 5-cell halos from strips
constexpr uint8_t kHasUp = 16;    // upstream halo present
constexpr uint8_t kHasDn = 32;    // downstream halo present
constexpr uint8_t kRingSeg = 128; // a segment of the periodic link run as a row tile

// One tile = cells [a, a+w) of all lanes of one link.  Lane l of the tile
// is a "row" of Wp = roundup(w, 4) cells: codes at code[off + l*Wp + i],
// and the vids of the row's vehicles, in cell order, at vid[off + l*Wp + j]
// (j < number of vehicles in the row).  32 bytes.
struct TileDesc {
  int64_t off;
  int32_t link;
  int32_t a;
  int32_t lane_gid;  // global id of lane 0 of the link
  int32_t strip;     // first strip slot of this tile (one per lane) or -1
  int32_t n;         // cells of the link
  uint16_t w;
  uint8_t L;
  uint8_t flags;
};
static_assert(sizeof(TileDesc) == 32, "TileDesc must be 32 bytes");

// 5-cell strips next to a tile boundary: written by the
// tile every time it writes its state; read as halo by its neighbours (or,
// across domains, copied into a mirror slot by the exchange).
struct Strip {
  uint8_t head_code[8];
  uint8_t tail_code[8];
  int32_t head_vid[8];
  int32_t tail_vid[8];
  int64_t tail_pos[8];  // route position (VehPos::p) of the tail vehicles
};

// where a vehicle is on its route: p = absolute index of its current link
// in the route arrays (route_off[vid] + cursor), e = route_off[vid + 1]
struct VehPos {
  int64_t p, e;
};

// smem workspace of one warp for a tile with L lanes and row stride S
struct WarpLayout {
  int NC, NW;
  int o_cin, o_cout, o_bin, o_bout, o_vout, o_vpos, o_lf, bytes;
};

__host__ __device__ inline int row_pitch(int w) { return (w + 3) & ~3; }

// smem row stride of a tile in the general (warp-per-tile) kernels
__host__ __device__ inline int tile_stride(int w, uint8_t flags) {
  return (flags & kHalo) ? (((w + 15) & ~15) + 2 * kHaloPad) : row_pitch(w);
}

// global cells occupied by a tile (16-cell aligned)
__host__ __device__ inline int64_t tile_cells_padded(int w, int L) {
  return ((int64_t)row_pitch(w) * L + 15) & ~(int64_t)15;
}

// ---------------------------------------------------------------- row mode
// Fast path for whole links of <= kRowMaxCells cells: one
// thread per lane-row ("row"), the lanes of a link on consecutive threads
// of one warp, 32 row slots per group (one warp).  A row's state is six
// bit-planes of kRowWords 32-bit words each -- occupancy O, velocity bits
// V0..V2 and the vehicle's allowed-lane class A0/A1 (0 all lanes, 1 curb
// lane, 2 median lane; reading R7) for its current link -- bit x of word
// x >> 5 being cell x.  Planes are stored group-interleaved so that every
// warp access is one contiguous 128-byte line:
//   planes[group_plane_base(g) + (p * kRowWords + i) * 32 + slot].
// The vehicles of a group are listed in one contiguous block at vid[voff]
// (capacity: the group's cells): row after row in slot order, each row's
// vehicles in cell order, as entries vid | slot << 27 (the out-slot travels
// with the vehicle in its list entry; list order is preserved by the
// move).  A row's list starts at the prefix sum of the vehicle counts of
// the rows before it (popcounts of their occupancy planes), so the block
// is read and written with dense, coalesced warp accesses.
#ifndef TS_ROWS_TPB
#define TS_ROWS_TPB 128  // k_rows threads per block (one warp per group)
#endif
constexpr int kSlotShift = 27;
// entrant record (node kernel -> move kernels): vid | code << 32 | y << 40 |
// ((t + 1) mod 2^21) << 43; all ones = none (reset when consumed)
constexpr uint32_t kNoEntrant = 0xFFFFFFFFu;
constexpr uint32_t kVidMask = (1u << kSlotShift) - 1u;
constexpr int kRowWords = 4;
constexpr int kRowMaxCells = 32 * kRowWords;
constexpr int kStatePlanes = 6;

__host__ __device__ inline size_t group_plane_base(int64_t g) {
  return (size_t)g * kStatePlanes * kRowWords * 32;
}

struct RowDesc {
  int32_t nli;   // node-lane index of the row (tail record and node grant)
  int32_t link;
  int32_t lg;    // node-out-lane index (head occupancy and entrant record)
  uint8_t w;     // cells (0 = empty slot)
  uint8_t l, L;  // lane, lanes of the link
  uint8_t vk;    // vmax of the link
};
static_assert(sizeof(RowDesc) == 16, "RowDesc must be 16 bytes");
// k_rows reads w, l, L, vk as one little-endian word (bytes 12..15)
static_assert(offsetof(RowDesc, w) == 12 && offsetof(RowDesc, vk) == 15, "RowDesc packed word");

// shared memory of one k_rows warp (4-byte words): the group's vid block in
// and out (cap entries each; the out area first serves as the list of the
// vehicles that draw), then an aux area: the brake bits of the 32 rows
// during the draws, the masks and list offsets of the rows the lane change
// touched during the list rebuild
constexpr int kRowsAuxWords = 4 * 32 * kRowWords + 5 * 32 + 4 + 64;
#ifndef TS_ROWS_FIRST_STATIC
#define TS_ROWS_FIRST_STATIC 1  // k_rows: a warp's first group is its index (no atomic)
#endif
// per warp: vid block in, vid block out (cap entries each), the aux area
__host__ __device__ inline int rows_stage_words(int cap) {
  return 2 * cap + kRowsAuxWords;  // cap % 4 == 0: 16-byte aligned
}

// Warp-cooperative node kernel: the incoming lanes of every node, in the
// priority order (major class first, then link id, then lane; R9), packed
// into chunks of 32 entries that never split a node (unused entries have
// lane_gid = -1).  The position of a lane in this array is its node-lane
// index (nli): the tail record (written with S1) and the node grant `ext`
// of the lane are stored at that index, so the node kernel reads and
// writes them coalesced.
struct __align__(16) NodeLane {
  int32_t lane_gid;
  int32_t out_base;  // first NodeOut entry of the node (its out-slots)
  uint32_t tt;       // turn types of the link's out-slots (2 bits each)
  uint8_t lane, major, vk;
  uint8_t first;     // the node's first lane within its chunk (node key)
};
static_assert(sizeof(NodeLane) == 16, "NodeLane must be 16 bytes");

// an outgoing link of a node, by out-slot: what a winner needs to enter it
struct NodeOut {
  int32_t lgid;  // node-out-lane index of its lane 0 (head occupancy, entrant record)
  int16_t L;     // lanes
  int16_t n;     // cells
  int32_t row0;  // row slot of its lane 0 in the row kernel (lanes consecutive), or -1
};

__host__ __device__ inline WarpLayout warp_layout(int NCmax) {
  WarpLayout l;
  l.NC = (NCmax + 31) & ~31;
  l.NW = l.NC / 32 + 3;  // front pad word + data + 2 back pad words
  int o = 0;
  l.o_cin = o;
  o += l.NC;
  l.o_cout = o;
  o += l.NC;
  l.o_bin = o;
  o += 4 * l.NW;
  l.o_bout = o;
  o += 4 * l.NW;
  o = (o + 15) & ~15;
  l.o_vout = o;
  o += 4 * l.NC;
  l.o_vpos = o;  // vpos[NC], dpos[NC], vrow[NC] (uint16)
  o += 6 * l.NC;
  o = (o + 15) & ~15;
  l.o_lf = o;  // first rank of each lane
  o += 4 * 8;
  l.bytes = (o + 127) & ~127;
  return l;
}

// stats slot layout (uint64 each)
enum { ST_HASH = 0, ST_ACTIVE, ST_ARR, ST_INJ, ST_LC, ST_CROSS, ST_SUMV, ST_N };

// kernel modes
constexpr int kModeMove = 1;    // velocity update + move (H4/H5)
constexpr int kModeInject = 2;  // injection (H6)
constexpr int kModeLC = 4;      // lane change on the output state (H1)
constexpr int kModeHash = 8;    // accumulate state hash
constexpr int kModeWork = 16;   // per-link work counters
constexpr int kModeHalo = 32;   // ring segment rows: the lane change reads the neighbour segments

struct StepParams {
  const TileDesc *tiles;
  int32_t ntiles;
  int32_t t;  // step t: S1(t) -> S(t+1); k_lc: S(t) -> S1(t)
  const int32_t *tdev;  // CUDA-graph replay: t = *tdev + t (NULL: t as is)
  int32_t mode;
  int32_t D;
  uint32_t Dmul;  // ceil(2^32 / D): floor(x / D) = umulhi(x, Dmul) for x < 2^32 / D
  uint32_t k0, k1;
  uint32_t rk[20];  // Philox round keys (k0 + r W0, k1 + r W1), r = 0..9
  uint64_t p32;
  WarpLayout lay;
  // state (in / out buffers)
  const uint8_t *code_in;
  uint8_t *code_out;
  const int32_t *vid_in;
  int32_t *vid_out;
  const Strip *strip_in;
  Strip *strip_out;
  const int32_t *halo_up;  // per strip slot of lane 0: strip of upstream neighbour
  const int32_t *halo_dn;
  // network
  const uint8_t *vmax_link;
  const uint32_t *tt_link;  // 2 bits per out-slot: 0 T, 1 L, 2 R
  const int32_t *out_pos;   // slot of each link at its from-node
  // vehicles
  const uint8_t *rslot;  // per route entry j >= 1: out-slot of link R[j] at its from-node
  VehPos *vpos;
  const int32_t *dep;
  const int32_t *entry;
  int32_t *inj_time;
  int32_t *arr_time;
  const int32_t *pend_off;   // per link
  const int32_t *pend_list;  // vids in (departure, vid) order
  int32_t *pend_head;
  // node interface
  const int32_t *nli;  // node-lane index of every global lane id
  const int32_t *nlo;  // node-out-lane index of every global lane id
  uint64_t *tail_rec;  // per node-lane index, written with S1
  uint8_t *head_occ;   // per node-out-lane index, written with S1
  const uint8_t *ext;  // per node-lane index, from k_node
  uint64_t *entr;  // per node-out-lane index (cleared when consumed)
  // the same two node outputs for the row-kernel lanes by ROW SLOT, so the
  // row kernel loads them contiguously without its row descriptors first;
  // ext_row is kGmax for a lane whose front vehicle is on its final link
  // (the open end, R12), and a crossing's entrant record of a row-kernel
  // lane is written here only (entr holds those of general-tile lanes)
  const uint8_t *ext_row;
  uint64_t *entr_row;  // (cleared when consumed)
  // outputs
  unsigned long long *stats;  // [kHist][ST_N]
  unsigned long long *link_work;
};

struct NodeParams {
  int32_t nnodes;            // nodes of this domain
  const int32_t *node_ids;   // their ids (NULL: 0..nnodes-1)
  int32_t t;
  const int32_t *tdev;       // CUDA-graph replay: t = *tdev + t (NULL: t as is)
  int32_t G;
  uint32_t k0, k1;
  uint64_t p32;
  const int32_t *in_off, *in_list, *out_off, *out_list;
  const int32_t *link_ncell, *link_lanes, *link_lgid, *link_cls;
  const uint8_t *vmax_link;
  const uint32_t *tt_link;
  const int32_t *out_pos;
  const uint8_t *rslot;
  VehPos *vpos;
  const NodeOut *nodeout;  // [out_off[node] + slot]
  const uint32_t *node_sig;  // per node, phase-0 signal word (phase 1 derived); NULL = none
  const uint64_t *tail_rec;  // by node-lane index (k_node: identity)
  const uint8_t *head_occ;
  uint8_t *ext;              // by node-lane index (k_node: identity)
  uint64_t *entr;
  uint8_t *ext_row;          // by row slot (row-kernel lanes): the grant again (kGmax: final link)
  uint64_t *entr_row;        // by row slot: the entrant record of a row-kernel lane
  const int32_t *lane_row;   // row slot of every global lane id, or -1 (k_node)
  unsigned long long *stats;
  // per-node work counters (load statistics), by node id;
  // NULL unless TS_FLAG_LINK_WORK: incoming lanes whose front vehicle is in
  // the interaction range, plus crossings
  unsigned long long *node_work;
};

// tail record of a lane in S1 (read by k_node):
//   bits 0-31 front vid, 32-39 front code, 40-42 d = n-1-x, 43 has-front
//   (front vehicle inside the last 5 cells), 44-48 occupancy of the last 5
//   cells (bit i = cell n-1-i)
// entrant record (written by k_node for the target lane):
//   bits 0-31 vid, 32-39 code, 40-42 landing cell, 43-63 stamp (t+1)

struct RowsParams {
  const RowDesc *rows;        // [ngroups * 32]
  // ring segment rows (kModeHalo): per row slot the slot of the next
  // segment's row in the same lane, and of the previous one | its width << 24;
  // the segment's first cell (for the state hash); NULL otherwise
  const int32_t *ring_next, *ring_prev, *row_a;
  const int32_t *gvoff;       // first entry of each group's vid block (multiple of 4)
  const uint32_t *planes_in;  // S1(t) (fused) or S(t)
  uint32_t *planes_out;
  const int32_t *vid_in;      // row vid lists
  int32_t *vid_out;
  int32_t *inj_scratch;       // [row slot * kRowMaxCells + cell]: entry of a vehicle injected there
  const int32_t *gcnt_in;     // vehicles of each group (input state)
  int32_t *gcnt_out;
  int32_t ngroups;
  int32_t cap;                // smem staging capacity (entries) of a group's vid block
  unsigned long long *gctr;   // work counter, monotonic across launches
  unsigned long long gbase;   // its value at the start of this launch
};

// signal word of an incoming lane (reading R23): 0 = unsignalized, else
// bit 31 | cycle (bits 0-9) | shift (10-19) | green length (20-29); the lane
// is green at time t iff (t + shift) mod cycle < green length
__host__ __device__ inline bool sig_green(uint32_t s, int t) {
  const int c = (int)(s & 1023u), sh = (int)((s >> 10) & 1023u), len = (int)((s >> 20) & 1023u);
  return (t + sh) % c < len;
}

struct NodeWarpParams {
  const uint32_t *sig;  // per lane (same order as lanes); NULL = no signals
  const NodeLane *lanes;  // [32 * nchunks]
  int32_t nchunks;
  const int32_t *nl_node;  // node id of every node-lane index (-1 for pads; node work only)
  const int32_t *nl_row;   // row slot of every node-lane index, or -1
};

void launch_lc(const StepParams &p, int blocks, int threads, int smem, void *stream);
// CUDA-graph clock: zero the stats slots of steps *clock + 1 .. *clock + n
// (before the replayed steps), or advance *clock by n (after them)
void launch_clock(int32_t *clock, unsigned long long *stats, int n, bool advance, void *stream);
void launch_rows(const StepParams &p, const RowsParams &r, int blocks, int threads, int smem,
                 void *stream, bool pdl = false);
void launch_node_warp(const NodeParams &p, const NodeWarpParams &w, void *stream, bool pdl = false);
void launch_step(const StepParams &p, int blocks, int threads, int smem, void *stream);
void launch_node(const NodeParams &p, void *stream);
void launch_strip_copy(const Strip *src, const int32_t *sslot, Strip *dst, const int32_t *dslot,
                       int64_t n, void *stream);
// Direct strip delivery among the in-process domains of one device (one
// kernel per exchange instead of pack + copies + unpack): entry j moves
// strip sslot of handle sh to slot dslot of handle dh, between the handles'
// current strip buffers
constexpr int kDirectMax = 64;  // domains of one partition
struct DirectParams {
  const Strip *src[kDirectMax];
  Strip *dst[kDirectMax];
  const int4 *plan;  // (sh, sslot, dh, dslot) per strip
  int64_t n;
};
void launch_strip_direct(const DirectParams &p, void *stream);
void launch_hash(const StepParams &p, int blocks, int threads, int smem, void *stream,
                 unsigned long long *out);
void launch_rows_hash(const StepParams &p, const RowsParams &r, void *stream,
                      unsigned long long *out);

}  // namespace tsim
