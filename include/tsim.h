/*
 * tsim.h -- C-ABI of the B200-native TRANSIMS cellular-automaton time step
 * (Nagel & Rickert, "Parallel implementation of the TRANSIMS
 * micro-simulation", arxiv cs/0105004; §3-§4).
 *
 * One handle = one simulation (one domain of a partitioned network, or the
 * whole network).  The library copies every input array into its own host
 * and device memory; callers own all buffers they pass.  Outputs go into
 * caller buffers.  A handle is not thread-safe.  All results depend only on
 * (inputs, config, seed): not on the partition, the launch configuration or
 * the number of devices.
 *
 * Return codes: TS_OK = 0, TS_EINTERNAL = 1 (CUDA or internal
 * error), TS_EINVAL = 2 (invalid input).  ts_last_error() returns a
 * human-readable message for the last failing call.
 *
 * Readings R1-R22 of the paper are listed in DESIGN.md §3.
 */
#ifndef TSIM_H
#define TSIM_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TS_OK 0
#define TS_EINTERNAL 1
#define TS_EINVAL 2

/* vehicle status (ts_read_vehicles) */
#define TS_PENDING 0
#define TS_ACTIVE 1
#define TS_ARRIVED 2
#define TS_ABSENT 3 /* domain mode: the vehicle is reported by another domain */

/* config flags */
#define TS_FLAG_FUSED 1u       /* fuse lane change of step t+1 into the move
                                  kernel of step t (whole-link tiles only) */
#define TS_FLAG_HASH 2u        /* state hash of S(t+1) every step */
#define TS_FLAG_LINK_WORK 4u   /* per-link work counters (load feedback) */
#define TS_FLAG_GRAPH 8u       /* replay steps through a CUDA graph */
#define TS_FLAG_GENERAL 16u     /* force the general warp-per-tile kernels (testing) */
#define TS_FLAG_NODE_GENERAL 32u /* force the thread-per-node kernel (testing) */

typedef struct ts_sim ts_sim;

typedef struct {
  double p_slow;          /* random-slowdown probability, PAPER.md:334-335 (R3) */
  uint64_t seed;          /* Philox key = (seed & 0xffffffff, seed >> 32) (R3) */
  int32_t gap_accept_G;   /* unprotected-turn gap, cells (R9), <= 5 */
  int32_t desperation_D;  /* lane-change desperation distance, cells (R6), 1..4096 */
  uint32_t flags;         /* TS_FLAG_* */
  int32_t device;         /* CUDA device ordinal */
  int32_t tile_cells;     /* max cells per lane in one tile (0 = default) */
  int32_t group_cells;    /* max cells per warp in the row kernel (0 = default) */
} ts_config;

/* Create a simulation.  *out receives the handle (NULL on failure). */
int ts_create(const ts_config *cfg, ts_sim **out);
void ts_destroy(ts_sim *h);
/* message of the last failing call on h (or of ts_create when h is NULL) */
const char *ts_last_error(const ts_sim *h);

/* Road network: n_nodes planar nodes (integer mm
 * coordinates, used for the exact turn classification R7) and n_links
 * directed links with length in mm (cells = round-half-up(len/7.5 m), R1),
 * lanes (1..8), vmax in cells/s (1..5), priority class (R9).
 * periodic_link = id of the one periodic link of a ring network, or -1.
 * Errors (TS_EINVAL): dangling node, non-positive length, < 10 cells (R11),
 * node out-degree > 15, bad lanes/vmax. */
int ts_load_network(ts_sim *h, int32_t n_nodes, const int64_t *node_x_mm,
                    const int64_t *node_y_mm, int32_t n_links,
                    const int32_t *from, const int32_t *to,
                    const int64_t *length_mm, const int32_t *lanes,
                    const int32_t *vmax, const int32_t *prio_class,
                    int32_t periodic_link);

/* Vehicles vid = 0..n-1 (plans): route CSR route_off[n+1]
 * into route_links (consecutive links must share a node), departure second
 * and entry cell on route[0] (R13).  Host arrays, read
 * during the call only.  Validated in parallel on the host cores; a bad
 * record returns TS_EINVAL naming the first failing vehicle in input order
 * ("vehicle i: empty route | bad link | route links not consecutive |
 * entry cell outside link") and loads nothing. */
int ts_load_vehicles(ts_sim *h, int32_t n, const int64_t *route_off,
                     const int32_t *route_links, const int32_t *depart,
                     const int32_t *entry_cell);

/* Optional initial placement of active vehicles on their route[0]
 * (ring / dense starts): vid, lane, cell, velocity. */
int ts_place_vehicles(ts_sim *h, int32_t n, const int32_t *vid,
                      const int32_t *lane, const int32_t *cell,
                      const int32_t *v);

/* Placement on any link of the route (checkpoint restore, repartitioning):
 * vehicle vid[i] stands on link route[cursor[i]] (cursor NULL = 0) at
 * (lane, cell) with velocity v.  Vehicles neither placed nor marked arrived
 * are pending.  A batch is all or nothing: a bad record (bad vid, vehicle
 * placed twice, cursor outside the route, cell outside link, velocity)
 * returns TS_EINVAL naming the first failing index of the batch and places
 * none of it.  Two placements on one cell are found by ts_init ("placement
 * i: cell taken", i the later one in placement order). */
int ts_place_vehicles_at(ts_sim *h, int32_t n, const int32_t *vid, const int32_t *cursor,
                         const int32_t *lane, const int32_t *cell, const int32_t *v);
/* Vehicles that already arrived (restore): vid[i] left at t_arrive[i]. */
int ts_set_arrived(ts_sim *h, int32_t n, const int32_t *vid, const int32_t *t_arrive);

/* Domain decomposition (§4, :366-452).  This handle simulates
 * domain `me` of a k-way node partition domain_of_node[n_nodes] (e.g. from
 * ts_orb_partition).  Call after ts_load_network, before ts_init.  Nodes
 * are never split; a link with both end nodes in `me` is owned whole; a
 * link whose end nodes lie in different domains is split at h = floor(n/2)
 * (reading R16): cells [0, h) belong to the domain of its from-node,
 * [h, n) to the domain of its to-node.  Every handle of a partition gets
 * the same inputs (network, all vehicles, placement); each keeps only its
 * own cells.  k = 1 is the undivided network.  TS_EINVAL: k < 1, me out of
 * range, k > n_nodes, a ring network, a node's domain out of range.
 * Results do not depend on k or the partition. */
int ts_set_domain(ts_sim *h, int32_t k, const int32_t *domain_of_node, int32_t me);

/* Pure host: the exchange partners of domain `me` (ascending domain id) and
 * the number of strips of one message to / from each (one per lane of
 * every split link the two share); a message is strips x ts_strip_bytes()
 * bytes, the same in both directions.  cap bounds the outputs; *n_out
 * receives the partner count.  No device needed. */
int ts_domain_plan(int32_t n_nodes, int32_t n_links, const int32_t *from, const int32_t *to,
                   const int64_t *length_mm, const int32_t *lanes, int32_t k,
                   const int32_t *domain_of_node, int32_t me, int32_t cap, int32_t *nbr_dom,
                   int64_t *nbr_strips, int32_t *n_out);
int32_t ts_strip_bytes(void);

/* SPEC text formats (SPEC.md "External Interfaces"; load_network
 * SPEC.md:46-54).  Network file: line-oriented text, `#` comments, sections
 * NODES (`id x y`, metres), LINKS (`id from to length lanes vmax`, metres,
 * cells/s), TURNS (`node in_link out_link control [red_s green_s]`).  Ids
 * are arbitrary integers, mapped to indices in file order; the priority
 * class of a link is its lane count (reading R9); turn permissions are not
 * restricted (all turns allowed); a `signal` TURNS record gives its node a
 * fixed-time two-phase plan (reading R23): phase 0 green for green_s, the
 * other phase for red_s (the node's first such record counts).
 * ts_parse_network_text: pure host parser into caller arrays (NULL pointers
 * = count only): node coordinates in mm, links (from / to as node indices,
 * length in mm, lanes, vmax, class, file id), signals (node index, green,
 * red).  TS_EINVAL with "line N: ..." in errbuf (char[256]) on a parse
 * error, a dangling node reference or a non-positive length.
 * ts_load_network_text: parse + ts_load_network (+ ts_set_signals).
 * Plans file: `vehicle_id departure_s entry_cell link_1 ... link_n` per
 * line, link ids of the network file; vids are the line order.
 * ts_parse_plans_text: pure host parser (route_off[n_veh + 1], route links
 * as indices); ts_load_plans_text: parse + ts_load_vehicles. */
int ts_parse_network_text(const char *text, size_t len, int32_t *n_nodes, int32_t *n_links,
                          int32_t *n_sig, int64_t *node_x_mm, int64_t *node_y_mm, int32_t *from,
                          int32_t *to, int64_t *length_mm, int32_t *lanes, int32_t *vmax,
                          int32_t *prio_class, int32_t *link_id, int32_t *sig_node,
                          int32_t *sig_green, int32_t *sig_red, char *errbuf);
int ts_load_network_text(ts_sim *h, const char *text, size_t len);
int ts_parse_plans_text(const char *text, size_t len, int32_t n_links, const int32_t *link_id,
                        int32_t *n_veh, int64_t *n_entries, int64_t *route_off,
                        int32_t *route_links, int32_t *depart, int32_t *entry_cell,
                        int32_t *vehicle_id, char *errbuf);
int ts_load_plans_text(ts_sim *h, const char *text, size_t len);

/* Fixed-time two-phase signals (reading R23) at the given
 * nodes: phase 0 = the incoming links of the node's maximal priority class,
 * green for the first green0 seconds of every (green0 + green1)-second
 * cycle shifted by offset (tau = (t + offset) mod cycle < green0); phase 1
 * green for the rest.  A red approach has the paper's virtual vehicle of
 * maximum velocity zero beyond its last cell (no crossing); green
 * approaches need no gap acceptance.  green0 + green1 in [1, 1023],
 * offset >= 0.  Before ts_init.  TS_EINVAL: bad node or plan. */
int ts_set_signals(ts_sim *h, int32_t n, const int32_t *node, const int32_t *green0,
                   const int32_t *green1, const int32_t *offset);

/* Build the device layout, upload, and run the initial injection of
 * vehicles with departure <= t0 (clock starts at t0).  In domain mode with
 * partners the boundary strips of S(t0) are packed at the end: exchange
 * them (below), then call ts_step_phase(h, 2, 0).  The initial placement of
 * the row tiles is built on the device (TSIM_HOST_INIT=1: on the host); a
 * cell claimed twice is TS_EINVAL naming the first such placement in input
 * order.  The handle keeps the route upload's pinned staging (2 x 64 MB of
 * page-locked host memory) for ts_read_vehicles until ts_destroy. */
int ts_init(ts_sim *h, int32_t t0);
/* As ts_init without the initial injection: the placed / arrived /
 * pending vehicles ARE the state S(t) (restore at time t). */
int ts_resume(ts_sim *h, int32_t t);

/* Advance n_steps one-second steps.  Synchronous. */
int ts_step(ts_sim *h, int32_t n_steps);

/* Enqueue n_steps on the handle's stream without synchronising (for
 * device-side timing); ts_sync waits. */
int ts_step_async(ts_sim *h, int32_t n_steps);
int ts_sync(ts_sim *h);

/* One step in three phases, for domains that exchange boundary strips
 * (PAPER.md:412-427).  With S(t) and its mirrors in place:
 *   phase 0: lane change (H1); packs exchange #1 (post-lane-change strips)
 *   -- the caller moves every send segment to its partner's receive segment
 *   phase 1: unpacks #1; intersections, velocity update, move, injection
 *            (H3-H6); time becomes t+1; packs exchange #2.  more != 0: a
 *            further step follows (lets whole-link tiles fuse the next lane
 *            change into this move).
 *   -- exchange
 *   phase 2: unpacks #2.
 * Kernels are enqueued on the handle's stream (ts_stream) in order. */
int ts_step_phase(ts_sim *h, int32_t phase, int32_t more);

/* Exchange plan after ts_init: partner domains, strips per message and the
 * first strip of each partner's segment in the send / receive buffers. */
int ts_exchange_plan(const ts_sim *h, int32_t cap, int32_t *nbr_dom, int64_t *nbr_strips,
                     int64_t *nbr_off, int32_t *n_out);
/* Device pointers of the packed send and receive buffers (owned by h). */
int ts_exchange_buffers(ts_sim *h, void **send_dev, void **recv_dev);
/* The CUDA stream (cudaStream_t) all of h's work is enqueued on. */
void *ts_stream(const ts_sim *h);
/* In-process exchange among the k handles of one partition (any devices):
 * copies every send segment into its partner's receive segment, ordered by
 * events after the senders' packs and before the receivers' next work. */
int ts_exchange_local(ts_sim **hs, int32_t k);

/* n_steps whole steps of the k domains of one partition held by this
 * process (the k handles in any order; any devices), with the in-process
 * exchanges between them (lane change, exchange #1,
 * intersections + move + injection, exchange #2, per step), enqueued by the
 * library with no host round trip per phase.  With TS_FLAG_GRAPH on every
 * handle (one device), blocks of 15 steps replay one CUDA graph that holds
 * all k domains' streams and both exchanges of every step.  Synchronous.
 * The handles must be at the same time t with no step in progress; not with
 * a native communicator.  Each domain's busy time (ts_busy_time) covers its
 * phases (not the exchange waits), except inside replayed graphs.  Not
 * thread-safe (the captured graphs are kept per handle set). */
int ts_local_step(ts_sim **hs, int32_t k, int32_t n_steps);

/* current time t (state is S(t)) */
int32_t ts_time(const ts_sim *h);

/* Per-vehicle state, arrays of n_vehicles entries (NULL to skip): status
 * (TS_*), link, lane, cell, v (-1 unless active), route cursor (-1 while
 * pending), arrival time (-1 unless arrived).  Domain mode: vehicles on
 * another domain's cells read TS_ABSENT; a pending vehicle is reported by
 * the domain owning its entry cell; merge by taking, per vehicle, the
 * domain that reports it ACTIVE, else ARRIVED, else PENDING. */
/* (single-domain handles: gathered by vid on the device; copies of >= 64
 * MB go through the handle's pinned double buffer, TSIM_PAGEABLE_READ=1:
 * plain cudaMemcpy.  TS_EINTERNAL "corrupt state" if a vid is held twice or
 * an unfinished vehicle is missing.) */
int ts_read_vehicles(ts_sim *h, int8_t *status, int32_t *link, int32_t *lane,
                     int32_t *cell, int32_t *v, int32_t *cursor,
                     int32_t *t_arrive);

/* vid per lane-cell of one link, lane-major (lanes * cells entries, -1 =
 * empty), and the link's cell count. */
int ts_read_cells(ts_sim *h, int32_t link, int32_t *vid_out);
int32_t ts_link_cells(const ts_sim *h, int32_t link);

/* Diagnostics: raw device state of a link -- for each lane, Wp =
 * roundup(cells, 4) code bytes and the Wp-entry vid region of the lane
 * (the first k entries are the vids of its k vehicles, in cell order).
 * code_out / vid_out hold lanes * Wp entries; *pitch receives Wp.
 * Single-tile links only. */
int ts_read_raw(ts_sim *h, int32_t link, uint8_t *code_out, int32_t *vid_out,
                int32_t *pitch);

/* Debug build check (race / bounds detection without a sanitizer): a
 * library compiled with -DTS_CHECKED (paper_cs_0105004_b200/build.py
 * build_checked, never the benchmarked library) counts, per device, every
 * violation of the row and node kernels' state invariants -- one vehicle
 * per cell, v <= vmax, vid lists
 * consistent with the occupancy planes and ranked onto occupied cells,
 * nothing past a row end, a node crosser landing before the first occupied
 * cell of its target lane and only with a next link on its route.
 * out[0] = 1 for a checked build (0 otherwise: out[1..3] = 0,
 * 0xFFFFFFFF, 0), out[1] = OR of the violated invariants' bits
 * (csrc/tsim_rows.cu, csrc/tsim_kernels.cu), out[2] = the smallest row
 * group that violated a row-kernel one (0xFFFFFFFF if none),
 * out[3] = the number of violations.  reset != 0 zeroes the counters after
 * reading; reset = 2 also arms a self-test (every row group of every later
 * launch counts bit 128 until the next reset = 1) so a test can prove the
 * counters reach the host.  Synchronises the current device.  TS_EINVAL: out NULL;
 * TS_EINTERNAL: CUDA error.  Caller owns out (4 entries). */
int ts_debug_checks(uint32_t *out, int32_t reset);

/* Order-independent state hash of S(t). */
int ts_state_hash(ts_sim *h, uint64_t *out);

/* Per-step history for steps whose result time is in [t_from, t_from+n):
 * hash of S(t) (if TS_FLAG_HASH), active vehicles in S(t), arrivals,
 * injections, lane changes, crossings.  NULL skips an array.  Only the
 * last 4096 steps are kept. */
int ts_read_history(ts_sim *h, int32_t t_from, int32_t n, uint64_t *hash,
                    int64_t *active, int64_t *arrivals, int64_t *injections,
                    int64_t *lane_changes, int64_t *crossings);

/* Sum of the velocities of S(t) (cells moved in the step that produced
 * it) for t in [t_from, t_from + n): the flow q(t) = sumv(t) / lane-cells
 * of the fundamental diagram.  Same range rules as
 * ts_read_history. */
int ts_read_flow(ts_sim *h, int32_t t_from, int32_t n, int64_t *sumv);

/* Totals: [0] active [1] pending [2] arrived [3] vehicle-updates since
 * init [4] lane-cells [5] tiles [6] device bytes allocated
 * [7] algorithmic bytes per step at the current state. */
int ts_get_totals(ts_sim *h, int64_t out[8]);

/* Per-link accumulated work (vehicle-updates) when TS_FLAG_LINK_WORK is
 * set (PAPER.md:730-735 load statistics). link_work[n_links]. */
int ts_get_link_work(ts_sim *h, int64_t *link_work);

/* Load statistics (§7: "the execution time of each link
 * and each intersection"), accumulated since ts_init when TS_FLAG_LINK_WORK
 * is set (zeros otherwise): link_work[n_links] = vehicle updates on the
 * link's cells owned by this handle; node_work[n_nodes] = per step, the
 * incoming lanes of the node whose front vehicle is inside the interaction
 * range plus the node's crossings (nodes of this domain only).  Either
 * pointer may be NULL.  Synchronises the handle's stream. */
int ts_get_load(ts_sim *h, int64_t *link_work, int64_t *node_work);

/* Pure host, for the adaptive rebalancing: apportion one
 * domain's measured device time domain_ms over a window (ts_busy_time) to
 * its links and nodes in proportion to their work counts over the same
 * window (differences of ts_get_load; one vehicle update and one node unit
 * count alike).  ADDS into link_time[n_links] and node_time[n_nodes]
 * (node_work / node_time may be NULL), so the k domains of a partition
 * accumulate into one pair of arrays (across ranks: sum them).  A domain
 * without work adds nothing.  TS_EINVAL on negative counts or time. */
int ts_load_times(double domain_ms, int32_t n_links, const int64_t *link_work, int32_t n_nodes,
                  const int64_t *node_work, double *link_time, double *node_time);

/* Pure host: the next partition from measured times (
 * SPEC.md:373-379).  Node weight = node_time (NULL = 0) + half of the time
 * of every attached link, links without measured time keeping a floor of
 * 1e-3 x total time x their share of cells x lanes; then a k-way
 * partition, method 0 = ORB (ts_orb_partition), 1 = multilevel
 * (ts_multilevel_partition with imbalance and seed).  Outputs the node
 * weights (nullable, [n_nodes]) and domain_of_node_out[n_nodes].  The
 * caller migrates the state (read, ts_place_vehicles_at / ts_set_arrived
 * into handles of the new partition, ts_resume); results are unchanged,
 * only speed.  TS_EINVAL: bad network, k, method or a negative time. */
int ts_rebalance(int32_t n_nodes, const int64_t *node_x_mm, const int64_t *node_y_mm,
                 int32_t n_links, const int32_t *from, const int32_t *to, const int32_t *lanes,
                 const int64_t *length_mm, const double *link_time, const double *node_time,
                 int32_t k, int32_t method, double imbalance, uint64_t seed,
                 double *node_weight_out, int32_t *domain_of_node_out);

/* Orthogonal recursive bisection of the nodes (SPEC.md
 * :210-218): node weights (the load of the attached half-links; NULL =
 * uniform), k domains, output domain_of_node[n_nodes].  Vertical cut first;
 * the larger piece is cut next; non-power-of-two k splits proportionally.
 * Pure host function (no device needed). */
int ts_orb_partition(int32_t n_nodes, const int64_t *node_x_mm,
                     const int64_t *node_y_mm, const double *node_weight,
                     int32_t k, int32_t *domain_of_node);

/* ts_orb_partition of this handle's network (node weights: NULL = half of
 * cells x lanes of every attached link) followed by
 * ts_set_domain(h, k, partition, me); the partition is copied to
 * domain_of_node_out[n_nodes] (nullable).  Before ts_init. */
int ts_partition(ts_sim *h, int32_t k, const double *node_weight, int32_t me,
                 int32_t *domain_of_node_out);

/* Multilevel k-way partition of the node graph (the
 * METIS-style alternative to ORB): heavy-edge matching
 * coarsening (seeded), ORB of the coarsest graph, greedy boundary
 * refinement at every level keeping each domain's load <= (1 + imbalance)
 * x average.  Vertex weight = node_weight (NULL = 1), edge weight = lanes
 * of the links joining two nodes (the strips a cut there costs per
 * exchange).  Pure host function; deterministic for a seed. */
int ts_multilevel_partition(int32_t n_nodes, const int64_t *node_x_mm, const int64_t *node_y_mm,
                            int32_t n_links, const int32_t *from, const int32_t *to,
                            const int32_t *lanes, const double *node_weight, int32_t k,
                            double imbalance, uint64_t seed, int32_t *domain_of_node);

/* Native exchange transport for domain mode (G1, H2/H7; PAPER.md:404-427,
 * 897-900): NCCL point-to-point inside the library, so that ts_step(n) runs
 * whole steps (lane change, exchange #1, move, exchange #2) for a domain with
 * neighbours without a host round trip per exchange.  libnccl.so.2 is opened
 * at run time (the copy already loaded by the process, else the system's).
 * ts_nccl_unique_id: writes a 128-byte ncclUniqueId (one rank creates it, the
 * caller distributes it).  ts_nccl_init: after ts_init, join the
 * communicator of nranks = k ranks as rank = this handle's domain (one GPU
 * per rank).  ts_exchange: one exchange of the packed strips now (e.g. the
 * one after ts_init), enqueued on the handle's stream.  TS_EINTERNAL if NCCL
 * is missing or fails; TS_EINVAL for ranks that are not the domains. */
int ts_nccl_unique_id(void *id128);
int ts_nccl_init(ts_sim *h, const void *id128, int32_t nranks, int32_t rank);
int ts_exchange(ts_sim *h);

/* Device time (ms, CUDA events on the handle's stream) of all step work --
 * ts_step calls and ts_step_phase calls -- since the previous call; resets.
 * The measured per-domain step time of the adaptive rebalancing
 * (PAPER.md:730-735).  Synchronises the handle's stream. */
int ts_busy_time(ts_sim *h, double *ms);

/* Exchange timing of the last ts_step call of a domain with the native
 * transport: total ms of the timed exchanges (both exchanges of every 8th
 * step, CUDA events around the NCCL group on the handle's stream) and their
 * count; n = 0 otherwise. */
int ts_last_exchange_timing(ts_sim *h, double *ms, int64_t *n);

/* Kernel-level timing of the last ts_step call (CUDA events on the
 * handle's stream): total ms, and ms inside the dominant (move) kernel. */
int ts_last_timing(ts_sim *h, double *total_ms, double *move_ms,
                   int64_t *move_launches);

#ifdef __cplusplus
}
#endif
#endif
