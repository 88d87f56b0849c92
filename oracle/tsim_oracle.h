/*
 * tsim_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle of the TRANSIMS cellular-automaton
 * time step (Nagel & Rickert, arxiv cs/0105004, §3 lines 306-362 and
 * §4) under the readings R1-R22 of SURVEY.md §8(c), which are
 * restated in DESIGN.md §3.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or constant generator with the CUDA path
 * (paper_cs_0105004_b200/csrc).
 *
 * Conventions: every function returns 0 on success, 2 on invalid input,
 * 1 on an internal error; or_last_error() gives the message.  Arrays passed
 * in are copied, except where stated.
 */
#ifndef TSIM_ORACLE_H
#define TSIM_ORACLE_H
#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc orc;

/* vehicle status */
#define OR_PENDING 0
#define OR_ACTIVE 1
#define OR_ARRIVED 2

orc *or_create(double p_slow, uint64_t seed, int32_t gap_G, int32_t desp_D);
void or_destroy(orc *o);
const char *or_last_error(const orc *o);

/* network: node coordinates in integer mm; links with length in mm
 * (cells = floor((mm + 3750) / 7500), min 1, reading R1), lanes, vmax
 * (cells/s), priority class; periodic_link = id of the single periodic
 * link (ring) or -1. */
int or_load_network(orc *o, int32_t n_nodes, const int64_t *node_x_mm,
                    const int64_t *node_y_mm, int32_t n_links,
                    const int32_t *from, const int32_t *to,
                    const int64_t *length_mm, const int32_t *lanes,
                    const int32_t *vmax, const int32_t *prio_class,
                    int32_t periodic_link);

/* vehicles vid = 0..n-1: route CSR (route_off[n+1], route_links), departure
 * second and entry cell on route[0]. */
int or_load_vehicles(orc *o, int32_t n, const int64_t *route_off,
                     const int32_t *route_links, const int32_t *depart,
                     const int32_t *entry_cell);

/* initial placement of active vehicles (ring, dense starts) on route[0]. */
int or_place_vehicles(orc *o, int32_t n, const int32_t *vid,
                      const int32_t *lane, const int32_t *cell,
                      const int32_t *v);

/* finish initialisation: injection for departure <= t0 (O1 §Init step 3),
 * time starts at t0 (normally 0). */
/* fixed-time two-phase signals at the given nodes (reading R23): phase 0 =
 * incoming links of the node's maximal class, green for the first green0
 * seconds of each (green0 + green1)-second cycle shifted by offset; phase
 * 1 green for the rest.  green0 + green1 in [1, 1023].  Before or_init. */
int or_set_signals(orc *o, int32_t n, const int32_t *node, const int32_t *green0,
                   const int32_t *green1, const int32_t *offset);

int or_init(orc *o, int32_t t0);

/* advance n steps (single domain or k-domain emulation, see below). */
int or_step(orc *o, int32_t n);

int32_t or_time(const orc *o);
int32_t or_n_cells(const orc *o, int32_t link);
int64_t or_total_lane_cells(const orc *o);

/* order-independent state hash of S(t) */
uint64_t or_state_hash(const orc *o);

/* counters: [0]=active [1]=pending [2]=arrived [3]=collisions (must be 0)
 * [4]=lane changes last step [5]=node crossings last step
 * [6]=injections last step [7]=arrivals last step [8]=vehicle-updates
 * (sum over steps of active vehicles at step start)
 * [9]=sum of velocities in S(t) */
void or_counters(const orc *o, int64_t out[10]);

/* per-vehicle state: status, link, lane, cell, v, cursor, arrival time
 * (-1 where not applicable). Each array has n_veh entries; NULL skips. */
int or_read_vehicles(const orc *o, int8_t *status, int32_t *link,
                     int32_t *lane, int32_t *cell, int32_t *v, int32_t *cursor,
                     int32_t *t_arrive);

/* vid per lane-cell of one link, lane-major (L*n entries, -1 empty) */
int or_read_cells(const orc *o, int32_t link, int32_t *vid_out);

/* turn type of (in_link, out_link): 0=T 1=L 2=R (reading R7) */
int32_t or_turn_type(const orc *o, int32_t k, int32_t k2);

/* Philox4x32-10 (PAPER: random slowdown; reading R3) for pinning */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                      uint32_t out[4]);

/* State hash mixing function, exposed for tests. */
uint64_t or_mix(int32_t vid, int32_t link, int32_t lane, int32_t cell,
                int32_t v);

/* k-domain emulation (§4): node -> domain; network
 * links whose ends lie in different domains are split at h = n/2; the
 * periodic link is cut at k equally spaced points.  May be called at any
 * time after or_init; the current state is gathered and re-scattered.
 * k == 1 returns to single-domain mode. */
int or_set_partition(orc *o, int32_t k, const int32_t *domain_of_node);

/* per-domain counters of the last step (emulation mode):
 * [d*4+0]=owned vehicles [1]=messages sent [2]=bytes sent [3]=poison reads */
int or_domain_stats(const orc *o, int64_t *out, int32_t cap);

/* test hooks: override the brake decision of the next step with a mask
 * indexed by vid (1 = brake if v2 > 0); NULL restores Philox. */
int or_set_brake_override(orc *o, const uint8_t *mask);

#ifdef __cplusplus
}
#endif
#endif
