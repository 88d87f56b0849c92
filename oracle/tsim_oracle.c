/*
 * tsim_oracle.c -- TEST INFRASTRUCTURE ONLY (see tsim_oracle.h).
 *
 * A plain, slow, single-threaded CPU implementation of one TRANSIMS
 * cellular-automaton time step as PAPER.md defines it, under the readings
 * R1-R22 listed in DESIGN.md §3.  Written for a reader who
 * checks it against the paper line by line: no blocking, no fusion, no
 * bit tricks.  The state is a vid per lane-cell (EMPTY = -1) plus per-vehicle
 * records; every sub-step reads a snapshot and writes a fresh array.
 *
 * Paper passages followed:
 *   cells / hopping / car following (i)-(iii) ........ PAPER.md:320-335 (§3)
 *   lane changing as a sideways sub-step ............... PAPER.md:337-349 (§3)
 *   signals / unprotected turns (gap acceptance) ....... PAPER.md:351-358 (§3)
 *   parking entry / exit ............................... PAPER.md:428-432 (§4)
 *   interaction range 5 cells .......................... PAPER.md:390-395 (§4)
 *   split links, update sequence, boundary exchange .... PAPER.md:396-427 (§4)
 *
 * The pseudo-random slowdown uses Philox4x32-10 (Salmon et al., SC'11) with
 * the round constants of the curand implementation (reading R3); it is
 * written out here from the algorithm's definition and pinned in
 * tests/test_oracle_philox.py against the CUDA toolkit's host code path.
 */
#include "tsim_oracle.h"

#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define EMPTY (-1)
#define POISON (-2) /* cell not visible to a domain (emulation mode) */
#define GMAX 5      /* interaction range; reading R2 */
#define NOT_HELD (-1)

enum { TURN_T = 0, TURN_L = 1, TURN_R = 2 };

/* one domain's knowledge of the world; single-domain mode uses one view */
typedef struct {
  int32_t *occ;   /* vid per lane-cell, EMPTY, or POISON (not visible) */
  int8_t *status; /* per vehicle; NOT_HELD if another domain holds it */
  int32_t *vel, *vlink, *vlane, *vcell, *cur, *tarr;
} view;

typedef struct { /* one cut of a link between two domains */
  int32_t k, c, up, dn;
} cut_t;

struct orc {
  char err[512];
  double p;
  uint64_t p32;
  uint32_t key[2];
  int32_t G, D;
  /* network */
  int32_t nn, nl, periodic;
  int64_t *nx, *ny;
  int32_t *from, *to, *lanes, *vmax, *cls, *ncell;
  int64_t *base;  /* index of cell (k, 0, 0) */
  int64_t *lbase; /* global lane id of (k, 0) */
  int64_t ncells, nlanes;
  int32_t *in_off, *in_list; /* incoming links per node, ascending id */
  int32_t *sig_g0, *sig_g1, *sig_off; /* fixed-time signal per node (g0 = 0: none) */
  /* vehicles */
  int32_t nv;
  int64_t *roff;
  int32_t *route, *dep, *entry;
  int32_t *pend_order; /* vids in (departure, vid) order */
  int64_t pend_head, npend;
  int have_net, have_veh, inited;
  /* state */
  view g;
  int32_t t;
  int64_t ctr[10];
  uint8_t *brake_mask;
  /* scratch */
  int32_t *S0;
  int32_t *ext; /* per lane id: entry space granted to the front vehicle */
  /* k-domain emulation */
  int32_t k;
  view *dom;
  int32_t *dom_of_node;
  int32_t *seg_off, *seg_start, *seg_owner; /* per link segment lists */
  cut_t *cuts;
  int32_t ncuts;
  int64_t *dstats;
  int64_t poison_reads;
};

static int fail(orc *o, int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(o->err, sizeof o->err, fmt, ap);
  va_end(ap);
  return code;
}

static void *xcalloc(size_t n, size_t s) {
  void *p = calloc(n ? n : 1, s);
  if (!p) {
    fprintf(stderr, "tsim_oracle: out of memory\n");
    abort();
  }
  return p;
}

static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* ---------------------------------------------------------------- Philox */
/* Philox4x32 round: two 32x32->64 products, the high words xor-ed with the
 * other counter words and the key (Salmon et al. 2011, Fig. 2). */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
  uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
  uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
  uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
  uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
  uint32_t r0 = hi1 ^ c[1] ^ k[0];
  uint32_t r1 = lo1;
  uint32_t r2 = hi0 ^ c[3] ^ k[1];
  uint32_t r3 = lo0;
  c[0] = r0;
  c[1] = r1;
  c[2] = r2;
  c[3] = r3;
}

void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2],
                      uint32_t out[4]) {
  uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
  uint32_t k[2] = {key[0], key[1]};
  for (int round = 0; round < 10; round++) {
    if (round > 0) { /* key schedule: Weyl sequence */
      k[0] += 0x9E3779B9u;
      k[1] += 0xBB67AE85u;
    }
    philox_round(c, k);
  }
  memcpy(out, c, sizeof c);
}

/* reading R3: brake iff word 0 of Philox(key=(seed lo, seed hi),
 * ctr=(t, vid, 0, 0)) < floor(p * 2^32). */
static int brake_draw(const orc *o, int32_t t, int32_t vid) {
  if (o->brake_mask) return o->brake_mask[vid] != 0;
  uint32_t c[4] = {(uint32_t)t, (uint32_t)vid, 0u, 0u}, out[4];
  or_philox4x32_10(c, o->key, out);
  return (uint64_t)out[0] < o->p32;
}

/* ------------------------------------------------------------------ hash */
static uint64_t fmix64(uint64_t z) {
  z ^= z >> 33;
  z *= 0xff51afd7ed558ccdULL;
  z ^= z >> 33;
  z *= 0xc4ceb9fe1a85ec53ULL;
  z ^= z >> 33;
  return z;
}

uint64_t or_mix(int32_t vid, int32_t link, int32_t lane, int32_t cell,
                int32_t v) {
  uint64_t a = (uint64_t)(uint32_t)vid | ((uint64_t)(uint32_t)link << 32);
  uint64_t b = (uint64_t)(uint32_t)cell | ((uint64_t)(uint32_t)lane << 32) |
               ((uint64_t)(uint32_t)v << 40);
  return fmix64(fmix64(a) + b * 0x9E3779B97F4A7C15ULL);
}

/* -------------------------------------------------------------- creation */
orc *or_create(double p_slow, uint64_t seed, int32_t gap_G, int32_t desp_D) {
  orc *o = (orc *)xcalloc(1, sizeof(orc));
  if (p_slow < 0.0) p_slow = 0.0;
  if (p_slow > 1.0) p_slow = 1.0;
  o->p = p_slow;
  /* floor(p * 2^32); the product by a power of two is exact in binary64 */
  o->p32 = (uint64_t)(p_slow * 4294967296.0);
  o->key[0] = (uint32_t)(seed & 0xffffffffu);
  o->key[1] = (uint32_t)(seed >> 32);
  o->G = gap_G;
  o->D = desp_D;
  o->periodic = -1;
  o->k = 1;
  return o;
}

static void free_view(view *v) {
  free(v->occ);
  free(v->status);
  free(v->vel);
  free(v->vlink);
  free(v->vlane);
  free(v->vcell);
  free(v->cur);
  free(v->tarr);
  memset(v, 0, sizeof *v);
}

static void free_domains(orc *o) {
  if (o->dom) {
    for (int d = 0; d < o->k; d++) free_view(&o->dom[d]);
    free(o->dom);
  }
  o->dom = NULL;
  free(o->dom_of_node);
  free(o->seg_off);
  free(o->seg_start);
  free(o->seg_owner);
  free(o->cuts);
  free(o->dstats);
  o->dom_of_node = NULL;
  o->seg_off = o->seg_start = o->seg_owner = NULL;
  o->cuts = NULL;
  o->dstats = NULL;
  o->ncuts = 0;
  o->k = 1;
}

void or_destroy(orc *o) {
  if (!o) return;
  free_domains(o);
  free(o->nx);
  free(o->ny);
  free(o->from);
  free(o->to);
  free(o->lanes);
  free(o->vmax);
  free(o->cls);
  free(o->ncell);
  free(o->base);
  free(o->lbase);
  free(o->in_off);
  free(o->in_list);
  free(o->sig_g0);
  free(o->sig_g1);
  free(o->sig_off);
  free(o->roff);
  free(o->route);
  free(o->dep);
  free(o->entry);
  free(o->pend_order);
  free_view(&o->g);
  free(o->S0);
  free(o->ext);
  free(o->brake_mask);
  free(o);
}

const char *or_last_error(const orc *o) { return o->err; }

/* --------------------------------------------------------------- network */
static int64_t cidx(const orc *o, int32_t k, int32_t l, int32_t x) {
  return o->base[k] + (int64_t)l * o->ncell[k] + x;
}

int or_load_network(orc *o, int32_t n_nodes, const int64_t *node_x_mm,
                    const int64_t *node_y_mm, int32_t n_links,
                    const int32_t *from, const int32_t *to,
                    const int64_t *length_mm, const int32_t *lanes,
                    const int32_t *vmax, const int32_t *prio_class,
                    int32_t periodic_link) {
  if (o->have_net) return fail(o, 2, "network already loaded");
  if (n_nodes < 1 || n_links < 1) return fail(o, 2, "empty network");
  if (periodic_link >= 0 && n_links != 1)
    return fail(o, 2, "a periodic link must be the only link");
  for (int32_t k = 0; k < n_links; k++) {
    if (from[k] < 0 || from[k] >= n_nodes || to[k] < 0 || to[k] >= n_nodes)
      return fail(o, 2, "link %d: dangling node reference", k);
    if (from[k] == to[k] && k != periodic_link)
      return fail(o, 2, "link %d: from == to", k);
    if (length_mm[k] <= 0) return fail(o, 2, "link %d: non-positive length", k);
    if (lanes[k] < 1 || lanes[k] > 8) return fail(o, 2, "link %d: lanes", k);
    if (vmax[k] < 1 || vmax[k] > GMAX) return fail(o, 2, "link %d: vmax", k);
  }
  o->nn = n_nodes;
  o->nl = n_links;
  o->periodic = periodic_link;
  o->nx = (int64_t *)xcalloc(n_nodes, sizeof(int64_t));
  o->ny = (int64_t *)xcalloc(n_nodes, sizeof(int64_t));
  memcpy(o->nx, node_x_mm, n_nodes * sizeof(int64_t));
  memcpy(o->ny, node_y_mm, n_nodes * sizeof(int64_t));
  o->from = (int32_t *)xcalloc(n_links, 4);
  o->to = (int32_t *)xcalloc(n_links, 4);
  o->lanes = (int32_t *)xcalloc(n_links, 4);
  o->vmax = (int32_t *)xcalloc(n_links, 4);
  o->cls = (int32_t *)xcalloc(n_links, 4);
  o->ncell = (int32_t *)xcalloc(n_links, 4);
  o->base = (int64_t *)xcalloc(n_links + 1, 8);
  o->lbase = (int64_t *)xcalloc(n_links + 1, 8);
  for (int32_t k = 0; k < n_links; k++) {
    o->from[k] = from[k];
    o->to[k] = to[k];
    o->lanes[k] = lanes[k];
    o->vmax[k] = vmax[k];
    o->cls[k] = prio_class[k];
    /* reading R1: cells = round-half-up(length / 7.5 m) in integer mm,
     * at least 1 ("we currently use 7.5 meters") */
    int64_t n = (length_mm[k] + 3750) / 7500;
    if (n < 1) n = 1;
    if (n > 100000000) return fail(o, 2, "link %d: too long", k);
    o->ncell[k] = (int32_t)n;
    /* reading R11: links are at least 10 cells, so each half of a split
     * link covers the 5-cell interaction range */
    if (n < 10) return fail(o, 2, "link %d: %lld cells < 10 (R11)", k, (long long)n);
    o->base[k + 1] = o->base[k] + n * lanes[k];
    o->lbase[k + 1] = o->lbase[k] + lanes[k];
  }
  o->ncells = o->base[n_links];
  o->nlanes = o->lbase[n_links];
  /* incoming links per node in ascending link id (used by the priority
   * order (class, link id, lane) of reading R9) */
  o->in_off = (int32_t *)xcalloc(n_nodes + 1, 4);
  o->in_list = (int32_t *)xcalloc(n_links, 4);
  for (int32_t k = 0; k < n_links; k++)
    if (k != periodic_link) o->in_off[to[k] + 1]++;
  for (int32_t i = 0; i < n_nodes; i++) o->in_off[i + 1] += o->in_off[i];
  int32_t *fill = (int32_t *)xcalloc(n_nodes, 4);
  for (int32_t k = 0; k < n_links; k++)
    if (k != periodic_link) o->in_list[o->in_off[to[k]] + fill[to[k]]++] = k;
  free(fill);
  o->g.occ = (int32_t *)xcalloc(o->ncells, 4);
  for (int64_t i = 0; i < o->ncells; i++) o->g.occ[i] = EMPTY;
  o->S0 = (int32_t *)xcalloc(o->ncells, 4);
  o->ext = (int32_t *)xcalloc(o->nlanes, 4);
  o->have_net = 1;
  return 0;
}

int32_t or_n_cells(const orc *o, int32_t link) {
  if (!o->have_net || link < 0 || link >= o->nl) return -1;
  return o->ncell[link];
}

int64_t or_total_lane_cells(const orc *o) { return o->ncells; }

/* reading R7: turn type from the integer direction vectors a (in-link) and
 * b (out-link): straight if |angle| <= 45 deg, else left / right by the sign
 * of the cross product; a U-turn counts as left. */
int32_t or_turn_type(const orc *o, int32_t k, int32_t k2) {
  int64_t ax = o->nx[o->to[k]] - o->nx[o->from[k]];
  int64_t ay = o->ny[o->to[k]] - o->ny[o->from[k]];
  int64_t bx = o->nx[o->to[k2]] - o->nx[o->from[k2]];
  int64_t by = o->ny[o->to[k2]] - o->ny[o->from[k2]];
  int64_t cross = ax * by - ay * bx;
  int64_t dot = ax * bx + ay * by;
  int64_t acr = cross < 0 ? -cross : cross;
  if (dot > 0 && acr <= dot) return TURN_T;
  if (cross > 0) return TURN_L;
  if (cross < 0) return TURN_R;
  return TURN_L; /* U-turn */
}

/* reading R8: lane entered on the next link */
static int32_t entry_lane(const orc *o, int32_t k, int32_t l, int32_t k2) {
  int32_t tt = or_turn_type(o, k, k2);
  if (tt == TURN_T) return imin(l, o->lanes[k2] - 1);
  if (tt == TURN_R) return 0;
  return o->lanes[k2] - 1;
}

/* -------------------------------------------------------------- vehicles */
static int alloc_view(orc *o, view *v, int poison) {
  v->occ = (int32_t *)xcalloc(o->ncells, 4);
  for (int64_t i = 0; i < o->ncells; i++) v->occ[i] = poison ? POISON : EMPTY;
  v->status = (int8_t *)xcalloc(o->nv, 1);
  v->vel = (int32_t *)xcalloc(o->nv, 4);
  v->vlink = (int32_t *)xcalloc(o->nv, 4);
  v->vlane = (int32_t *)xcalloc(o->nv, 4);
  v->vcell = (int32_t *)xcalloc(o->nv, 4);
  v->cur = (int32_t *)xcalloc(o->nv, 4);
  v->tarr = (int32_t *)xcalloc(o->nv, 4);
  for (int32_t i = 0; i < o->nv; i++) {
    v->status[i] = NOT_HELD;
    v->vlink[i] = v->vlane[i] = v->vcell[i] = v->tarr[i] = -1;
  }
  return 0;
}

int or_load_vehicles(orc *o, int32_t n, const int64_t *route_off,
                     const int32_t *route_links, const int32_t *depart,
                     const int32_t *entry_cell) {
  if (!o->have_net) return fail(o, 2, "load the network first");
  if (o->have_veh) return fail(o, 2, "vehicles already loaded");
  if (n < 0) return fail(o, 2, "negative vehicle count");
  if (route_off[0] != 0) return fail(o, 2, "route_off[0] != 0");
  for (int32_t i = 0; i < n; i++) {
    int64_t a = route_off[i], b = route_off[i + 1];
    if (b <= a) return fail(o, 2, "vehicle %d: empty route", i);
    for (int64_t j = a; j < b; j++) {
      int32_t k = route_links[j];
      if (k < 0 || k >= o->nl) return fail(o, 2, "vehicle %d: bad link", i);
      if (j > a && o->to[route_links[j - 1]] != o->from[k])
        return fail(o, 2, "vehicle %d: route links not consecutive", i);
    }
    int32_t k0 = route_links[a];
    if (entry_cell[i] < 0 || entry_cell[i] >= o->ncell[k0])
      return fail(o, 2, "vehicle %d: entry cell outside link", i);
  }
  o->nv = n;
  int64_t m = route_off[n];
  o->roff = (int64_t *)xcalloc(n + 1, 8);
  memcpy(o->roff, route_off, (n + 1) * 8);
  o->route = (int32_t *)xcalloc(m, 4);
  memcpy(o->route, route_links, m * 4);
  o->dep = (int32_t *)xcalloc(n, 4);
  o->entry = (int32_t *)xcalloc(n, 4);
  memcpy(o->dep, depart, n * 4);
  memcpy(o->entry, entry_cell, n * 4);
  free_view(&o->g);
  alloc_view(o, &o->g, 0);
  for (int32_t i = 0; i < n; i++) {
    o->g.status[i] = OR_PENDING;
    o->g.cur[i] = 0;
  }
  o->have_veh = 1;
  return 0;
}

int or_place_vehicles(orc *o, int32_t n, const int32_t *vid,
                      const int32_t *lane, const int32_t *cell,
                      const int32_t *v) {
  if (!o->have_veh) return fail(o, 2, "load vehicles first");
  if (o->inited) return fail(o, 2, "already initialised");
  for (int32_t i = 0; i < n; i++) {
    int32_t f = vid[i];
    if (f < 0 || f >= o->nv) return fail(o, 2, "placement %d: bad vid", i);
    if (o->g.status[f] != OR_PENDING)
      return fail(o, 2, "placement %d: vehicle placed twice", i);
    int32_t k = o->route[o->roff[f]];
    if (lane[i] < 0 || lane[i] >= o->lanes[k] || cell[i] < 0 ||
        cell[i] >= o->ncell[k])
      return fail(o, 2, "placement %d: cell outside link", i);
    if (v[i] < 0 || v[i] > o->vmax[k])
      return fail(o, 2, "placement %d: velocity", i);
    int64_t c = cidx(o, k, lane[i], cell[i]);
    if (o->g.occ[c] != EMPTY) return fail(o, 2, "placement %d: cell taken", i);
    o->g.occ[c] = f;
    o->g.status[f] = OR_ACTIVE;
    o->g.vel[f] = v[i];
    o->g.vlink[f] = k;
    o->g.vlane[f] = lane[i];
    o->g.vcell[f] = cell[i];
    o->g.cur[f] = 0;
  }
  return 0;
}

static int cmp_dep_vid_ctx_dep(const int32_t *dep, int32_t a, int32_t b) {
  if (dep[a] != dep[b]) return dep[a] < dep[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* merge sort by (departure, vid): plain and stable */
static void sort_pending(int32_t *a, int32_t n, const int32_t *dep) {
  if (n < 2) return;
  int32_t *tmp = (int32_t *)xcalloc(n, 4);
  for (int32_t w = 1; w < n; w *= 2) {
    for (int32_t lo = 0; lo < n; lo += 2 * w) {
      int32_t mid = imin(lo + w, n), hi = imin(lo + 2 * w, n);
      int32_t i = lo, j = mid, q = lo;
      while (i < mid && j < hi)
        tmp[q++] = cmp_dep_vid_ctx_dep(dep, a[i], a[j]) <= 0 ? a[i++] : a[j++];
      while (i < mid) tmp[q++] = a[i++];
      while (j < hi) tmp[q++] = a[j++];
    }
    memcpy(a, tmp, n * 4);
  }
  free(tmp);
}

static void inject(orc *o, view *V, int32_t tnext, int dom, int64_t *n_inj);

int or_init(orc *o, int32_t t0) {
  if (!o->have_veh) return fail(o, 2, "load vehicles first");
  if (o->inited) return fail(o, 2, "already initialised");
  int32_t np = 0;
  for (int32_t i = 0; i < o->nv; i++) np += o->g.status[i] == OR_PENDING;
  o->pend_order = (int32_t *)xcalloc(np, 4);
  np = 0;
  for (int32_t i = 0; i < o->nv; i++)
    if (o->g.status[i] == OR_PENDING) o->pend_order[np++] = i;
  sort_pending(o->pend_order, np, o->dep);
  o->pend_head = 0;
  o->npend = np;
  o->t = t0;
  /* O1 §Init step 3: injection for departure <= t0 ("t+1 := t0") */
  int64_t n_inj = 0;
  inject(o, &o->g, t0, -1, &n_inj);
  o->inited = 1;
  return 0;
}

/* --------------------------------------------------------- rule helpers */
static int32_t rd(orc *o, const int32_t *S, int64_t i) {
  int32_t s = S[i];
  if (s == POISON) {
    o->poison_reads++;
    return EMPTY;
  }
  return s;
}

/* reading R2: ahead = consecutive empty cells at x+1, x+2, ... in lane l,
 * capped at 5, stopping at the first occupied cell or the link end
 * (periodic link: wraps). */
static int32_t ahead(orc *o, const int32_t *S, int32_t k, int32_t l, int32_t x) {
  int32_t n = o->ncell[k], g = 0;
  for (int32_t j = 1; j <= GMAX; j++) {
    int32_t y = x + j;
    if (y > n - 1) {
      if (k == o->periodic) y -= n;
      else break;
    }
    if (rd(o, S, cidx(o, k, l, y)) != EMPTY) break;
    g++;
  }
  return g;
}

/* reading R2: behind = the same towards x-1, x-2, ...; positions before the
 * link start count as empty (periodic link: wraps). */
static int32_t behind(orc *o, const int32_t *S, int32_t k, int32_t l, int32_t x) {
  int32_t n = o->ncell[k], g = 0;
  for (int32_t j = 1; j <= GMAX; j++) {
    int32_t y = x - j;
    if (y < 0) {
      if (k == o->periodic) y += n;
      else {
        g++;
        continue;
      }
    }
    if (rd(o, S, cidx(o, k, l, y)) != EMPTY) break;
    g++;
  }
  return g;
}

static int is_final(const orc *o, const view *V, int32_t f) {
  return o->roff[f] + V->cur[f] == o->roff[f + 1] - 1;
}

/* reading R7: allowed lanes for the vehicle f on link k.
 * returns 0 = all lanes, 1 = {0} (right turn), 2 = {L-1} (left turn) */
static int allowed_set(const orc *o, const view *V, int32_t f, int32_t k) {
  if (k == o->periodic || is_final(o, V, f)) return 0;
  int32_t k2 = o->route[o->roff[f] + V->cur[f] + 1];
  int32_t tt = or_turn_type(o, k, k2);
  if (tt == TURN_T) return 0;
  if (tt == TURN_R) return 1;
  return 2;
}

static int in_allowed(int set, int32_t l, int32_t L) {
  if (set == 0) return 1;
  if (set == 1) return l == 0;
  return l == L - 1;
}

/* O1 §LC: decision of the vehicle f at (k, l, x) on the
 * snapshot S0.  Returns the new lane or -1. */
static int32_t lc_decide(orc *o, const view *V, const int32_t *S0, int32_t f,
                         int32_t k, int32_t l, int32_t x, int32_t dir) {
  int32_t L = o->lanes[k];
  int32_t l2 = l + dir;
  if (l2 < 0 || l2 >= L) return -1;
  if (rd(o, S0, cidx(o, k, l2, x)) != EMPTY) return -1;
  int32_t v = V->vel[f];
  int32_t Vk = o->vmax[k];
  int set = allowed_set(o, V, f, k);
  if (!in_allowed(set, l, L)) {
    /* turn-motivated ("needs to get into the correct lane"); only towards
     * the allowed lane */
    int toward = (set == 1 && dir < 0) || (set == 2 && dir > 0);
    if (!toward) return -1;
    int32_t d = o->ncell[k] - 1 - x;
    int32_t bf = imin(v + 1, Vk), bb = Vk;
    int32_t rf = bf, rb = bb;
    if (d < o->D) { /* reading R6: desperation, linear over the last D cells */
      rf = (bf * d) / o->D;
      rb = (bb * d) / o->D;
    }
    if (ahead(o, S0, k, l2, x) >= rf && behind(o, S0, k, l2, x) >= rb) return l2;
    return -1;
  }
  if (!in_allowed(set, l2, L)) return -1;
  /* speed-motivated ("the other lane is faster") + gap check; reading R5 */
  int32_t gcur = ahead(o, S0, k, l, x);
  if (gcur < v + 1 && ahead(o, S0, k, l2, x) > gcur &&
      behind(o, S0, k, l2, x) >= Vk)
    return l2;
  return -1;
}

/* O1 §Move gap (PAPER.md:330-335 rule (ii)); ext = entry space granted by
 * the node step for the front vehicle. */
static int32_t gap_move(orc *o, const view *V, const int32_t *S, int32_t f,
                        int32_t k, int32_t l, int32_t x, int32_t ext) {
  int32_t n = o->ncell[k];
  for (int32_t j = 1; j <= GMAX; j++) {
    int32_t y = x + j;
    if (y > n - 1) {
      if (k == o->periodic) {
        y -= n;
      } else { /* no vehicle between x and the link end */
        if (is_final(o, V, f)) return GMAX; /* reading R12: open end */
        return imin(GMAX, (n - 1 - x) + ext);
      }
    }
    if (rd(o, S, cidx(o, k, l, y)) != EMPTY) return j - 1;
  }
  return GMAX;
}

/* Nagel-Schreckenberg velocity update (rules (i)-(iii), reading R15):
 * accelerate, limit to the gap, random slowdown. */
static int32_t new_velocity(const orc *o, int32_t t, int32_t f, int32_t v,
                            int32_t Vk, int32_t g) {
  int32_t v1 = imin(v + 1, Vk);
  int32_t v2 = imin(v1, g);
  int32_t v3 = v2;
  if (v2 > 0 && brake_draw(o, t, f)) v3 = v2 - 1;
  return v3;
}

/* entry space E at the start of (k2, l2): consecutive empty cells, capped
 * at min(5, n) (reading R10) */
static int32_t entry_space(orc *o, const int32_t *S, int32_t k2, int32_t l2) {
  int32_t lim = imin(GMAX, o->ncell[k2]), e = 0;
  while (e < lim && rd(o, S, cidx(o, k2, l2, e)) == EMPTY) e++;
  return e;
}

typedef struct {
  int32_t rank, k, l, f, k2, l2;
} cand_t;

static int cand_less(const cand_t *a, const cand_t *b) {
  if (a->rank != b->rank) return a->rank < b->rank;
  if (a->k != b->k) return a->k < b->k;
  return a->l < b->l;
}

/* O1 §Node for one node (readings R8-R10): sets o->ext
 * for the lanes of every incoming link of the node. */
/* Signalized node (reading R23): a fixed-time two-phase
 * plan; phase 0 = the incoming links of the node's maximal priority class,
 * phase 1 = the others.  With cycle c = g0 + g1 and tau = (t + offset) mod
 * c, phase 0 is green for tau < g0, phase 1 for tau >= g0.  A red approach
 * has the paper's "virtual vehicle of maximum velocity zero at the end of
 * the lane": its front vehicle gets no entry space (ext = 0); green
 * approaches need no gap acceptance. */
static int signal_green(const orc *o, int32_t node, int phase, int32_t t) {
  const int32_t g0 = o->sig_g0[node], c = g0 + o->sig_g1[node];
  const int32_t tau = (int32_t)((((int64_t)t + o->sig_off[node]) % c + c) % c);
  return phase == 0 ? tau < g0 : tau >= g0;
}

static void node_resolve(orc *o, const view *V, const int32_t *S, int32_t node, int32_t t) {
  int32_t a = o->in_off[node], b = o->in_off[node + 1];
  if (a == b) return;
  const int signalized = o->sig_g0 && o->sig_g0[node] + o->sig_g1[node] > 0;
  int32_t maxcls = o->cls[o->in_list[a]];
  for (int32_t i = a; i < b; i++) maxcls = imax(maxcls, o->cls[o->in_list[i]]);
  int32_t ncand = 0, cap = 0;
  for (int32_t i = a; i < b; i++) cap += o->lanes[o->in_list[i]];
  cand_t *cand = (cand_t *)xcalloc(cap, sizeof(cand_t));
  for (int32_t i = a; i < b; i++) {
    int32_t k = o->in_list[i], n = o->ncell[k];
    for (int32_t l = 0; l < o->lanes[k]; l++) {
      o->ext[o->lbase[k] + l] = 0;
      /* the front vehicle: largest x in (k, l).  Only a front vehicle
       * with d < min(v+1, V) <= 5 can be a candidate, so the search stops
       * after the last 5 cells (the interaction range). */
      int32_t x = n - 1, f = EMPTY;
      for (; x >= n - GMAX; x--) {
        f = rd(o, S, cidx(o, k, l, x));
        if (f != EMPTY) break;
      }
      if (f == EMPTY) continue;
      if (is_final(o, V, f)) continue;
      int32_t d = n - 1 - x;
      if (!(d < imin(V->vel[f] + 1, o->vmax[k]))) continue;
      /* red: the virtual blocker beyond the last cell */
      if (signalized && !signal_green(o, node, o->cls[k] == maxcls ? 0 : 1, t)) continue;
      cand_t c;
      c.rank = o->cls[k] == maxcls ? 0 : 1;
      c.k = k;
      c.l = l;
      c.f = f;
      c.k2 = o->route[o->roff[f] + V->cur[f] + 1];
      c.l2 = entry_lane(o, k, l, c.k2);
      cand[ncand++] = c;
    }
  }
  /* gap acceptance: the last G cells of every lane of every major
   * incoming link are empty */
  int majorfree = 1;
  for (int32_t i = a; i < b && majorfree && !signalized; i++) {
    int32_t j = o->in_list[i];
    if (o->cls[j] != maxcls) continue;
    for (int32_t l = 0; l < o->lanes[j] && majorfree; l++)
      for (int32_t y = o->ncell[j] - o->G; y <= o->ncell[j] - 1; y++)
        if (rd(o, S, cidx(o, j, l, y)) != EMPTY) {
          majorfree = 0;
          break;
        }
  }
  /* insertion sort by the priority key (class rank, link id, lane) */
  for (int32_t i = 1; i < ncand; i++) {
    cand_t c = cand[i];
    int32_t j = i - 1;
    while (j >= 0 && cand_less(&c, &cand[j])) {
      cand[j + 1] = cand[j];
      j--;
    }
    cand[j + 1] = c;
  }
  /* one winner per target lane (k2, l2) */
  int32_t *taken_k = (int32_t *)xcalloc(ncand, 4), *taken_l = (int32_t *)xcalloc(ncand, 4);
  int32_t ntaken = 0;
  for (int32_t i = 0; i < ncand; i++) {
    if (cand[i].rank == 1 && !majorfree) continue;
    int dup = 0;
    for (int32_t j = 0; j < ntaken; j++)
      if (taken_k[j] == cand[i].k2 && taken_l[j] == cand[i].l2) dup = 1;
    if (dup) continue;
    taken_k[ntaken] = cand[i].k2;
    taken_l[ntaken] = cand[i].l2;
    ntaken++;
    o->ext[o->lbase[cand[i].k] + cand[i].l] = entry_space(o, S, cand[i].k2, cand[i].l2);
  }
  free(taken_k);
  free(taken_l);
  free(cand);
}

static void place(orc *o, view *V, int32_t *S, int32_t f, int32_t k, int32_t l,
                  int32_t x, int32_t v) {
  int64_t c = cidx(o, k, l, x);
  if (S[c] != EMPTY) {
    o->ctr[3]++; /* collision: must never happen */
    return;
  }
  S[c] = f;
  V->vel[f] = v;
  V->vlink[f] = k;
  V->vlane[f] = l;
  V->vcell[f] = x;
}

/* ----------------------------------------------------- domain ownership */
/* owner domain of cell x of link k (single-domain mode: 0) */
static int32_t owner_of(const orc *o, int32_t k, int32_t x) {
  if (o->k == 1) return 0;
  int32_t s = o->seg_off[k];
  while (s + 1 < o->seg_off[k + 1] && o->seg_start[s + 1] <= x) s++;
  return o->seg_owner[s];
}

/* O1 §Inject (reading R13): pending vehicles with
 * departure <= tnext, in (departure, vid) order, each try (R[0], lane 0,
 * entry cell); the first to find it empty takes it with v = 0.
 * dom < 0: single domain; otherwise only vehicles that domain holds. */
static void inject(orc *o, view *V, int32_t tnext, int dom, int64_t *n_inj) {
  for (int64_t i = o->pend_head; i < o->npend; i++) {
    int32_t f = o->pend_order[i];
    if (o->dep[f] > tnext) break;
    if (V->status[f] != OR_PENDING) continue;
    int32_t k0 = o->route[o->roff[f]], e = o->entry[f];
    if (dom >= 0 && owner_of(o, k0, e) != dom) continue;
    int64_t c = cidx(o, k0, 0, e);
    if (rd(o, V->occ, c) != EMPTY) continue; /* retry next step */
    place(o, V, V->occ, f, k0, 0, e, 0);
    V->status[f] = OR_ACTIVE;
    V->cur[f] = 0;
    (*n_inj)++;
  }
  if (dom < 0) /* skip the prefix that is no longer pending */
    while (o->pend_head < o->npend &&
           V->status[o->pend_order[o->pend_head]] != OR_PENDING)
      o->pend_head++;
}

/* move one vehicle f of S1 at (k, l, x): returns 0 stays on link, 1 arrived,
 * 2 crossed.  The destination is written to S2 through place(). */
static int move_vehicle(orc *o, view *V, const int32_t *S1, int32_t *S2,
                        int32_t f, int32_t k, int32_t l, int32_t x,
                        int32_t ext, int32_t t, int dom, int ghost) {
  int32_t n = o->ncell[k];
  int32_t g = gap_move(o, V, S1, f, k, l, x, ext);
  int32_t v3 = new_velocity(o, t, f, V->vel[f], o->vmax[k], g);
  int32_t y = x + v3;
  if (k == o->periodic) y %= n;
  if (y <= n - 1) {
    /* hop along the lane */
    if (dom < 0 || owner_of(o, k, y) == dom) {
      place(o, V, S2, f, k, l, y, v3);
      if (ghost) V->status[f] = OR_ACTIVE; /* migrant arrives here */
    } else {
      V->status[f] = NOT_HELD; /* crossed the cut: the other domain has it */
      V->vlink[f] = V->vlane[f] = V->vcell[f] = -1;
    }
    return 0;
  }
  if (ghost) { /* cannot happen: segments are >= 5 cells (R11) */
    o->ctr[3]++;
    return 0;
  }
  if (is_final(o, V, f)) { /* exit to parking (R12) */
    V->status[f] = OR_ARRIVED;
    V->tarr[f] = t + 1;
    V->vel[f] = v3;
    V->vlink[f] = V->vlane[f] = V->vcell[f] = -1;
    return 1;
  }
  if (ext <= 0) o->ctr[3]++; /* only node winners can pass the link end */
  int32_t k2 = o->route[o->roff[f] + V->cur[f] + 1];
  int32_t l2 = entry_lane(o, k, l, k2);
  V->cur[f] += 1;
  place(o, V, S2, f, k2, l2, y - n, v3);
  return 2;
}

static void count_step_start(orc *o) {
  int64_t act = 0;
  for (int32_t f = 0; f < o->nv; f++) act += o->g.status[f] == OR_ACTIVE;
  o->ctr[8] += act;
  o->ctr[4] = o->ctr[5] = o->ctr[6] = o->ctr[7] = 0;
}

/* one time step t -> t+1 in a single domain (PAPER.md:412-427 without the
 * exchanges): lane change, node resolution, velocity update + move,
 * injection. */
static void step_single(orc *o) {
  view *V = &o->g;
  int32_t t = o->t;
  count_step_start(o);
  /* --- §LC on the snapshot S0 = S(t) --- */
  int32_t dir = (t % 2 == 0) ? +1 : -1; /* reading R4 */
  memcpy(o->S0, V->occ, o->ncells * sizeof(int32_t));
  for (int32_t k = 0; k < o->nl; k++)
    for (int32_t l = 0; l < o->lanes[k]; l++)
      for (int32_t x = 0; x < o->ncell[k]; x++) {
        int32_t f = o->S0[cidx(o, k, l, x)];
        if (f < 0) continue;
        int32_t l2 = lc_decide(o, V, o->S0, f, k, l, x, dir);
        if (l2 < 0) continue;
        /* apply: pure sideways move, v and cursor unchanged (R14) */
        if (V->occ[cidx(o, k, l2, x)] != EMPTY) o->ctr[3]++;
        V->occ[cidx(o, k, l, x)] = EMPTY;
        V->occ[cidx(o, k, l2, x)] = f;
        V->vlane[f] = l2;
        o->ctr[4]++;
      }
  /* --- §Node on S1 --- */
  for (int64_t i = 0; i < o->nlanes; i++) o->ext[i] = 0;
  for (int32_t node = 0; node < o->nn; node++) node_resolve(o, V, V->occ, node, t);
  /* --- §Move S1 -> S2 --- */
  int32_t *S1 = V->occ;
  int32_t *S2 = o->S0;
  for (int64_t i = 0; i < o->ncells; i++) S2[i] = EMPTY;
  for (int32_t k = 0; k < o->nl; k++)
    for (int32_t l = 0; l < o->lanes[k]; l++)
      for (int32_t x = 0; x < o->ncell[k]; x++) {
        int32_t f = S1[cidx(o, k, l, x)];
        if (f < 0) continue;
        int r = move_vehicle(o, V, S1, S2, f, k, l, x, o->ext[o->lbase[k] + l],
                             t, -1, 0);
        if (r == 1) o->ctr[7]++;
        if (r == 2) o->ctr[5]++;
      }
  o->S0 = S1;
  V->occ = S2;
  /* --- §Inject --- */
  inject(o, V, t + 1, -1, &o->ctr[6]);
  o->t = t + 1;
}

/* ------------------------------------------------ k-domain emulation */
typedef struct {
  int32_t k, l, x, vid, v, cur;
} rec_t;

/* positions of the 5-cell strips on each side of a cut (PAPER.md:404-411,
 * reading R17): up side sends [c-5, c), down side sends [c, c+5) */
static int32_t strip_pos(const orc *o, int32_t k, int32_t c, int32_t j,
                         int up) {
  int32_t n = o->ncell[k];
  int32_t x = up ? c - GMAX + j : c + j;
  if (x < 0) x += n; /* periodic link only */
  if (x >= n) x -= n;
  return x;
}

/* one boundary exchange: every domain sends, batched
 * into one message per neighbour domain, the five cells
 * of its own side next to every cut.  which == 1 (after lane change): the
 * up side also sends velocity and route cursor of its vehicles, which the
 * down side moves as ghosts; which == 2: occupancy only. */
static void exchange(orc *o, int which) {
  int32_t K = o->k;
  int64_t *cnt = (int64_t *)xcalloc((size_t)K * K, 8);
  for (int32_t i = 0; i < o->ncuts; i++) {
    cut_t c = o->cuts[i];
    cnt[c.up * K + c.dn] += (int64_t)o->lanes[c.k] * GMAX;
    cnt[c.dn * K + c.up] += (int64_t)o->lanes[c.k] * GMAX;
  }
  rec_t **msg = (rec_t **)xcalloc((size_t)K * K, sizeof(rec_t *));
  int64_t *fill = (int64_t *)xcalloc((size_t)K * K, 8);
  for (int64_t p = 0; p < (int64_t)K * K; p++)
    if (cnt[p]) msg[p] = (rec_t *)xcalloc(cnt[p], sizeof(rec_t));
  /* pack */
  for (int32_t i = 0; i < o->ncuts; i++) {
    cut_t c = o->cuts[i];
    for (int side = 0; side < 2; side++) {
      int up = side == 0;
      int32_t src = up ? c.up : c.dn, dst = up ? c.dn : c.up;
      view *S = &o->dom[src];
      for (int32_t l = 0; l < o->lanes[c.k]; l++)
        for (int32_t j = 0; j < GMAX; j++) {
          int32_t x = strip_pos(o, c.k, c.c, j, up);
          rec_t r;
          r.k = c.k;
          r.l = l;
          r.x = x;
          r.vid = rd(o, S->occ, cidx(o, c.k, l, x));
          r.v = r.cur = -1;
          if (which == 1 && up && r.vid >= 0) {
            r.v = S->vel[r.vid];
            r.cur = S->cur[r.vid];
          }
          msg[src * K + dst][fill[src * K + dst]++] = r;
        }
    }
  }
  /* deliver: one message per ordered neighbour pair */
  for (int32_t s = 0; s < K; s++)
    for (int32_t d = 0; d < K; d++) {
      int64_t p = (int64_t)s * K + d;
      if (!cnt[p]) continue;
      o->dstats[s * 4 + 1] += 1;
      o->dstats[s * 4 + 2] += cnt[p] * (int64_t)sizeof(rec_t);
      view *D = &o->dom[d];
      for (int64_t q = 0; q < cnt[p]; q++) {
        rec_t r = msg[p][q];
        D->occ[cidx(o, r.k, r.l, r.x)] = r.vid;
        if (r.vid >= 0 && r.cur >= 0 && D->status[r.vid] == NOT_HELD) {
          D->vel[r.vid] = r.v;
          D->cur[r.vid] = r.cur;
        }
      }
    }
  for (int64_t p = 0; p < (int64_t)K * K; p++) free(msg[p]);
  free(msg);
  free(fill);
  free(cnt);
}

/* copy the domains' owned state into the global read-only snapshot o->g */
static void gather(orc *o) {
  view *G = &o->g;
  for (int32_t k = 0; k < o->nl; k++)
    for (int32_t l = 0; l < o->lanes[k]; l++)
      for (int32_t x = 0; x < o->ncell[k]; x++) {
        int64_t c = cidx(o, k, l, x);
        int32_t s = o->dom[owner_of(o, k, x)].occ[c];
        if (s == POISON) {
          o->poison_reads++;
          s = EMPTY;
        }
        G->occ[c] = s;
      }
  for (int32_t f = 0; f < o->nv; f++) {
    int holders = 0;
    for (int32_t d = 0; d < o->k; d++) {
      view *D = &o->dom[d];
      if (D->status[f] == NOT_HELD) continue;
      holders++;
      G->status[f] = D->status[f];
      G->vel[f] = D->vel[f];
      G->vlink[f] = D->vlink[f];
      G->vlane[f] = D->vlane[f];
      G->vcell[f] = D->vcell[f];
      G->cur[f] = D->cur[f];
      G->tarr[f] = D->tarr[f];
    }
    if (holders != 1) o->ctr[3]++; /* a vehicle must live in one domain */
  }
}

/* distribute the global state o->g over the domains (also used to
 * re-partition mid-run, SURVEY G1 "rebalancing") */
static void scatter(orc *o) {
  view *G = &o->g;
  for (int32_t d = 0; d < o->k; d++) alloc_view(o, &o->dom[d], 1);
  for (int32_t k = 0; k < o->nl; k++)
    for (int32_t l = 0; l < o->lanes[k]; l++)
      for (int32_t x = 0; x < o->ncell[k]; x++) {
        int64_t c = cidx(o, k, l, x);
        o->dom[owner_of(o, k, x)].occ[c] = G->occ[c];
      }
  for (int32_t f = 0; f < o->nv; f++) {
    int32_t d = 0;
    if (G->status[f] == OR_ACTIVE) d = owner_of(o, G->vlink[f], G->vcell[f]);
    if (G->status[f] == OR_PENDING)
      d = owner_of(o, o->route[o->roff[f]], o->entry[f]);
    view *D = &o->dom[d];
    D->status[f] = G->status[f];
    D->vel[f] = G->vel[f];
    D->vlink[f] = G->vlink[f];
    D->vlane[f] = G->vlane[f];
    D->vcell[f] = G->vcell[f];
    D->cur[f] = G->cur[f];
    D->tarr[f] = G->tarr[f];
  }
  exchange(o, 2); /* initial mirrors */
}

int or_set_partition(orc *o, int32_t k, const int32_t *domain_of_node) {
  if (!o->inited) return fail(o, 2, "call or_init first");
  if (k < 1) return fail(o, 2, "k < 1");
  if (o->k > 1) free_domains(o); /* o->g is the gathered current state */
  if (k == 1) return 0;
  for (int32_t i = 0; i < o->nn; i++)
    if (domain_of_node[i] < 0 || domain_of_node[i] >= k)
      return fail(o, 2, "node %d: domain out of range", i);
  if (o->G > GMAX) return fail(o, 2, "G > 5 not supported in emulation");
  o->k = k;
  o->dom_of_node = (int32_t *)xcalloc(o->nn, 4);
  memcpy(o->dom_of_node, domain_of_node, o->nn * 4);
  /* segments: whole link, split at h = floor(n/2) (R16), or the periodic
   * link cut at k equally spaced points */
  o->seg_off = (int32_t *)xcalloc(o->nl + 1, 4);
  int32_t cap = o->nl * 2 + k;
  o->seg_start = (int32_t *)xcalloc(cap, 4);
  o->seg_owner = (int32_t *)xcalloc(cap, 4);
  o->cuts = (cut_t *)xcalloc(cap, sizeof(cut_t));
  int32_t ns = 0;
  for (int32_t e = 0; e < o->nl; e++) {
    o->seg_off[e] = ns;
    int32_t n = o->ncell[e];
    if (e == o->periodic) {
      if (n < GMAX * k) return fail(o, 2, "ring too short for k segments");
      for (int32_t i = 0; i < k; i++) {
        o->seg_start[ns] = (int32_t)(((int64_t)i * n) / k);
        o->seg_owner[ns++] = i;
      }
      for (int32_t i = 0; i < k; i++) {
        cut_t c = {e, o->seg_start[o->seg_off[e] + i], (i + k - 1) % k, i};
        o->cuts[o->ncuts++] = c;
      }
    } else if (domain_of_node[o->from[e]] == domain_of_node[o->to[e]]) {
      o->seg_start[ns] = 0;
      o->seg_owner[ns++] = domain_of_node[o->to[e]];
    } else {
      int32_t h = n / 2;
      o->seg_start[ns] = 0;
      o->seg_owner[ns++] = domain_of_node[o->from[e]];
      o->seg_start[ns] = h;
      o->seg_owner[ns++] = domain_of_node[o->to[e]];
      cut_t c = {e, h, domain_of_node[o->from[e]], domain_of_node[o->to[e]]};
      o->cuts[o->ncuts++] = c;
    }
  }
  o->seg_off[o->nl] = ns;
  o->dom = (view *)xcalloc(k, sizeof(view));
  o->dstats = (int64_t *)xcalloc((size_t)k * 4, 8);
  scatter(o);
  return 0;
}

/* one time step in k-domain emulation (PAPER.md:412-427 update sequence:
 * change lanes, exchange, compute speed and move, exchange). */
static void step_domains(orc *o) {
  int32_t t = o->t, K = o->k;
  count_step_start(o);
  for (int32_t i = 0; i < K * 4; i++) o->dstats[i] = 0;
  int32_t dir = (t % 2 == 0) ? +1 : -1;
  /* 1. change lanes, each domain on its own vehicles */
  for (int32_t d = 0; d < K; d++) {
    view *V = &o->dom[d];
    memcpy(o->S0, V->occ, o->ncells * sizeof(int32_t));
    for (int32_t k = 0; k < o->nl; k++)
      for (int32_t l = 0; l < o->lanes[k]; l++)
        for (int32_t x = 0; x < o->ncell[k]; x++) {
          if (owner_of(o, k, x) != d) continue;
          int32_t f = o->S0[cidx(o, k, l, x)];
          if (f < 0) continue;
          int32_t l2 = lc_decide(o, V, o->S0, f, k, l, x, dir);
          if (l2 < 0) continue;
          if (V->occ[cidx(o, k, l2, x)] != EMPTY) o->ctr[3]++;
          V->occ[cidx(o, k, l, x)] = EMPTY;
          V->occ[cidx(o, k, l2, x)] = f;
          V->vlane[f] = l2;
          o->ctr[4]++;
        }
  }
  /* 2. exchange boundary information */
  exchange(o, 1);
  /* 3. node resolution: nodes are never split */
  for (int64_t i = 0; i < o->nlanes; i++) o->ext[i] = 0;
  for (int32_t node = 0; node < o->nn; node++)
    node_resolve(o, &o->dom[o->dom_of_node[node]],
                 o->dom[o->dom_of_node[node]].occ, node, t);
  /* 4. compute speed and move: own vehicles plus the up-side strips
   *    received in exchange 1 ("ghosts") */
  int32_t *S2 = (int32_t *)xcalloc(o->ncells, 4);
  for (int32_t d = 0; d < K; d++) {
    view *V = &o->dom[d];
    int32_t *S1 = V->occ;
    for (int32_t k = 0; k < o->nl; k++)
      for (int32_t l = 0; l < o->lanes[k]; l++)
        for (int32_t x = 0; x < o->ncell[k]; x++)
          S2[cidx(o, k, l, x)] = owner_of(o, k, x) == d ? EMPTY : POISON;
    for (int32_t k = 0; k < o->nl; k++)
      for (int32_t l = 0; l < o->lanes[k]; l++)
        for (int32_t x = 0; x < o->ncell[k]; x++) {
          if (owner_of(o, k, x) != d) continue;
          int32_t f = S1[cidx(o, k, l, x)];
          if (f < 0) continue;
          int r = move_vehicle(o, V, S1, S2, f, k, l, x,
                               o->ext[o->lbase[k] + l], t, d, 0);
          if (r == 1) o->ctr[7]++;
          if (r == 2) o->ctr[5]++;
        }
    for (int32_t i = 0; i < o->ncuts; i++) {
      cut_t c = o->cuts[i];
      if (c.dn != d) continue;
      for (int32_t l = 0; l < o->lanes[c.k]; l++)
        for (int32_t j = 0; j < GMAX; j++) {
          int32_t x = strip_pos(o, c.k, c.c, j, 1);
          int32_t f = rd(o, S1, cidx(o, c.k, l, x));
          if (f < 0) continue;
          move_vehicle(o, V, S1, S2, f, c.k, l, x, 0, t, d, 1);
        }
    }
    memcpy(V->occ, S2, o->ncells * sizeof(int32_t));
  }
  free(S2);
  /* 5. parking: injection needs no further exchange */
  for (int32_t d = 0; d < K; d++) inject(o, &o->dom[d], t + 1, d, &o->ctr[6]);
  /* 6. exchange boundary information */
  exchange(o, 2);
  o->t = t + 1;
  gather(o);
  while (o->pend_head < o->npend &&
         o->g.status[o->pend_order[o->pend_head]] != OR_PENDING)
    o->pend_head++;
  for (int32_t d = 0; d < K; d++) {
    int64_t own = 0;
    for (int32_t f = 0; f < o->nv; f++) own += o->dom[d].status[f] == OR_ACTIVE;
    o->dstats[d * 4 + 0] = own;
  }
  o->dstats[3] = o->poison_reads;
}

int or_step(orc *o, int32_t n) {
  if (!o->inited) return fail(o, 2, "call or_init first");
  for (int32_t i = 0; i < n; i++) {
    if (o->k == 1) step_single(o);
    else step_domains(o);
  }
  if (o->brake_mask) { /* a brake override applies to one step only */
    free(o->brake_mask);
    o->brake_mask = NULL;
  }
  return 0;
}

int or_set_brake_override(orc *o, const uint8_t *mask) {
  free(o->brake_mask);
  o->brake_mask = NULL;
  if (mask) {
    o->brake_mask = (uint8_t *)xcalloc(o->nv, 1);
    memcpy(o->brake_mask, mask, o->nv);
  }
  return 0;
}

/* --------------------------------------------------------------- readers */
/* fixed-time signals (reading R23): node ids and their plans */
int or_set_signals(orc *o, int32_t n, const int32_t *node, const int32_t *green0,
                   const int32_t *green1, const int32_t *offset) {
  if (!o->have_net) return fail(o, 2, "load the network first");
  if (o->inited) return fail(o, 2, "already initialised");
  if (!o->sig_g0) {
    o->sig_g0 = (int32_t *)xcalloc(o->nn, 4);
    o->sig_g1 = (int32_t *)xcalloc(o->nn, 4);
    o->sig_off = (int32_t *)xcalloc(o->nn, 4);
  }
  for (int32_t i = 0; i < n; i++) {
    if (node[i] < 0 || node[i] >= o->nn) return fail(o, 2, "signal %d: bad node", i);
    if (green0[i] < 0 || green1[i] < 0 || green0[i] + green1[i] < 1 ||
        green0[i] + green1[i] > 1023 || offset[i] < 0)
      return fail(o, 2, "signal %d: bad plan", i);
    o->sig_g0[node[i]] = green0[i];
    o->sig_g1[node[i]] = green1[i];
    o->sig_off[node[i]] = offset[i];
  }
  return 0;
}

int32_t or_time(const orc *o) { return o->t; }

uint64_t or_state_hash(const orc *o) {
  uint64_t h = 0;
  const view *G = &o->g;
  for (int32_t f = 0; f < o->nv; f++)
    if (G->status[f] == OR_ACTIVE)
      h += or_mix(f, G->vlink[f], G->vlane[f], G->vcell[f], G->vel[f]);
  return h;
}

void or_counters(const orc *o, int64_t out[10]) {
  int64_t a = 0, p = 0, r = 0, sv = 0;
  for (int32_t f = 0; f < o->nv; f++) {
    int s = o->g.status[f];
    a += s == OR_ACTIVE;
    p += s == OR_PENDING;
    r += s == OR_ARRIVED;
    if (s == OR_ACTIVE) sv += o->g.vel[f];
  }
  for (int i = 0; i < 10; i++) out[i] = o->ctr[i];
  out[0] = a;
  out[1] = p;
  out[2] = r;
  out[9] = sv;
}

int or_read_vehicles(const orc *o, int8_t *status, int32_t *link,
                     int32_t *lane, int32_t *cell, int32_t *v, int32_t *cursor,
                     int32_t *t_arrive) {
  const view *G = &o->g;
  for (int32_t f = 0; f < o->nv; f++) {
    int act = G->status[f] == OR_ACTIVE;
    if (status) status[f] = G->status[f];
    if (link) link[f] = act ? G->vlink[f] : -1;
    if (lane) lane[f] = act ? G->vlane[f] : -1;
    if (cell) cell[f] = act ? G->vcell[f] : -1;
    if (v) v[f] = act ? G->vel[f] : -1;
    if (cursor) cursor[f] = G->status[f] == OR_PENDING ? -1 : G->cur[f];
    if (t_arrive) t_arrive[f] = G->status[f] == OR_ARRIVED ? G->tarr[f] : -1;
  }
  return 0;
}

int or_read_cells(const orc *o, int32_t link, int32_t *vid_out) {
  if (link < 0 || link >= o->nl) return 2;
  int64_t n = (int64_t)o->lanes[link] * o->ncell[link];
  memcpy(vid_out, o->g.occ + o->base[link], n * sizeof(int32_t));
  return 0;
}

int or_domain_stats(const orc *o, int64_t *out, int32_t cap) {
  if (o->k == 1 || !o->dstats) return 0;
  int32_t n = imin(cap, o->k * 4);
  for (int32_t i = 0; i < n; i++) out[i] = o->dstats[i];
  out[3] = o->poison_reads;
  return 0;
}
