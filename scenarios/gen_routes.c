/*
 * gen_routes.c -- seeded INPUT generator helper (no simulation arithmetic).
 *
 * Fills canonical x-then-y Manhattan routes on a rows x cols lattice for the
 * 256x256 grid workload (BASELINE.json configs[3]),
 * where the route table has billions of entries and numpy would need tens of
 * GB of temporaries.  Shared by the oracle and the CUDA path as plain input.
 *
 * Lattice link numbering (must match scenarios/__init__.py grid()):
 *   node id = r * cols + c  (x = c, y = r)
 *   east  (r, c) -> (r, c+1) : E(r, c) = r*(cols-1) + c
 *   west  (r, c+1) -> (r, c) : W(r, c) = H + r*(cols-1) + c,   H = rows*(cols-1)
 *   north (r, c) -> (r+1, c) : N(r, c) = 2H + r*cols + c
 *   south (r+1, c) -> (r, c) : S(r, c) = 2H + V + r*cols + c,  V = (rows-1)*cols
 */
#include <stdint.h>

static int64_t head_node(int64_t k, int64_t rows, int64_t cols) {
  int64_t H = rows * (cols - 1), V = (rows - 1) * cols;
  if (k < H) return (k / (cols - 1)) * cols + (k % (cols - 1)) + 1;
  k -= H;
  if (k < H) return (k / (cols - 1)) * cols + (k % (cols - 1));
  k -= H;
  if (k < V) return (k / cols + 1) * cols + (k % cols);
  k -= V;
  return (k / cols) * cols + (k % cols);
}

/* route lengths: 1 + |dx| + |dy| from the head node of the first link */
void manhattan_lengths(int64_t nv, const int32_t *first, const int32_t *dest,
                       int64_t rows, int64_t cols, int64_t *len_out) {
  for (int64_t i = 0; i < nv; i++) {
    int64_t h = head_node(first[i], rows, cols);
    int64_t hr = h / cols, hc = h % cols, dr = dest[i] / cols, dc = dest[i] % cols;
    int64_t dx = dc > hc ? dc - hc : hc - dc, dy = dr > hr ? dr - hr : hr - dr;
    len_out[i] = 1 + dx + dy;
  }
}

/* routes: first link, then x steps towards the destination column, then y */
void manhattan_fill(int64_t nv, const int32_t *first, const int32_t *dest,
                    int64_t rows, int64_t cols, const int64_t *off,
                    int32_t *route) {
  int64_t H = rows * (cols - 1), V = (rows - 1) * cols;
  for (int64_t i = 0; i < nv; i++) {
    int64_t j = off[i];
    route[j++] = first[i];
    int64_t h = head_node(first[i], rows, cols);
    int64_t r = h / cols, c = h % cols, dr = dest[i] / cols, dc = dest[i] % cols;
    while (c < dc) { route[j++] = (int32_t)(r * (cols - 1) + c); c++; }
    while (c > dc) { route[j++] = (int32_t)(H + r * (cols - 1) + c - 1); c--; }
    while (r < dr) { route[j++] = (int32_t)(2 * H + r * cols + c); r++; }
    while (r > dr) { route[j++] = (int32_t)(2 * H + V + (r - 1) * cols + c); r--; }
  }
}
