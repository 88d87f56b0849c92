// tsim_text.cpp -- the SPEC text formats of the network and plans files
// (SPEC.md "External Interfaces"; load_network SPEC.md:46-54): pure host
// parsers behind the C-ABI (include/tsim.h), no device needed.
//
// Network file: line-oriented, `#` starts a comment, sections
//   NODES  `id x y`                               (metres)
//   LINKS  `id from to length lanes vmax`         (metres, cells/s)
//   TURNS  `node in_link out_link control [red_s green_s]`
// Plans file: `vehicle_id departure_s entry_cell link_1 link_2 ... link_n`.
// Ids are arbitrary integers, mapped to dense indices in file order.
#include <algorithm>
#include <cerrno>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

constexpr int kOk = 0, kInval = 2;

struct Lines {
  const char *p, *end;
  int no = 0;
  // next non-empty line without its comment; false at the end
  bool next(std::string &out) {
    while (p < end) {
      const char *e = (const char *)memchr(p, '\n', (size_t)(end - p));
      if (!e) e = end;
      std::string ln(p, (size_t)(e - p));
      p = e < end ? e + 1 : end;
      no++;
      const size_t h = ln.find('#');
      if (h != std::string::npos) ln.resize(h);
      size_t a = ln.find_first_not_of(" \t\r");
      if (a == std::string::npos) continue;
      size_t b = ln.find_last_not_of(" \t\r");
      out = ln.substr(a, b - a + 1);
      return true;
    }
    return false;
  }
};

std::vector<std::string> fields(const std::string &s) {
  std::vector<std::string> f;
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && (s[i] == ' ' || s[i] == '\t')) i++;
    size_t j = i;
    while (j < s.size() && s[j] != ' ' && s[j] != '\t') j++;
    if (j > i) f.push_back(s.substr(i, j - i));
    i = j;
  }
  return f;
}

bool to_i64(const std::string &s, int64_t &v) {
  errno = 0;
  char *e = nullptr;
  const long long x = strtoll(s.c_str(), &e, 10);
  if (errno || !e || *e) return false;
  v = x;
  return true;
}

bool to_f64(const std::string &s, double &v) {
  errno = 0;
  char *e = nullptr;
  v = strtod(s.c_str(), &e);
  return !errno && e && !*e && std::isfinite(v);
}

int err(char *buf, const char *fmt, int line, const char *what) {
  if (buf) snprintf(buf, 256, fmt, line, what);
  return kInval;
}

struct Net {
  std::vector<int64_t> nx, ny, len;
  std::vector<int32_t> from, to, lanes, vmax, link_id;
  std::vector<int32_t> sig_node, sig_green, sig_red;
};

int parse_network(const char *text, size_t n, Net &net, char *ebuf) {
  Lines L{text, text + n};
  std::unordered_map<int64_t, int32_t> node_of, link_of;
  enum { NONE, NODES, LINKS, TURNS } sec = NONE;
  std::string ln;
  struct Turn {
    int line;
    int64_t node;
    std::string control;
    int64_t red, green;
  };
  std::vector<Turn> turns;
  std::vector<std::pair<int64_t, int64_t>> ends;  // raw node ids of each link
  std::vector<int> link_line;
  while (L.next(ln)) {
    if (ln == "NODES") { sec = NODES; continue; }
    if (ln == "LINKS") { sec = LINKS; continue; }
    if (ln == "TURNS") { sec = TURNS; continue; }
    const std::vector<std::string> f = fields(ln);
    if (sec == NODES) {
      int64_t id;
      double x, y;
      if (f.size() != 3 || !to_i64(f[0], id) || !to_f64(f[1], x) || !to_f64(f[2], y))
        return err(ebuf, "line %d: %s", L.no, "NODES record must be `id x y`");
      if (node_of.count(id)) return err(ebuf, "line %d: %s", L.no, "duplicate node id");
      node_of[id] = (int32_t)net.nx.size();
      net.nx.push_back((int64_t)llround(x * 1000.0));
      net.ny.push_back((int64_t)llround(y * 1000.0));
    } else if (sec == LINKS) {
      int64_t id, a, b, lanes, vmax;
      double len;
      if (f.size() != 6 || !to_i64(f[0], id) || !to_i64(f[1], a) || !to_i64(f[2], b) ||
          !to_f64(f[3], len) || !to_i64(f[4], lanes) || !to_i64(f[5], vmax))
        return err(ebuf, "line %d: %s", L.no, "LINKS record must be `id from to length lanes vmax`");
      if (link_of.count(id)) return err(ebuf, "line %d: %s", L.no, "duplicate link id");
      if (!(len > 0)) return err(ebuf, "line %d: %s", L.no, "non-positive length");
      if (lanes < 1 || lanes > 8) return err(ebuf, "line %d: %s", L.no, "lanes must be 1..8");
      if (vmax < 1 || vmax > 5) return err(ebuf, "line %d: %s", L.no, "vmax must be 1..5");
      link_of[id] = (int32_t)net.len.size();
      ends.push_back({a, b});
      link_line.push_back(L.no);
      net.len.push_back((int64_t)llround(len * 1000.0));
      net.lanes.push_back((int32_t)lanes);
      net.vmax.push_back((int32_t)vmax);
      net.link_id.push_back((int32_t)id);
    } else if (sec == TURNS) {
      int64_t node, in, out, red = 0, green = 0;
      if ((f.size() != 4 && f.size() != 6) || !to_i64(f[0], node) || !to_i64(f[1], in) ||
          !to_i64(f[2], out) || (f.size() == 6 && (!to_i64(f[4], red) || !to_i64(f[5], green))))
        return err(ebuf, "line %d: %s", L.no,
                   "TURNS record must be `node in_link out_link control [red_s green_s]`");
      if (!link_of.count(in) || !link_of.count(out))
        return err(ebuf, "line %d: %s", L.no, "turn references an unknown link");
      turns.push_back({L.no, node, f[3], red, green});
    } else {
      return err(ebuf, "line %d: %s", L.no, "record outside a NODES / LINKS / TURNS section");
    }
  }
  if (net.nx.empty() || net.len.empty()) return err(ebuf, "line %d: %s", L.no, "empty network");
  for (size_t k = 0; k < ends.size(); k++) {
    auto a = node_of.find(ends[k].first), b = node_of.find(ends[k].second);
    if (a == node_of.end() || b == node_of.end())
      return err(ebuf, "line %d: %s", link_line[k], "dangling node reference");
    net.from.push_back(a->second);
    net.to.push_back(b->second);
  }
  // fixed-time two-phase signals: one plan per node (the first `signal`
  // record of the node gives red / green); other controls need no plan
  std::unordered_map<int64_t, bool> seen;
  for (const Turn &t : turns) {
    auto nd = node_of.find(t.node);
    if (nd == node_of.end()) return err(ebuf, "line %d: %s", t.line, "dangling node reference");
    if (t.control != "signal") continue;
    if (t.red < 0 || t.green < 0 || t.red + t.green < 1 || t.red + t.green > 1023)
      return err(ebuf, "line %d: %s", t.line, "signal needs red_s, green_s with 1 <= cycle <= 1023");
    if (seen[t.node]) continue;
    seen[t.node] = true;
    net.sig_node.push_back(nd->second);
    net.sig_green.push_back((int32_t)t.green);
    net.sig_red.push_back((int32_t)t.red);
  }
  return kOk;
}

}  // namespace

extern "C" {

int ts_parse_network_text(const char *text, size_t len, int32_t *n_nodes, int32_t *n_links,
                          int32_t *n_sig, int64_t *node_x_mm, int64_t *node_y_mm, int32_t *from,
                          int32_t *to, int64_t *length_mm, int32_t *lanes, int32_t *vmax,
                          int32_t *prio_class, int32_t *link_id, int32_t *sig_node,
                          int32_t *sig_green, int32_t *sig_red, char *errbuf) {
  if (!text || !n_nodes || !n_links || !n_sig) return kInval;
  Net net;
  if (int rc = parse_network(text, len, net, errbuf)) return rc;
  *n_nodes = (int32_t)net.nx.size();
  *n_links = (int32_t)net.len.size();
  *n_sig = (int32_t)net.sig_node.size();
  auto put = [](auto *dst, const auto &v) {
    if (dst) std::copy(v.begin(), v.end(), dst);
  };
  put(node_x_mm, net.nx);
  put(node_y_mm, net.ny);
  put(from, net.from);
  put(to, net.to);
  put(length_mm, net.len);
  put(lanes, net.lanes);
  put(vmax, net.vmax);
  put(prio_class, net.lanes);  // priority class = lanes (reading R9; the file has none)
  put(link_id, net.link_id);
  put(sig_node, net.sig_node);
  put(sig_green, net.sig_green);
  put(sig_red, net.sig_red);
  return kOk;
}

int ts_parse_plans_text(const char *text, size_t len, int32_t n_links, const int32_t *link_id,
                        int32_t *n_veh, int64_t *n_entries, int64_t *route_off,
                        int32_t *route_links, int32_t *depart, int32_t *entry_cell,
                        int32_t *vehicle_id, char *errbuf) {
  if (!text || !n_veh || !n_entries || n_links < 1 || !link_id) return kInval;
  std::unordered_map<int64_t, int32_t> link_of;
  for (int32_t k = 0; k < n_links; k++) link_of[link_id[k]] = k;
  Lines L{text, text + len};
  std::string ln;
  int64_t nv = 0, ne = 0;
  while (L.next(ln)) {
    const std::vector<std::string> f = fields(ln);
    int64_t vid, dep, entry;
    if (f.size() < 4 || !to_i64(f[0], vid) || !to_i64(f[1], dep) || !to_i64(f[2], entry))
      return err(errbuf, "line %d: %s", L.no,
                 "plan record must be `vehicle_id departure_s entry_cell link_1 ... link_n`");
    if (dep < 0) return err(errbuf, "line %d: %s", L.no, "negative departure time");
    if (route_off) route_off[nv] = ne;
    for (size_t i = 3; i < f.size(); i++) {
      int64_t lid;
      if (!to_i64(f[i], lid)) return err(errbuf, "line %d: %s", L.no, "bad link id");
      auto it = link_of.find(lid);
      if (it == link_of.end()) return err(errbuf, "line %d: %s", L.no, "unknown link id");
      if (route_links) route_links[ne] = it->second;
      ne++;
    }
    if (depart) depart[nv] = (int32_t)dep;
    if (entry_cell) entry_cell[nv] = (int32_t)entry;
    if (vehicle_id) vehicle_id[nv] = (int32_t)vid;
    nv++;
  }
  if (route_off) route_off[nv] = ne;
  *n_veh = (int32_t)nv;
  *n_entries = ne;
  return kOk;
}

}  // extern "C"
