// Mesh ingest and connectivity for the B200 path.
//
// Produces the same Mesh the reference builds (proj/src/mesh.cpp:186-306):
// CCW elements with det(J), tau = det(J) J^-1 and inradius; one edge per
// vertex pair with left = lower element id, unit normal from the left
// element's traversal, boundary edges first grouped by code and then ordered
// by (left, side_left) (mesh.cpp:282-288).  The grouping of half-edges uses a
// linear counting sort on the lower vertex id instead of the reference's
// std::map, so 8M-triangle meshes build in seconds.  The structured
// generators build the precursor directly with the same floating-point
// expressions as the reference's GMSH-text generators (problems.cpp:123-199),
// whose 17-digit text round-trips exactly, so both paths give identical bits.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>

#include "setup.hpp"

namespace dgb {

namespace {

[[noreturn]] void fail_line(int line, const std::string& what) {
  throw MeshError("mesh file, line " + std::to_string(line) + ": " + what);
}

// Line scanner over an in-memory buffer; blank lines are skipped but counted.
struct Scanner {
  const char* p;
  const char* end;
  int line_no = 0;
  std::string cur;
  Scanner(const char* text, std::size_t len) : p(text), end(text + len) {}
  bool next() {
    while (p < end) {
      const char* nl = static_cast<const char*>(std::memchr(p, '\n', end - p));
      const char* stop = nl ? nl : end;
      ++line_no;
      cur.assign(p, stop);
      p = nl ? nl + 1 : end;
      if (!cur.empty() && cur.back() == '\r') cur.pop_back();
      if (!cur.empty()) return true;
    }
    return false;
  }
};

// Whitespace-separated token reader over one line.
struct Tokens {
  const char* s;
  explicit Tokens(const std::string& line) : s(line.c_str()) {}
  bool i64(long long& v) {
    char* e = nullptr;
    errno = 0;
    v = std::strtoll(s, &e, 10);
    if (e == s || errno) return false;
    s = e;
    return true;
  }
  bool f64(double& v) {
    char* e = nullptr;
    v = std::strtod(s, &e);
    if (e == s) return false;
    s = e;
    return true;
  }
  bool word(std::string& w) {
    while (*s == ' ' || *s == '\t') ++s;
    const char* b = s;
    while (*s && *s != ' ' && *s != '\t') ++s;
    w.assign(b, s);
    return !w.empty();
  }
};

inline double hypot2(double dx, double dy) { return std::sqrt(dx * dx + dy * dy); }

}  // namespace

Precursor parse_msh(const char* text, std::size_t len) {
  Scanner sc(text, len);
  Precursor pre;
  std::unordered_map<long long, int> node_index;
  bool saw_format = false, saw_nodes = false, saw_elements = false;
  while (sc.next()) {
    if (sc.cur[0] != '$') continue;
    const std::string section = sc.cur;
    if (section == "$MeshFormat") {
      if (!sc.next()) fail_line(sc.line_no, "unexpected end of file in $MeshFormat");
      Tokens tk(sc.cur);
      std::string version;
      long long file_type = -1, data_size = 0;
      if (!tk.word(version) || !tk.i64(file_type) || !tk.i64(data_size))
        fail_line(sc.line_no, "malformed $MeshFormat header");
      if (version != "2.2")
        fail_line(sc.line_no, "unsupported mesh format version '" + version + "', expected 2.2");
      if (file_type != 0) fail_line(sc.line_no, "binary .msh files are not supported");
      if (!sc.next() || sc.cur != "$EndMeshFormat") fail_line(sc.line_no, "missing $EndMeshFormat");
      saw_format = true;
    } else if (section == "$Nodes") {
      if (!sc.next()) fail_line(sc.line_no, "unexpected end of file in $Nodes");
      long long count = 0;
      {
        Tokens tk(sc.cur);
        if (!tk.i64(count) || count < 0) fail_line(sc.line_no, "malformed node count");
      }
      pre.vx.reserve(count);
      pre.vy.reserve(count);
      node_index.reserve(static_cast<std::size_t>(count) * 2);
      for (long long i = 0; i < count; ++i) {
        if (!sc.next()) fail_line(sc.line_no, "unexpected end of file in $Nodes");
        Tokens tk(sc.cur);
        long long id;
        double x, y, z;
        if (!tk.i64(id) || !tk.f64(x) || !tk.f64(y) || !tk.f64(z))
          fail_line(sc.line_no, "malformed node line");
        if (!std::isfinite(x) || !std::isfinite(y)) fail_line(sc.line_no, "non-finite node coordinates");
        if (!node_index.emplace(id, static_cast<int>(pre.vx.size())).second)
          fail_line(sc.line_no, "duplicate node id " + std::to_string(id));
        pre.vx.push_back(x);
        pre.vy.push_back(y);
      }
      if (!sc.next() || sc.cur != "$EndNodes") fail_line(sc.line_no, "missing $EndNodes");
      saw_nodes = true;
    } else if (section == "$Elements") {
      if (!saw_nodes) fail_line(sc.line_no, "$Elements section before $Nodes");
      if (!sc.next()) fail_line(sc.line_no, "unexpected end of file in $Elements");
      long long count = 0;
      {
        Tokens tk(sc.cur);
        if (!tk.i64(count) || count < 0) fail_line(sc.line_no, "malformed element count");
      }
      auto node = [&](long long id, int line) {
        auto it = node_index.find(id);
        if (it == node_index.end()) fail_line(line, "undefined node " + std::to_string(id));
        return it->second;
      };
      for (long long i = 0; i < count; ++i) {
        if (!sc.next()) fail_line(sc.line_no, "unexpected end of file in $Elements");
        Tokens tk(sc.cur);
        long long id, type, ntags;
        if (!tk.i64(id) || !tk.i64(type) || !tk.i64(ntags)) fail_line(sc.line_no, "malformed element line");
        int first_tag = 0;
        for (long long t = 0; t < ntags; ++t) {
          long long tag;
          if (!tk.i64(tag)) fail_line(sc.line_no, "malformed element tags");
          if (t == 0) first_tag = static_cast<int>(tag);
        }
        if (type == 2) {
          long long a, b, c;
          if (!tk.i64(a) || !tk.i64(b) || !tk.i64(c)) fail_line(sc.line_no, "triangle needs 3 node ids");
          pre.tris.push_back({node(a, sc.line_no), node(b, sc.line_no), node(c, sc.line_no)});
        } else if (type == 1) {
          long long a, b;
          if (!tk.i64(a) || !tk.i64(b)) fail_line(sc.line_no, "line element needs 2 node ids");
          pre.lines.push_back({node(a, sc.line_no), node(b, sc.line_no), ntags > 0 ? first_tag : 0});
        } else if (type == 15) {
          // point elements carry no solver information
        } else {
          fail_line(sc.line_no, "unsupported element type " + std::to_string(type) +
                                    " (only 3-node triangles, 2-node lines and points)");
        }
      }
      if (!sc.next() || sc.cur != "$EndElements") fail_line(sc.line_no, "missing $EndElements");
      saw_elements = true;
    } else {
      const std::string end = "$End" + section.substr(1);
      bool closed = false;
      while (sc.next())
        if (sc.cur == end) {
          closed = true;
          break;
        }
      if (!closed) fail_line(sc.line_no, "unterminated section " + section);
    }
  }
  if (!saw_format) throw MeshError("mesh file: missing $MeshFormat section");
  if (!saw_nodes) throw MeshError("mesh file: missing $Nodes section");
  if (!saw_elements) throw MeshError("mesh file: missing $Elements section");
  return pre;
}

Mesh build_connectivity(const Precursor& pre) {
  Mesh m;
  m.vx = pre.vx;
  m.vy = pre.vy;
  const int nv = static_cast<int>(m.vx.size());
  const int n = static_cast<int>(pre.tris.size());
  m.n_elem = n;
  m.elem_v.resize(3 * static_cast<std::size_t>(n));
  m.elem_edge.assign(3 * static_cast<std::size_t>(n), -1);
  m.det.resize(n);
  m.tau.resize(4 * static_cast<std::size_t>(n));
  m.inradius.resize(n);
  const bool periodic = !pre.key_of.empty();
  auto key_vertex = [&](int v) { return periodic ? pre.key_of[v] : v; };

  for (int i = 0; i < n; ++i) {
    int v[3] = {pre.tris[i][0], pre.tris[i][1], pre.tris[i][2]};
    if (v[0] == v[1] || v[1] == v[2] || v[0] == v[2])
      throw MeshError("triangle " + std::to_string(i) + " has repeated vertices");
    for (int k = 0; k < 3; ++k)
      if (v[k] < 0 || v[k] >= nv)
        throw MeshError("triangle " + std::to_string(i) + " references missing vertex");
    {
      const double abx = m.vx[v[1]] - m.vx[v[0]], aby = m.vy[v[1]] - m.vy[v[0]];
      const double acx = m.vx[v[2]] - m.vx[v[0]], acy = m.vy[v[2]] - m.vy[v[0]];
      if (abx * acy - aby * acx < 0.0) std::swap(v[1], v[2]);  // CW -> CCW
    }
    const double ax = m.vx[v[0]], ay = m.vy[v[0]];
    const double bx = m.vx[v[1]], by = m.vy[v[1]];
    const double cx = m.vx[v[2]], cy = m.vy[v[2]];
    const double j00 = bx - ax, j01 = cx - ax, j10 = by - ay, j11 = cy - ay;
    const double det = j00 * j11 - j01 * j10;
    const double scale = std::max({std::abs(j00), std::abs(j01), std::abs(j10), std::abs(j11)});
    if (det <= 1e-14 * scale * scale)
      throw MeshError("degenerate (collinear or clockwise) triangle, det(J) = " + std::to_string(det));
    for (int k = 0; k < 3; ++k) m.elem_v[3 * i + k] = v[k];
    m.det[i] = det;
    m.tau[4 * i + 0] = j11;
    m.tau[4 * i + 1] = -j01;
    m.tau[4 * i + 2] = -j10;
    m.tau[4 * i + 3] = j00;
    const double perim = hypot2(bx - ax, by - ay) + hypot2(cx - bx, cy - by) + hypot2(ax - cx, ay - cy);
    m.inradius[i] = det / perim;
  }

  // Boundary tags keyed by the unordered (representative) vertex pair.
  auto pack = [](int a, int b) {
    const int lo = std::min(a, b), hi = std::max(a, b);
    return (static_cast<unsigned long long>(static_cast<unsigned>(lo)) << 32) | static_cast<unsigned>(hi);
  };
  std::unordered_map<unsigned long long, int> tag_of;
  tag_of.reserve(pre.lines.size() * 2 + 1);
  for (const auto& ln : pre.lines) {
    if (ln.tag <= 0)
      throw MeshError("boundary line (" + std::to_string(ln.v0) + "," + std::to_string(ln.v1) +
                      ") has no positive physical tag");
    auto [it, inserted] = tag_of.emplace(pack(key_vertex(ln.v0), key_vertex(ln.v1)), ln.tag);
    if (!inserted && it->second != ln.tag)
      throw MeshError("conflicting boundary tags on edge (" + std::to_string(ln.v0) + "," +
                      std::to_string(ln.v1) + ")");
  }

  // Half-edges bucketed by lower representative vertex (counting sort), then
  // by the upper vertex inside each (small) bucket.
  const std::size_t nh = 3 * static_cast<std::size_t>(n);
  std::vector<int> start(nv + 1, 0);
  for (int i = 0; i < n; ++i)
    for (int q = 0; q < 3; ++q) {
      const int a = key_vertex(m.elem_v[3 * i + q]), b = key_vertex(m.elem_v[3 * i + (q + 1) % 3]);
      ++start[std::min(a, b) + 1];
    }
  for (int v = 0; v < nv; ++v) start[v + 1] += start[v];
  struct Half {
    int hi, elem, side;
  };
  std::vector<Half> half(nh);
  {
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (int i = 0; i < n; ++i)
      for (int q = 0; q < 3; ++q) {
        const int a = key_vertex(m.elem_v[3 * i + q]), b = key_vertex(m.elem_v[3 * i + (q + 1) % 3]);
        half[fill[std::min(a, b)]++] = {std::max(a, b), i, q + 1};
      }
  }
  struct EdgeRec {
    unsigned long long order;
    int v0, v1, left, right, sl, sr;
  };
  std::vector<EdgeRec> edges;
  edges.reserve(nh / 2 + nv);
  for (int lo = 0; lo < nv; ++lo) {
    Half* b = half.data() + start[lo];
    Half* e = half.data() + start[lo + 1];
    std::sort(b, e, [](const Half& x, const Half& y) {
      return x.hi != y.hi ? x.hi < y.hi : x.elem < y.elem;
    });
    for (Half* g = b; g < e;) {
      Half* h = g;
      while (h < e && h->hi == g->hi) ++h;
      const long cnt = h - g;
      const unsigned long long key = pack(lo, g->hi);
      EdgeRec r{};
      if (cnt > 2)
        throw MeshError("non-manifold edge (" + std::to_string(lo) + "," + std::to_string(g->hi) +
                        ") shared by more than two triangles");
      if (cnt == 2) {
        if (tag_of.count(key))
          throw MeshError("boundary tag on interior edge (" + std::to_string(lo) + "," +
                          std::to_string(g->hi) + ")");
        r.left = g[0].elem;  // sorted by element id: lower id is the left element
        r.sl = g[0].side;
        r.right = g[1].elem;
        r.sr = g[1].side;
        r.order = (1ull << 62) | (static_cast<unsigned long long>(r.left) << 2) | r.sl;
      } else {
        auto it = tag_of.find(key);
        if (it == tag_of.end())
          throw MeshError("hull edge (" + std::to_string(lo) + "," + std::to_string(g->hi) +
                          ") has no boundary tag");
        r.left = g[0].elem;
        r.sl = g[0].side;
        r.right = -it->second;
        r.sr = 0;
        // codes descending (-1 first), then (left, side_left)
        r.order = (static_cast<unsigned long long>(it->second) << 33) |
                  (static_cast<unsigned long long>(r.left) << 2) | r.sl;
      }
      r.v0 = m.elem_v[3 * r.left + r.sl - 1];
      r.v1 = m.elem_v[3 * r.left + r.sl % 3];
      edges.push_back(r);
      g = h;
    }
  }
  std::sort(edges.begin(), edges.end(),
            [](const EdgeRec& a, const EdgeRec& b) { return a.order < b.order; });

  const int ne = static_cast<int>(edges.size());
  m.n_edges = ne;
  m.ev0.resize(ne);
  m.ev1.resize(ne);
  m.eleft.resize(ne);
  m.eright.resize(ne);
  m.eside_l.resize(ne);
  m.eside_r.resize(ne);
  m.enx.resize(ne);
  m.eny.resize(ne);
  m.eh.resize(ne);
  m.n_boundary = 0;
  for (int k = 0; k < ne; ++k) {
    const EdgeRec& r = edges[k];
    m.ev0[k] = r.v0;
    m.ev1[k] = r.v1;
    m.eleft[k] = r.left;
    m.eright[k] = r.right;
    m.eside_l[k] = r.sl;
    m.eside_r[k] = r.sr;
    const double dx = m.vx[r.v1] - m.vx[r.v0], dy = m.vy[r.v1] - m.vy[r.v0];
    const double len = hypot2(dx, dy);
    if (len == 0.0) throw MeshError("zero-length edge");
    m.enx[k] = dy / len;
    m.eny[k] = -dx / len;
    m.eh[k] = 0.5 * len;
    if (r.right < 0) ++m.n_boundary;
    m.elem_edge[3 * r.left + r.sl - 1] = k;
    if (r.right >= 0) m.elem_edge[3 * r.right + r.sr - 1] = k;
  }
  for (int i = 0; i < n; ++i)
    for (int q = 0; q < 3; ++q)
      if (m.elem_edge[3 * i + q] < 0)
        throw MeshError("element " + std::to_string(i) + " is missing edge on side " + std::to_string(q + 1));
  return m;
}

namespace {

void split_quads(int nx, int ny, std::vector<std::array<int, 3>>& tris) {
  tris.reserve(tris.size() + 2 * static_cast<std::size_t>(nx) * ny);
  auto vid = [nx](int i, int j) { return j * (nx + 1) + i; };
  for (int j = 0; j < ny; ++j)
    for (int i = 0; i < nx; ++i) {
      tris.push_back({vid(i, j), vid(i + 1, j), vid(i, j + 1)});
      tris.push_back({vid(i + 1, j), vid(i + 1, j + 1), vid(i, j + 1)});
    }
}

double param(const double* p, int n, int i, double dflt) { return (p && i < n) ? p[i] : dflt; }

}  // namespace

Precursor generate(int kind, int nx, int ny, const double* prm, int np) {
  Precursor pre;
  auto vid = [nx](int i, int j) { return j * (nx + 1) + i; };
  switch (kind) {
    case kBox:
    case kShearedBox:
    case kPeriodicBox: {
      if (nx < 1 || ny < 1) throw std::invalid_argument("box mesh needs nx, ny >= 1");
      const double width = param(prm, np, 0, 1.0), height = param(prm, np, 1, 1.0);
      const double shear = kind == kShearedBox ? param(prm, np, 2, 0.0) : 0.0;
      const int tag = static_cast<int>(param(prm, np, kind == kShearedBox ? 3 : 2, 1.0));
      if (kind == kPeriodicBox && (nx < 2 || ny < 2))
        throw std::invalid_argument("periodic box needs nx, ny >= 2");
      pre.vx.reserve(static_cast<std::size_t>(nx + 1) * (ny + 1));
      pre.vy.reserve(static_cast<std::size_t>(nx + 1) * (ny + 1));
      for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
          pre.vx.push_back(width * i / nx + shear * height * j / ny);
          pre.vy.push_back(height * j / ny);
        }
      split_quads(nx, ny, pre.tris);
      if (kind == kPeriodicBox) {
        pre.key_of.resize(pre.vx.size());
        for (int j = 0; j <= ny; ++j)
          for (int i = 0; i <= nx; ++i) pre.key_of[vid(i, j)] = vid(i % nx, j % ny);
      } else {
        for (int i = 0; i < nx; ++i) {
          pre.lines.push_back({vid(i, 0), vid(i + 1, 0), tag});
          pre.lines.push_back({vid(i, ny), vid(i + 1, ny), tag});
        }
        for (int j = 0; j < ny; ++j) {
          pre.lines.push_back({vid(0, j), vid(0, j + 1), tag});
          pre.lines.push_back({vid(nx, j), vid(nx, j + 1), tag});
        }
      }
      break;
    }
    case kDoubleMach: {
      if (nx < 2 || ny < 1) throw std::invalid_argument("double-mach mesh needs nx >= 2, ny >= 1");
      const double x0 = param(prm, np, 0, 1.0 / 6.0);
      const double lx = 4.0, ly = 1.0;
      for (int j = 0; j <= ny; ++j)
        for (int i = 0; i <= nx; ++i) {
          pre.vx.push_back(lx * i / nx);
          pre.vy.push_back(ly * j / ny);
        }
      split_quads(nx, ny, pre.tris);
      for (int i = 0; i < nx; ++i) {
        const double xm = lx * (i + 0.5) / nx;
        pre.lines.push_back({vid(i, 0), vid(i + 1, 0), xm < x0 ? 3 : 1});
        pre.lines.push_back({vid(i, ny), vid(i + 1, ny), 5});
      }
      for (int j = 0; j < ny; ++j) {
        pre.lines.push_back({vid(0, j), vid(0, j + 1), 3});
        pre.lines.push_back({vid(nx, j), vid(nx, j + 1), 4});
      }
      break;
    }
    case kVortex: {
      const int level = nx;
      if (level < 0 || level > 9) throw std::invalid_argument("vortex mesh level must be 0..9");
      const double r_in = param(prm, np, 0, 1.0), r_out = param(prm, np, 1, 1.384);
      const int nr = 5 << level, nt = 18 << level;
      auto rv = [nr](int i, int j) { return j * (nr + 1) + i; };
      pre.vx.reserve(static_cast<std::size_t>(nr + 1) * (nt + 1));
      pre.vy.reserve(static_cast<std::size_t>(nr + 1) * (nt + 1));
      for (int j = 0; j <= nt; ++j) {
        const double theta = 0.5 * M_PI * j / nt;
        for (int i = 0; i <= nr; ++i) {
          const double r = r_in + (r_out - r_in) * i / nr;
          pre.vx.push_back(r * std::cos(theta));
          pre.vy.push_back(r * std::sin(theta));
        }
      }
      split_quads(nr, nt, pre.tris);
      for (int i = 0; i < nr; ++i) {
        pre.lines.push_back({rv(i, 0), rv(i + 1, 0), 3});
        pre.lines.push_back({rv(i, nt), rv(i + 1, nt), 4});
      }
      for (int j = 0; j < nt; ++j) {
        pre.lines.push_back({rv(0, j), rv(0, j + 1), 2});
        pre.lines.push_back({rv(nr, j), rv(nr, j + 1), 2});
      }
      break;
    }
    default:
      throw std::invalid_argument("unknown mesh kind " + std::to_string(kind));
  }
  return pre;
}

std::string format_msh(const Precursor& pre) {
  if (!pre.key_of.empty()) throw std::invalid_argument("periodic meshes have no GMSH v2.2 text form here");
  std::string out;
  out.reserve(64 * (pre.vx.size() + pre.tris.size() + pre.lines.size()) + 128);
  char buf[160];
  out += "$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n";
  out += std::to_string(pre.vx.size()) + "\n";
  for (std::size_t i = 0; i < pre.vx.size(); ++i) {
    int len = std::snprintf(buf, sizeof buf, "%zu %.17g %.17g 0\n", i + 1, pre.vx[i], pre.vy[i]);
    out.append(buf, len);
  }
  out += "$EndNodes\n$Elements\n" + std::to_string(pre.tris.size() + pre.lines.size()) + "\n";
  long long id = 1;
  for (const auto& ln : pre.lines) {
    int len = std::snprintf(buf, sizeof buf, "%lld 1 2 %d %d %d %d\n", id++, ln.tag, ln.tag, ln.v0 + 1, ln.v1 + 1);
    out.append(buf, len);
  }
  for (const auto& t : pre.tris) {
    int len = std::snprintf(buf, sizeof buf, "%lld 2 2 10 10 %d %d %d\n", id++, t[0] + 1, t[1] + 1, t[2] + 1);
    out.append(buf, len);
  }
  out += "$EndElements\n";
  return out;
}

std::string dump_edges(const Mesh& m) {
  std::string out;
  char buf[256];
  for (int k = 0; k < m.n_edges; ++k) {
    int len = std::snprintf(buf, sizeof buf, "%d %d %d %d %d %d %.17g %.17g %.17g\n", m.ev0[k], m.ev1[k],
                            m.eleft[k], m.eright[k], m.eside_l[k], m.eside_r[k], m.enx[k], m.eny[k], m.eh[k]);
    out.append(buf, len);
  }
  return out;
}

}  // namespace dgb
