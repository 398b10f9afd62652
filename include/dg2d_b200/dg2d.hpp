// dg2d_b200/dg2d.hpp — header-only C++ mirror of the reference solver API
// (/root/reference/proj/include/dg2d/{mesh,basis,euler,solver,problems}.hpp) on top of
// the C ABI in dg2d_b200.h.  Same type and function names, argument meaning and
// exception types as namespace dg2d, in namespace dg2d_b200 so that both can be
// linked into one binary (the C++ parity test does exactly that).
//
// Differences a caller sees:
//   * SolverContext owns a device context (created on first use, one per
//     context, device `device`); every pass runs on the B200 through the C ABI.
//     There is no CPU fallback: without a device the first call throws.
//   * BoundaryConditions closures are evaluated once on the host at every
//     boundary Gauss point when the device context is created (the reference
//     calls them from inside the surface pass); set `time_dependent` to re-evaluate
//     the Dirichlet table before each RHS evaluation.
//   * SolverOptions::scheme selects SSP-RK2/3 (not in the reference) besides
//     rk_order 2 (midpoint) and 4 (classical).
//   * workers/chunk are accepted and ignored (the device decides the parallelism).
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <functional>
#include <utility>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "dg2d_b200.h"

namespace dg2d_b200 {

// ------------------------------------------------------------------ L0 (geometry.hpp, euler.hpp)
struct Vec2 {
  double x = 0.0, y = 0.0;
};

constexpr int kEq = 4;

struct EulerState {  // euler.hpp:15-23
  double rho = 0.0, mx = 0.0, my = 0.0, E = 0.0;
  double& operator[](int m) { return (&rho)[m]; }
  double operator[](int m) const { return (&rho)[m]; }
};

struct GasModel {  // euler.hpp:25-27
  double gamma = 1.4;
};

inline double pressure(const EulerState& u, const GasModel& gas) {  // euler.hpp:29-31
  return (gas.gamma - 1.0) * (u.E - 0.5 * (u.mx * u.mx + u.my * u.my) / u.rho);
}

struct MovingShock {  // euler.hpp:91-102
  double x0 = 0.0;
  double angle_deg = 60.0;
  double speed = 10.0;
  EulerState post;
  EulerState pre;
};

struct BoundaryConditions {  // euler.hpp:104-111
  EulerState inflow_state;
  std::function<EulerState(Vec2, double)> dirichlet;
  std::function<Vec2(Vec2)> wall_normal;
  std::optional<MovingShock> shock;
  bool time_dependent = false;  // (new) re-evaluate `dirichlet` before every RHS
};

// ------------------------------------------------------------------ errors
struct SolverAbort : std::runtime_error {  // solver.hpp:14-16
  using std::runtime_error::runtime_error;
};
struct MeshError : std::runtime_error {  // mesh.hpp:15-17
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int rc) {
  if (rc == DGB_OK) return;
  const char* m = dgb_last_message();
  const std::string msg = m ? m : "dg2d_b200 error";
  switch (rc) {
    case DGB_ERR_INADMISSIBLE:
    case DGB_ERR_BC:
    case DGB_ERR_NOT_REACHED: throw SolverAbort(msg);
    case DGB_ERR_ARG: throw std::invalid_argument(msg);
    case DGB_ERR_MESH: throw MeshError(msg);
    default: throw std::runtime_error(msg);
  }
}
}  // namespace detail

// ------------------------------------------------------------------ L1 mesh (mesh.hpp)
struct MeshPrecursor {  // the GMSH text; parsed together with the connectivity
  std::string text;
};

inline MeshPrecursor parse_msh(std::string_view text) { return MeshPrecursor{std::string(text)}; }

inline MeshPrecursor parse_msh_file(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw MeshError("cannot open mesh file '" + path + "'");
  return MeshPrecursor{std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>())};
}

class Mesh {  // mesh.hpp:46-63, SoA arrays behind a dgb_mesh handle
 public:
  explicit Mesh(dgb_mesh* h) : h_(h, &dgb_mesh_free) { detail::check(dgb_mesh_get_view(h, &v_)); }
  int n_elements() const { return v_.n_elements; }
  int n_edges() const { return v_.n_edges; }
  int n_boundary_edges() const { return v_.n_boundary_edges; }
  int neighbor(int i, int q) const {  // mesh.hpp:56-59
    const int e = v_.elem_edge[3 * i + q];
    return v_.edge_left[e] == i ? v_.edge_right[e] : v_.edge_left[e];
  }
  Vec2 vertex_of(int elem, int local) const {
    const int v = v_.elem_v[3 * elem + local];
    return {v_.vx[v], v_.vy[v]};
  }
  double det_jac(int i) const { return v_.det_jac[i]; }
  double total_area() const {
    double a = 0.0;
    for (int i = 0; i < n_elements(); ++i) a += 0.5 * v_.det_jac[i];
    return a;
  }
  std::string dump_edges() const {  // mesh.cpp:308-313
    size_t need = 0;
    detail::check(dgb_mesh_dump_edges(h_.get(), nullptr, 0, &need));
    std::string s(need, '\0');
    detail::check(dgb_mesh_dump_edges(h_.get(), s.data(), s.size(), &need));
    s.resize(need);
    while (!s.empty() && s.back() == '\0') s.pop_back();
    return s;
  }
  const dgb_mesh_view& view() const { return v_; }

 private:
  std::shared_ptr<dgb_mesh> h_;
  dgb_mesh_view v_{};
};

inline Mesh build_connectivity(const MeshPrecursor& pre) {  // mesh.cpp:186-306
  dgb_mesh* h = nullptr;
  detail::check(dgb_mesh_from_msh(pre.text.data(), pre.text.size(), &h));
  return Mesh(h);
}

namespace detail {
inline std::string gen_text(int kind, int nx, int ny, std::vector<double> prm) {
  size_t need = 0;
  detail::check(dgb_mesh_generate_text(kind, nx, ny, prm.data(), static_cast<int>(prm.size()), nullptr, 0, &need));
  std::string s(need, '\0');
  detail::check(
      dgb_mesh_generate_text(kind, nx, ny, prm.data(), static_cast<int>(prm.size()), s.data(), s.size(), &need));
  while (!s.empty() && s.back() == '\0') s.pop_back();
  return s;
}
}  // namespace detail

// ------------------------------------------------------------------ problems.hpp (generators, data)
struct VortexGeometry {  // problems.hpp:13-19
  double r_inner = 1.0;
  double r_outer = 1.384;
  double mach_inner = 2.25;
  double rho_inner = 1.0;
  double sound_speed_inner = 1.0;
};

inline std::string gen_vortex_msh(int level, const VortexGeometry& geo = {}) {
  return detail::gen_text(DGB_MESH_VORTEX, level, 0, {geo.r_inner, geo.r_outer});
}
inline std::string gen_double_mach_msh(int nx, int ny, double x0 = 1.0 / 6.0) {
  return detail::gen_text(DGB_MESH_DOUBLE_MACH, nx, ny, {x0});
}
inline std::string gen_box_msh(int nx, int ny, double width, double height, int tag) {
  return detail::gen_text(DGB_MESH_BOX, nx, ny, {width, height, static_cast<double>(tag)});
}
inline std::string gen_sheared_box_msh(int nx, int ny, double width, double height, double shear, int tag) {
  return detail::gen_text(DGB_MESH_SHEARED_BOX, nx, ny, {width, height, shear, static_cast<double>(tag)});
}
// Direct generator (identical to build_connectivity(parse_msh(gen_*_msh(...))), no text round trip).
inline Mesh generate_mesh(int kind, int nx, int ny, std::vector<double> prm) {
  dgb_mesh* h = nullptr;
  detail::check(dgb_mesh_generate(kind, nx, ny, prm.data(), static_cast<int>(prm.size()), &h));
  return Mesh(h);
}

inline EulerState vortex_exact(Vec2 p, const VortexGeometry& geo, const GasModel& gas) {  // problems.cpp:44-66
  double xy[2] = {p.x, p.y}, s[4];
  detail::check(dgb_vortex_exact(xy, 1, geo.r_inner, geo.r_outer, geo.mach_inner, geo.rho_inner,
                                 geo.sound_speed_inner, gas.gamma, s));
  return {s[0], s[1], s[2], s[3]};
}

inline BoundaryConditions vortex_boundary(const VortexGeometry& geo, const GasModel& gas) {  // problems.cpp:68-77
  BoundaryConditions bc;
  bc.inflow_state = vortex_exact({0.5 * (geo.r_inner + geo.r_outer), 0.0}, geo, gas);
  bc.dirichlet = [geo, gas](Vec2 x, double) { return vortex_exact(x, geo, gas); };
  bc.wall_normal = [](Vec2 x) {
    const double r = std::hypot(x.x, x.y);
    return Vec2{x.x / r, x.y / r};
  };
  return bc;
}

inline EulerState rankine_hugoniot_post(const EulerState& pre, double mach, Vec2 n, const GasModel& gas) {
  double u[4] = {pre.rho, pre.mx, pre.my, pre.E}, o[4];
  detail::check(dgb_rankine_hugoniot_post(u, mach, n.x, n.y, gas.gamma, o));
  return {o[0], o[1], o[2], o[3]};
}

struct DoubleMachSetup {  // problems.hpp:34-44
  double x0 = 1.0 / 6.0;
  double shock_mach = 10.0;
  double angle_deg = 60.0;
  EulerState pre{1.4, 0.0, 0.0, 1.0 / 0.4};
  EulerState post;
  DoubleMachSetup() {
    const double rad = angle_deg * M_PI / 180.0;
    post = rankine_hugoniot_post(pre, shock_mach, {std::sin(rad), -std::cos(rad)}, GasModel{});
  }
};

inline BoundaryConditions double_mach_boundary(const DoubleMachSetup& s, const GasModel& = {}) {  // :102-115
  BoundaryConditions bc;
  bc.inflow_state = s.post;
  MovingShock sh;
  sh.x0 = s.x0;
  sh.angle_deg = s.angle_deg;
  sh.speed = s.shock_mach * std::sqrt(1.4 * pressure(s.pre, GasModel{}) / s.pre.rho);
  sh.post = s.post;
  sh.pre = s.pre;
  bc.shock = sh;
  return bc;
}

inline EulerState double_mach_initial(Vec2 p, const DoubleMachSetup& s) {  // problems.cpp:117-121
  const double rad = s.angle_deg * M_PI / 180.0;
  const double front = s.x0 + p.y * std::cos(rad) / std::sin(rad);
  return p.x < front ? s.post : s.pre;
}

// ------------------------------------------------------------------ L1 basis (basis.hpp)
class BasisTables {
 public:
  explicit BasisTables(int p) {
    dgb_tables* h = nullptr;
    detail::check(dgb_tables_build(p, &h));
    h_ = std::shared_ptr<dgb_tables>(h, &dgb_tables_free);
    detail::check(dgb_tables_get_view(h, &v_));
    this->p = v_.p;
    n_p = v_.n_p;
    n_quad = v_.n_quad;
    n_edge_pts = v_.n_edge_pts;
  }
  int p = 0, n_p = 0, n_quad = 0, n_edge_pts = 0;
  double phi_int(int k, int j) const { return v_.phi_interior[k * n_p + j]; }
  double phi_side(int q, int k, int j) const { return v_.phi_edge[((q - 1) * n_edge_pts + k) * n_p + j]; }
  double w_int(int k) const { return v_.w_interior[k]; }
  const dgb_tables_view& view() const { return v_; }

 private:
  std::shared_ptr<dgb_tables> h_;
  dgb_tables_view v_{};
};

inline BasisTables build_tables(int p) { return BasisTables(p); }  // basis.cpp:201-242

// ------------------------------------------------------------------ L2 solver (solver.hpp)
struct CoefficientArray {  // solver.hpp:20-38
  int n_eq = 0, n_modes = 0, n_elem = 0;
  std::vector<double> data;
  CoefficientArray() = default;
  CoefficientArray(int eq, int modes, int elem)
      : n_eq(eq), n_modes(modes), n_elem(elem), data(static_cast<size_t>(eq) * modes * elem, 0.0) {}
  size_t idx(int m, int j, int i) const { return (static_cast<size_t>(m) * n_modes + j) * n_elem + i; }
  double& at(int m, int j, int i) { return data[idx(m, j, i)]; }
  double at(int m, int j, int i) const { return data[idx(m, j, i)]; }
  void fill_zero() { std::fill(data.begin(), data.end(), 0.0); }
};

struct RhsBuffers {  // solver.hpp:46-62
  CoefficientArray volume;
  std::vector<double> surface_left, surface_right;
  int n_eq = 0, n_modes = 0, n_elem = 0;
  RhsBuffers() = default;
  RhsBuffers(int eq, int modes, int elem)
      : volume(eq, modes, elem),
        surface_left(static_cast<size_t>(3) * eq * modes * elem, 0.0),
        surface_right(static_cast<size_t>(3) * eq * modes * elem, 0.0),
        n_eq(eq), n_modes(modes), n_elem(elem) {}
  size_t slot(int q, int m, int j, int i) const {
    return ((static_cast<size_t>(q) * n_eq + m) * n_modes + j) * n_elem + i;
  }
};

struct PassTimers {  // solver.hpp:64-70 (+ the fused stage kernels)
  double volume = 0.0, surface = 0.0, rhs = 0.0, limiter = 0.0, other = 0.0, stage = 0.0;
};

enum class RkScheme { kFromOrder = 0, kSspRk2 = DGB_SSP_RK2, kSspRk3 = DGB_SSP_RK3 };

struct SolverOptions {  // solver.hpp:72-78
  int rk_order = 4;  // 2 or 4
  double cfl = 0.3;
  bool limiting = false;
  int workers = 0;  // accepted, unused on the device
  int chunk = 256;  // accepted, unused on the device
  RkScheme scheme = RkScheme::kFromOrder;  // (new) SSP schemes
  int flux = DGB_FLUX_LLF;                 // (new) DGB_FLUX_LLF (euler.hpp:59-71) or DGB_FLUX_ROE
  int scheme_id() const { return scheme == RkScheme::kFromOrder ? rk_order : static_cast<int>(scheme); }
};

struct SolverState {  // solver.hpp:89-93
  CoefficientArray coeffs;
  double t = 0.0;
  std::int64_t step_count = 0;
};

struct SteadyResult {
  std::int64_t steps = 0;
  double residual = 0.0;
  bool converged = false;
};

using RhsOperator = std::function<void(const CoefficientArray& coeffs, double t, CoefficientArray& deriv)>;

namespace detail {
struct Device {
  dgb_ctx* ctx = nullptr;
  ~Device() {
    if (ctx) dgb_destroy(ctx);
  }
};

// Host evaluation of the BC closures at the boundary Gauss points (solver.cpp:198).
inline void bc_tables(const Mesh& mesh, const BasisTables& tb, const BoundaryConditions& bc, double t,
                      std::vector<double>& dir, std::vector<double>& wn) {
  const int nb = mesh.n_boundary_edges(), K = tb.n_edge_pts;
  std::vector<double> xy(2 * static_cast<size_t>(nb) * K + 2);
  detail::check(dgb_boundary_points(&mesh.view(), &tb.view(), xy.data()));
  dir.clear();
  wn.clear();
  if (bc.dirichlet) {
    dir.assign(4 * static_cast<size_t>(nb) * K, 0.0);
    for (int e = 0; e < nb; ++e)
      if (mesh.view().edge_right[e] == -3)
        for (int k = 0; k < K; ++k) {
          const size_t pk = static_cast<size_t>(e) * K + k;
          const EulerState s = bc.dirichlet({xy[2 * pk], xy[2 * pk + 1]}, t);
          for (int m = 0; m < 4; ++m) dir[4 * pk + m] = s[m];
        }
  }
  if (bc.wall_normal) {
    wn.assign(2 * static_cast<size_t>(nb) * K, 0.0);
    for (int e = 0; e < nb; ++e)
      if (mesh.view().edge_right[e] == -2)
        for (int k = 0; k < K; ++k) {
          const size_t pk = static_cast<size_t>(e) * K + k;
          const Vec2 n = bc.wall_normal({xy[2 * pk], xy[2 * pk + 1]});
          wn[2 * pk] = n.x;
          wn[2 * pk + 1] = n.y;
        }
  }
}
}  // namespace detail

struct SolverContext {  // solver.hpp:80-87
  const Mesh* mesh = nullptr;
  const BasisTables* tables = nullptr;
  GasModel gas;
  const BoundaryConditions* bc = nullptr;
  SolverOptions options;
  mutable PassTimers timers;
  int device = 0;  // (new) CUDA ordinal

  // The device context (created on first use).
  dgb_ctx* handle() const {
    if (!dev_) {
      dev_ = std::make_shared<detail::Device>();
      static const BoundaryConditions kNone{};
      const BoundaryConditions& b = bc ? *bc : kNone;
      std::vector<double> dir, wn;
      detail::bc_tables(*mesh, *tables, b, 0.0, dir, wn);
      dgb_bc_view v{};
      for (int m = 0; m < 4; ++m) v.inflow_state[m] = b.inflow_state[m];
      v.dirichlet_state = dir.empty() ? nullptr : dir.data();
      v.wall_normal = wn.empty() ? nullptr : wn.data();
      if (b.shock) {
        v.has_shock = 1;
        v.shock_x0 = b.shock->x0;
        v.shock_angle_deg = b.shock->angle_deg;
        v.shock_speed = b.shock->speed;
        for (int m = 0; m < 4; ++m) {
          v.shock_post[m] = b.shock->post[m];
          v.shock_pre[m] = b.shock->pre[m];
        }
      }
      detail::check(dgb_create(&mesh->view(), &tables->view(), &v, gas.gamma, device, &dev_->ctx));
      dgb_enable_timers(dev_->ctx, 1);
      detail::check(dgb_set_flux(dev_->ctx, options.flux));
    }
    return dev_->ctx;
  }
  void refresh_bc(double t) const {
    if (time_dependent()) {
      std::vector<double> dir, wn;
      detail::bc_tables(*mesh, *tables, *bc, t, dir, wn);
      detail::check(dgb_set_dirichlet(handle(), dir.data()));
    }
  }
  bool time_dependent() const { return bc && bc->time_dependent && bc->dirichlet; }
  // The Dirichlet closure at every stage time t + c_k dt of the next step (the reference
  // evaluates it inside each surface pass, solver.cpp:198-211).
  void stage_bc(double t, double dt) const {
    double c[8];
    int n = 0;
    detail::check(dgb_scheme_stage_times(options.scheme_id(), c, &n));
    std::vector<double> all, dir, wn;
    for (int k = 0; k < n; ++k) {
      detail::bc_tables(*mesh, *tables, *bc, t + c[k] * dt, dir, wn);
      all.insert(all.end(), dir.begin(), dir.end());
    }
    if (all.empty()) return;  // no boundary Gauss points (e.g. a periodic mesh)
    detail::check(dgb_set_dirichlet_stages(handle(), n, all.data()));
  }
  void read_timers() const {
    dgb_pass_timers t{};
    detail::check(dgb_timers(handle(), &t));
    timers = {t.volume, t.surface, t.rhs, t.limiter, t.other, t.stage};
  }

 private:
  mutable std::shared_ptr<detail::Device> dev_;
};

namespace detail {
inline void need_shape(const SolverContext& ctx, const CoefficientArray& c) {
  if (c.n_eq != kEq || c.n_modes != ctx.tables->n_p || c.n_elem != ctx.mesh->n_elements())
    throw std::invalid_argument("coefficient array shape does not match the mesh and tables");
}
inline void upload(const SolverContext& ctx, int slot, const CoefficientArray& c) {
  need_shape(ctx, c);
  detail::check(dgb_upload(ctx.handle(), slot, c.data.data()));
}
inline void download(const SolverContext& ctx, int slot, CoefficientArray& c) {
  if (c.n_elem != ctx.mesh->n_elements() || c.n_modes != ctx.tables->n_p || c.n_eq != kEq)
    c = CoefficientArray(kEq, ctx.tables->n_p, ctx.mesh->n_elements());
  detail::check(dgb_download(ctx.handle(), slot, c.data.data()));
}
inline void push_state(const SolverContext& ctx, const SolverState& s) {
  upload(ctx, DGB_SLOT_STATE, s.coeffs);
  detail::check(dgb_set_time(ctx.handle(), s.t, s.step_count));
}
inline void pull_state(const SolverContext& ctx, SolverState& s) {
  download(ctx, DGB_SLOT_STATE, s.coeffs);
  detail::check(dgb_get_time(ctx.handle(), &s.t, &s.step_count));
}
}  // namespace detail

// solver.cpp:74-97
inline CoefficientArray project_initial(const std::function<EulerState(Vec2)>& u0, const Mesh& mesh,
                                        const BasisTables& tb, const GasModel& gas) {
  const int n = mesh.n_elements(), nq = tb.n_quad;
  std::vector<double> xy(2 * static_cast<size_t>(n) * nq), ps(4 * static_cast<size_t>(n) * nq);
  detail::check(dgb_interior_points(&mesh.view(), &tb.view(), xy.data()));
  for (size_t k = 0; k < static_cast<size_t>(n) * nq; ++k) {
    const EulerState s = u0({xy[2 * k], xy[2 * k + 1]});
    for (int m = 0; m < 4; ++m) ps[4 * k + m] = s[m];
  }
  CoefficientArray c(kEq, tb.n_p, n);
  detail::check(dgb_project(&mesh.view(), &tb.view(), gas.gamma, ps.data(), c.data.data()));
  return c;
}

// solver.cpp:99-158
inline void eval_volume_pass(const SolverContext& ctx, const CoefficientArray& coeffs, CoefficientArray& vol) {
  detail::upload(ctx, DGB_SLOT_INPUT, coeffs);
  detail::check(dgb_eval_volume_pass(ctx.handle(), DGB_SLOT_INPUT));
  detail::download(ctx, DGB_SLOT_VOLUME, vol);
}

// solver.cpp:160-251 (slots not owned by an edge side keep their contents)
inline void eval_surface_pass(const SolverContext& ctx, const CoefficientArray& coeffs, double t, RhsBuffers& b) {
  ctx.refresh_bc(t);
  detail::upload(ctx, DGB_SLOT_INPUT, coeffs);
  detail::check(dgb_eval_surface_pass(ctx.handle(), DGB_SLOT_INPUT, t));
  const int n = ctx.mesh->n_elements(), np = ctx.tables->n_p;
  if (b.n_elem != n || b.n_modes != np) b = RhsBuffers(kEq, np, n);
  std::vector<double> sl(b.surface_left.size()), sr(b.surface_right.size());
  detail::check(dgb_download_surface(ctx.handle(), sl.data(), sr.data()));
  const dgb_mesh_view& v = ctx.mesh->view();
  for (int q = 0; q < 3; ++q)
    for (int i = 0; i < n; ++i) {
      const bool from_left = v.edge_left[v.elem_edge[3 * i + q]] == i;
      for (int m = 0; m < kEq; ++m)
        for (int j = 0; j < np; ++j) {
          const size_t s = b.slot(q, m, j, i);
          (from_left ? b.surface_left[s] : b.surface_right[s]) = from_left ? sl[s] : sr[s];
        }
    }
}

// solver.cpp:253-277
inline void eval_rhs_pass(const SolverContext& ctx, const RhsBuffers& b, CoefficientArray& deriv) {
  detail::upload(ctx, DGB_SLOT_VOLUME, b.volume);
  detail::check(dgb_upload_surface(ctx.handle(), b.surface_left.data(), b.surface_right.data()));
  detail::check(dgb_eval_rhs_pass(ctx.handle()));
  detail::download(ctx, DGB_SLOT_DERIV, deriv);
}

// solver.cpp:279-284 — one fused kernel; `bufs` is left untouched (no intermediate buffers exist)
inline void compute_rhs(const SolverContext& ctx, const CoefficientArray& coeffs, double t, RhsBuffers& /*bufs*/,
                        CoefficientArray& deriv) {
  ctx.refresh_bc(t);
  detail::upload(ctx, DGB_SLOT_INPUT, coeffs);
  detail::check(dgb_compute_rhs(ctx.handle(), DGB_SLOT_INPUT, t, DGB_SLOT_DERIV));
  detail::download(ctx, DGB_SLOT_DERIV, deriv);
}

// solver.cpp:286-425
inline void limit(const SolverContext& ctx, CoefficientArray& coeffs) {
  if (ctx.tables->p != 1) throw std::invalid_argument("slope limiting is only supported for p = 1");
  detail::upload(ctx, DGB_SLOT_INPUT, coeffs);
  detail::check(dgb_limit(ctx.handle(), DGB_SLOT_INPUT));
  detail::download(ctx, DGB_SLOT_INPUT, coeffs);
}

// solver.cpp:427-461
inline double stable_dt(const SolverContext& ctx, const CoefficientArray& coeffs) {
  detail::upload(ctx, DGB_SLOT_INPUT, coeffs);
  double dt = 0.0;
  detail::check(dgb_stable_dt(ctx.handle(), DGB_SLOT_INPUT, ctx.options.cfl, &dt));
  return dt;
}

// solver.cpp:545-557 — the whole step on the device
inline double rk_step(const SolverContext& ctx, SolverState& state, double dt) {
  if (ctx.time_dependent()) ctx.stage_bc(state.t, dt);
  detail::push_state(ctx, state);
  double res = 0.0;
  const int rc = dgb_rk_step(ctx.handle(), ctx.options.scheme_id(), dt, ctx.options.limiting ? 1 : 0, &res);
  detail::pull_state(ctx, state);
  detail::check(rc);
  return res;
}

// solver.cpp:506-541 with a caller operator (the plugin seam): stage algebra on the host
inline double rk_step(const SolverContext& ctx, SolverState& state, double dt, const RhsOperator& op, bool limiting) {
  const CoefficientArray& u = state.coeffs;
  const size_t n = u.data.size();
  auto axpy = [&](const CoefficientArray& a, double s, const CoefficientArray& b) {
    CoefficientArray r = a;
    for (size_t i = 0; i < n; ++i) r.data[i] = a.data[i] + s * b.data[i];
    return r;
  };
  auto lim = [&](CoefficientArray c) {
    if (limiting) limit(ctx, c);
    return c;
  };
  CoefficientArray k1(u.n_eq, u.n_modes, u.n_elem), k2 = k1, k3 = k1, k4 = k1, s;
  const double t = state.t;
  switch (ctx.options.scheme_id()) {
    case DGB_RK2_MIDPOINT:
      op(u, t, k1);
      s = lim(axpy(u, 0.5 * dt, k1));
      op(s, t + 0.5 * dt, k2);
      s = axpy(u, dt, k2);
      break;
    case DGB_RK4_CLASSIC:
      op(u, t, k1);
      s = lim(axpy(u, 0.5 * dt, k1));
      op(s, t + 0.5 * dt, k2);
      s = lim(axpy(u, 0.5 * dt, k2));
      op(s, t + 0.5 * dt, k3);
      s = lim(axpy(u, dt, k3));
      op(s, t + dt, k4);
      for (size_t i = 0; i < n; ++i)
        s.data[i] = u.data[i] + dt / 6.0 * (k1.data[i] + 2.0 * k2.data[i] + 2.0 * k3.data[i] + k4.data[i]);
      break;
    case DGB_SSP_RK2: {
      op(u, t, k1);
      const CoefficientArray s1 = lim(axpy(u, dt, k1));
      op(s1, t + dt, k2);
      s = s1;
      for (size_t i = 0; i < n; ++i) s.data[i] = 0.5 * u.data[i] + 0.5 * s1.data[i] + 0.5 * dt * k2.data[i];
      break;
    }
    case DGB_SSP_RK3: {
      op(u, t, k1);
      const CoefficientArray s1 = lim(axpy(u, dt, k1));
      op(s1, t + dt, k2);
      CoefficientArray s2 = s1;
      for (size_t i = 0; i < n; ++i) s2.data[i] = 0.75 * u.data[i] + 0.25 * s1.data[i] + 0.25 * dt * k2.data[i];
      s2 = lim(s2);
      op(s2, t + 0.5 * dt, k3);
      s = s2;
      for (size_t i = 0; i < n; ++i)
        s.data[i] = (1.0 / 3.0) * u.data[i] + (2.0 / 3.0) * s2.data[i] + (2.0 / 3.0) * dt * k3.data[i];
      break;
    }
    default:
      throw std::invalid_argument("rk_order must be 2 or 4");
  }
  s = lim(s);
  double res = 0.0;
  for (size_t i = 0; i < n; ++i) res = std::max(res, std::fabs(u.data[i] - s.data[i]));
  state.coeffs = std::move(s);
  state.t += dt;
  ++state.step_count;
  return res;
}

namespace detail {
// The drivers for time-dependent Dirichlet data: the reference's own step loop (solver.cpp:559-613)
// on the host — stable_dt, the stage-time tables, one device step — the state on the device.
inline std::pair<std::int64_t, double> host_stepped(const SolverContext& ctx, SolverState& state,
                                                    std::int64_t max_steps, const double* t_end, const double* tol,
                                                    const std::function<void(std::int64_t, double)>& on_step) {
  push_state(ctx, state);
  std::int64_t steps = 0;
  double residual = 0.0, t = state.t;
  std::int64_t sc = state.step_count;
  int rc = DGB_OK;
  while (rc == DGB_OK && steps < max_steps && (!t_end || t < *t_end)) {
    double dt = 0.0;
    rc = dgb_stable_dt(ctx.handle(), DGB_SLOT_STATE, ctx.options.cfl, &dt);
    if (rc != DGB_OK) break;
    if (t_end && t + dt > *t_end) dt = *t_end - t;
    ctx.stage_bc(t, dt);
    rc = dgb_rk_step(ctx.handle(), ctx.options.scheme_id(), dt, ctx.options.limiting ? 1 : 0, &residual);
    if (rc != DGB_OK) break;
    ++steps;
    dgb_get_time(ctx.handle(), &t, &sc);
    if (on_step) on_step(steps, residual);
    if (tol && residual <= *tol) break;
  }
  pull_state(ctx, state);
  check(rc);
  return {steps, residual};
}

inline void replay(const std::function<void(std::int64_t, double)>& on_step, const std::vector<double>& hist,
                   std::int64_t steps) {
  if (!on_step) return;
  for (std::int64_t s = 0; s < steps && s < static_cast<std::int64_t>(hist.size()); ++s) on_step(s + 1, hist[s]);
}
}  // namespace detail

// solver.cpp:559-579
inline SteadyResult run_to_steady(const SolverContext& ctx, SolverState& state, double tol, std::int64_t max_steps,
                                  const std::function<void(std::int64_t, double)>& on_step = {}) {
  if (ctx.time_dependent()) {
    const auto o = detail::host_stepped(ctx, state, max_steps, nullptr, &tol, on_step);
    return SteadyResult{o.first, o.second, o.first > 0 && o.second <= tol};
  }
  detail::push_state(ctx, state);
  SteadyResult r;
  int conv = 0;
  std::vector<double> hist(on_step ? static_cast<size_t>(std::max<std::int64_t>(max_steps, 1)) : 0);
  const int rc = dgb_run_to_steady(ctx.handle(), ctx.options.scheme_id(), ctx.options.cfl,
                                   ctx.options.limiting ? 1 : 0, tol, max_steps, &r.steps, &r.residual, &conv,
                                   hist.empty() ? nullptr : hist.data(), static_cast<std::int64_t>(hist.size()));
  detail::pull_state(ctx, state);
  detail::check(rc);
  r.converged = conv != 0;
  detail::replay(on_step, hist, r.steps);
  return r;
}

// solver.cpp:581-598
inline double run_to_time(const SolverContext& ctx, SolverState& state, double t_end, std::int64_t max_steps,
                          const std::function<void(std::int64_t, double)>& on_step = {}) {
  if (ctx.time_dependent()) {
    const auto o = detail::host_stepped(ctx, state, max_steps, &t_end, nullptr, on_step);
    if (state.t < t_end) throw SolverAbort("t_end not reached within " + std::to_string(max_steps) + " steps");
    return o.second;
  }
  detail::push_state(ctx, state);
  double res = 0.0;
  std::int64_t steps = 0;
  std::vector<double> hist(on_step ? static_cast<size_t>(std::max<std::int64_t>(max_steps, 1)) : 0);
  const int rc = dgb_run_to_time(ctx.handle(), ctx.options.scheme_id(), ctx.options.cfl,
                                 ctx.options.limiting ? 1 : 0, t_end, max_steps, &res, &steps,
                                 hist.empty() ? nullptr : hist.data(), static_cast<std::int64_t>(hist.size()));
  detail::pull_state(ctx, state);
  detail::check(rc);
  detail::replay(on_step, hist, steps);
  return res;
}

// solver.cpp:600-613
inline double run_fixed_steps(const SolverContext& ctx, SolverState& state, std::int64_t n_steps,
                              const std::function<void(std::int64_t, double)>& on_step = {}) {
  if (ctx.time_dependent()) return detail::host_stepped(ctx, state, n_steps, nullptr, nullptr, on_step).second;
  detail::push_state(ctx, state);
  double res = 0.0;
  std::vector<double> hist(static_cast<size_t>(std::max<std::int64_t>(n_steps, 1)));
  const int rc = dgb_run_fixed_steps(ctx.handle(), ctx.options.scheme_id(), ctx.options.cfl,
                                     ctx.options.limiting ? 1 : 0, n_steps, &res, hist.data());
  detail::pull_state(ctx, state);
  detail::check(rc);
  detail::replay(on_step, hist, n_steps);
  return res;
}

// solver.cpp:615-660 — little-endian DG2DCKP1
inline void save_checkpoint(const SolverState& s, const std::string& path) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open checkpoint file '" + path + "'");
  const std::int32_t m = s.coeffs.n_eq, np = s.coeffs.n_modes;
  const std::int64_t n = s.coeffs.n_elem, step = s.step_count;
  f.write("DG2DCKP1", 8);
  f.write(reinterpret_cast<const char*>(&m), 4);
  f.write(reinterpret_cast<const char*>(&np), 4);
  f.write(reinterpret_cast<const char*>(&n), 8);
  f.write(reinterpret_cast<const char*>(&s.t), 8);
  f.write(reinterpret_cast<const char*>(&step), 8);
  f.write(reinterpret_cast<const char*>(s.coeffs.data.data()), static_cast<std::streamsize>(8 * s.coeffs.data.size()));
}

inline SolverState load_checkpoint(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot open checkpoint file '" + path + "'");
  char magic[8];
  f.read(magic, 8);
  if (!f || std::memcmp(magic, "DG2DCKP1", 8) != 0) throw std::runtime_error("'" + path + "' is not a dg2d checkpoint");
  std::int32_t m = 0, np = 0;
  std::int64_t n = 0, step = 0;
  double t = 0.0;
  f.read(reinterpret_cast<char*>(&m), 4);
  f.read(reinterpret_cast<char*>(&np), 4);
  f.read(reinterpret_cast<char*>(&n), 8);
  f.read(reinterpret_cast<char*>(&t), 8);
  f.read(reinterpret_cast<char*>(&step), 8);
  if (!f || m <= 0 || np <= 0 || n <= 0) throw std::runtime_error("corrupt checkpoint header in '" + path + "'");
  SolverState s;
  s.coeffs = CoefficientArray(m, np, static_cast<int>(n));
  f.read(reinterpret_cast<char*>(s.coeffs.data.data()), static_cast<std::streamsize>(8 * s.coeffs.data.size()));
  if (!f) throw std::runtime_error("truncated checkpoint '" + path + "'");
  s.t = t;
  s.step_count = step;
  return s;
}

// output.cpp:30-65 — legacy VTK with 3 corner points per cell (corner states evaluated on the device)
inline void export_vtk(const SolverContext& ctx, const CoefficientArray& coeffs, const std::string& path) {
  const Mesh& mesh = *ctx.mesh;
  const BasisTables& tb = *ctx.tables;
  const int n = mesh.n_elements();
  std::vector<double> phic(3 * static_cast<size_t>(tb.n_p)), st(12 * static_cast<size_t>(n));
  const double corner[3][2] = {{0.0, 0.0}, {1.0, 0.0}, {0.0, 1.0}};
  for (int c = 0; c < 3; ++c)
    for (int j = 0; j < tb.n_p; ++j)
      detail::check(dgb_eval_basis(tb.p, j, corner[c][0], corner[c][1], &phic[c * tb.n_p + j], nullptr, nullptr));
  detail::upload(ctx, DGB_SLOT_INPUT, coeffs);
  detail::check(dgb_corner_states(ctx.handle(), DGB_SLOT_INPUT, phic.data(), st.data()));
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open output file '" + path + "'");
  out.precision(12);
  out << "# vtk DataFile Version 3.0\ndg2d solution\nASCII\nDATASET UNSTRUCTURED_GRID\n";
  out << "POINTS " << 3 * n << " double\n";
  for (int i = 0; i < n; ++i)
    for (int c = 0; c < 3; ++c) {
      const Vec2 v = mesh.vertex_of(i, c);
      out << v.x << ' ' << v.y << " 0\n";
    }
  out << "CELLS " << n << ' ' << 4 * n << "\n";
  for (int i = 0; i < n; ++i) out << "3 " << 3 * i << ' ' << 3 * i + 1 << ' ' << 3 * i + 2 << "\n";
  out << "CELL_TYPES " << n << "\n";
  for (int i = 0; i < n; ++i) out << "5\n";
  out << "POINT_DATA " << 3 * n << "\n";
  const char* names[5] = {"rho", "rho_u", "rho_v", "E", "p"};
  for (int field = 0; field < 5; ++field) {
    out << "SCALARS " << names[field] << " double 1\nLOOKUP_TABLE default\n";
    for (size_t k = 0; k < 3 * static_cast<size_t>(n); ++k) {
      const EulerState u{st[4 * k], st[4 * k + 1], st[4 * k + 2], st[4 * k + 3]};
      out << (field < kEq ? u[field] : pressure(u, ctx.gas)) << "\n";
    }
  }
  if (!out) throw std::runtime_error("failed writing '" + path + "'");
}

// output.cpp:67-81 — one row per cell: centroid, cell means, pressure
inline void export_csv(const SolverContext& ctx, const CoefficientArray& coeffs, const std::string& path) {
  const Mesh& mesh = *ctx.mesh;
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot open output file '" + path + "'");
  out.precision(12);
  const double sqrt2 = std::sqrt(2.0);
  out << "x,y,rho,rho_u,rho_v,E,p\n";
  for (int i = 0; i < mesh.n_elements(); ++i) {
    const Vec2 a = mesh.vertex_of(i, 0), b = mesh.vertex_of(i, 1), c = mesh.vertex_of(i, 2);
    const double cx = (1.0 / 3.0) * (a.x + b.x + c.x), cy = (1.0 / 3.0) * (a.y + b.y + c.y);
    EulerState mean;
    for (int m = 0; m < kEq; ++m) mean[m] = coeffs.at(m, 0, i) * sqrt2;
    out << cx << ',' << cy << ',' << mean.rho << ',' << mean.mx << ',' << mean.my << ',' << mean.E << ','
        << pressure(mean, ctx.gas) << "\n";
  }
  if (!out) throw std::runtime_error("failed writing '" + path + "'");
}

// solver.cpp:662-678 — deterministic host reductions
inline double total_mass(const Mesh& mesh, const CoefficientArray& c) {
  const double inv_sqrt2 = 1.0 / std::sqrt(2.0);
  double s = 0.0;
  for (int i = 0; i < mesh.n_elements(); ++i) s += mesh.det_jac(i) * c.at(0, 0, i) * inv_sqrt2;
  return s;
}

inline double max_abs_diff(const CoefficientArray& a, const CoefficientArray& b) {
  double d = 0.0;
  for (size_t i = 0; i < a.data.size(); ++i) d = std::max(d, std::fabs(a.data[i] - b.data[i]));
  return d;
}

}  // namespace dg2d_b200
