// C++ parity harness: the reference solver (namespace dg2d, compiled from its own
// sources into oracle/_ref/libdg2dref.so) and the B200 path through the C++ mirror
// header dg2d_b200/dg2d.hpp, called side by side with the same names — the way a
// maintainer of the reference would use the drop-in.  TEST INFRASTRUCTURE ONLY.
//
// Cases follow the reference's own tests (proj/tests/test_solver.cpp,
// test_limiter.cpp, test_mesh.cpp, acceptance.cpp); the bars are the north star's:
// per RHS term-scale relative error <= 1e-12, per run relative <= 1e-9.
// Build: oracle/Makefile target `cpptest` -> oracle/_ref/parity_cpp; run by
// tests/test_cpp_api.py (GPU) — prints one line per case and exits non-zero on failure.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <sstream>
#include <string>

#include <fstream>

#include "dg2d/mesh.hpp"
#include "dg2d/output.hpp"
#include "dg2d/problems.hpp"
#include "dg2d/solver.hpp"
#include "dg2d_b200/dg2d.hpp"

namespace R = dg2d;
namespace B = dg2d_b200;

static int g_fail = 0;
#define CHECK(cond, ...)                     \
  do {                                       \
    if (!(cond)) {                           \
      std::printf("  FAIL %s: ", #cond);     \
      std::printf(__VA_ARGS__);              \
      std::printf("\n");                     \
      ++g_fail;                              \
    }                                        \
  } while (0)

// acceptance.cpp:41-49 style smooth admissible field
static R::EulerState smooth(R::Vec2 x, int seed) {
  const double a1 = 0.7 + 0.13 * (seed % 7), a2 = 1.1 + 0.09 * (seed % 5), ph = 0.31 * (seed % 11);
  const double s1 = std::sin(a1 * x.x + a2 * x.y + ph), s2 = std::sin(a2 * x.x - a1 * x.y + 2 * ph);
  const double rho = 1.0 + 0.22 * s1, u = 0.3 * s2, v = 0.25 * s1, p = 1.0 + 0.2 * s2;
  return {rho, rho * u, rho * v, p / 0.4 + 0.5 * rho * (u * u + v * v)};
}

static B::CoefficientArray to_b(const R::CoefficientArray& c) {
  B::CoefficientArray o(c.n_eq, c.n_modes, c.n_elem);
  o.data = c.data;
  return o;
}

// per-equation max |a-b| / max scale
static double rel(const std::vector<double>& a, const std::vector<double>& b, const std::vector<double>& scale, int np,
                  int n) {
  double worst = 0.0;
  for (int m = 0; m < 4; ++m) {
    double d = 0.0, s = 0.0;
    for (size_t k = static_cast<size_t>(m) * np * n; k < static_cast<size_t>(m + 1) * np * n; ++k) {
      d = std::max(d, std::fabs(a[k] - b[k]));
      s = std::max(s, std::fabs(scale[k]));
    }
    worst = std::max(worst, d / std::max(s, 1e-300));
  }
  return worst;
}

struct Pair {
  R::Mesh rm;
  B::Mesh bm;
};

static Pair meshes(const std::string& text) { return {R::build_connectivity(R::parse_msh(text)), B::build_connectivity(B::parse_msh(text))}; }

static void case_connectivity() {
  std::printf("connectivity (test_mesh.cpp:247-255, mesh.cpp:308-313)\n");
  for (const std::string& text : {B::gen_vortex_msh(1), B::gen_double_mach_msh(24, 6), B::gen_box_msh(7, 5, 2.0, 3.0, 1)}) {
    Pair p = meshes(text);
    std::ostringstream os;
    R::dump_edges(p.rm, os);
    CHECK(os.str() == p.bm.dump_edges(), "edge dumps differ");
    CHECK(p.rm.n_elements() == p.bm.n_elements() && p.rm.n_edges() == p.bm.n_edges(), "counts differ");
  }
}

static void case_rhs(int p, int seed) {
  Pair m = meshes(B::gen_vortex_msh(1));
  const R::BasisTables rt = R::build_tables(p);
  const B::BasisTables bt = B::build_tables(p);
  const R::GasModel gas;
  const R::BoundaryConditions rbc = R::vortex_boundary(R::VortexGeometry{}, gas);
  const B::BoundaryConditions bbc = B::vortex_boundary(B::VortexGeometry{}, B::GasModel{});
  R::CoefficientArray c = R::project_initial([&](R::Vec2 x) { return smooth(x, seed); }, m.rm, rt, gas);
  R::SolverContext rc{&m.rm, &rt, gas, &rbc, {}, {}};
  B::SolverContext bc;
  bc.mesh = &m.bm;
  bc.tables = &bt;
  bc.bc = &bbc;
  R::RhsBuffers rb(4, rt.n_p, m.rm.n_elements());
  R::CoefficientArray rd(4, rt.n_p, m.rm.n_elements());
  R::compute_rhs(rc, c, 0.0, rb, rd);
  B::RhsBuffers bb;
  B::CoefficientArray bd;
  B::compute_rhs(bc, to_b(c), 0.0, bb, bd);
  // term scale: (|vol| + sum_q |slot_q|) / detJ
  const int n = m.rm.n_elements(), np = rt.n_p;
  std::vector<double> scale(rd.data.size());
  for (int mm = 0; mm < 4; ++mm)
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < n; ++i) {
        double s = std::fabs(rb.volume.at(mm, j, i));
        for (int q = 0; q < 3; ++q) s += std::fabs(rb.surface_left[rb.slot(q, mm, j, i)]) + std::fabs(rb.surface_right[rb.slot(q, mm, j, i)]);
        scale[rd.idx(mm, j, i)] = s / m.rm.elements[i].det_jac;
      }
  const double e = rel(bd.data, rd.data, scale, np, n);
  std::printf("compute_rhs p=%d seed=%d: term-scale rel err %.2e\n", p, seed, e);
  CHECK(e <= 1e-12, "p=%d rhs parity %.3e", p, e);
  // pass-level: volume
  R::CoefficientArray rv(4, np, n);
  R::eval_volume_pass(rc, c, rv);
  B::CoefficientArray bv;
  B::eval_volume_pass(bc, to_b(c), bv);
  std::vector<double> vs(rv.data.size());
  for (size_t k = 0; k < vs.size(); ++k) vs[k] = std::fabs(rv.data[k]);
  CHECK(rel(bv.data, rv.data, vs, np, n) <= 1e-12, "volume pass");
}

static void case_run(int p, int rk_order, bool dmr, int steps) {
  const std::string text = dmr ? B::gen_double_mach_msh(40, 10) : B::gen_vortex_msh(1);
  Pair m = meshes(text);
  const R::BasisTables rt = R::build_tables(p);
  const B::BasisTables bt = B::build_tables(p);
  const R::GasModel gas;
  R::DoubleMachSetup rsu;
  B::DoubleMachSetup bsu;
  const R::BoundaryConditions rbc = dmr ? R::double_mach_boundary(rsu, gas) : R::vortex_boundary({}, gas);
  const B::BoundaryConditions bbc = dmr ? B::double_mach_boundary(bsu, {}) : B::vortex_boundary({}, {});
  R::SolverContext rc{&m.rm, &rt, gas, &rbc, {rk_order, 0.3, dmr, 0, 256}, {}};
  B::SolverContext bc;
  bc.mesh = &m.bm;
  bc.tables = &bt;
  bc.bc = &bbc;
  bc.options.rk_order = rk_order;
  bc.options.cfl = 0.3;
  bc.options.limiting = dmr;
  R::SolverState rs;
  rs.coeffs = dmr ? R::project_initial([&](R::Vec2 x) { return R::double_mach_initial(x, rsu); }, m.rm, rt, gas)
                  : R::project_initial([&](R::Vec2 x) { return R::vortex_exact(x, {}, gas); }, m.rm, rt, gas);
  if (dmr) R::limit(rc, rs.coeffs);  // runner.cpp:177
  B::SolverState bs;
  bs.coeffs = to_b(rs.coeffs);
  int64_t seen = 0;
  const double rr = R::run_fixed_steps(rc, rs, steps);
  const double br = B::run_fixed_steps(bc, bs, steps, [&](int64_t, double) { ++seen; });
  std::vector<double> scale(rs.coeffs.data.size());
  for (size_t k = 0; k < scale.size(); ++k) scale[k] = std::fabs(rs.coeffs.data[k]);
  const double e = rel(bs.coeffs.data, rs.coeffs.data, scale, rt.n_p, m.rm.n_elements());
  std::printf("run_fixed_steps %s p=%d rk%d x%d: rel err %.2e, t %.17g vs %.17g, residual %.3e vs %.3e\n",
              dmr ? "DMR+limiter" : "vortex", p, rk_order, steps, e, bs.t, rs.t, br, rr);
  CHECK(e <= 1e-9, "run parity %.3e", e);
  CHECK(std::fabs(bs.t - rs.t) <= 1e-12 * rs.t && bs.step_count == rs.step_count, "time/steps");
  CHECK(seen == steps, "on_step calls %ld", static_cast<long>(seen));
  const double mr = R::total_mass(m.rm, rs.coeffs), mb = B::total_mass(m.bm, bs.coeffs);
  CHECK(std::fabs(mr - mb) <= 1e-12 * std::fabs(mr), "mass");
}

// Time-dependent Dirichlet data: the reference evaluates its closure at every stage time inside
// run_fixed_steps (solver.cpp:198-211); the mirror's drivers give the device one table per stage.
static void case_time_dependent_bc(int p, int rk_order, int steps) {
  Pair m = meshes(B::gen_vortex_msh(1));
  const R::BasisTables rt = R::build_tables(p);
  const B::BasisTables bt = B::build_tables(p);
  const R::GasModel gas;
  R::BoundaryConditions rbc = R::vortex_boundary({}, gas);
  B::BoundaryConditions bbc = B::vortex_boundary({}, {});
  auto scaled = [](auto s, double t) {
    const double f = 1.0 + 0.05 * std::sin(40.0 * t);
    for (int k = 0; k < 4; ++k) s[k] *= f;
    return s;
  };
  const auto r0 = rbc.dirichlet;
  const auto b0 = bbc.dirichlet;
  rbc.dirichlet = [r0, scaled](R::Vec2 x, double t) { return scaled(r0(x, t), t); };
  bbc.dirichlet = [b0, scaled](B::Vec2 x, double t) { return scaled(b0(x, t), t); };
  bbc.time_dependent = true;
  R::SolverContext rc{&m.rm, &rt, gas, &rbc, {rk_order, 0.3, false, 0, 256}, {}};
  B::SolverContext bc;
  bc.mesh = &m.bm;
  bc.tables = &bt;
  bc.bc = &bbc;
  bc.options.rk_order = rk_order;
  bc.options.cfl = 0.3;
  R::SolverState rs;
  rs.coeffs = R::project_initial([&](R::Vec2 x) { return R::vortex_exact(x, {}, gas); }, m.rm, rt, gas);
  B::SolverState bs;
  bs.coeffs = to_b(rs.coeffs);
  const double rr = R::run_fixed_steps(rc, rs, steps);
  const double br = B::run_fixed_steps(bc, bs, steps);
  std::vector<double> scale(rs.coeffs.data.size());
  for (size_t k = 0; k < scale.size(); ++k) scale[k] = std::fabs(rs.coeffs.data[k]);
  const double e = rel(bs.coeffs.data, rs.coeffs.data, scale, rt.n_p, m.rm.n_elements());
  std::printf("time-dependent Dirichlet p=%d rk%d x%d: rel err %.2e, t %.17g vs %.17g, residual %.3e vs %.3e\n", p,
              rk_order, steps, e, bs.t, rs.t, br, rr);
  CHECK(e <= 1e-9, "time-dependent BC run parity %.3e", e);
  CHECK(std::fabs(bs.t - rs.t) <= 1e-12 * rs.t && bs.step_count == rs.step_count, "time/steps");
}

static void case_errors() {
  std::printf("error behaviour (test_limiter.cpp:170-175, test_solver.cpp:413-422, 504-512)\n");
  Pair m = meshes(B::gen_vortex_msh(0));
  const B::BasisTables bt2 = B::build_tables(2);
  const B::BoundaryConditions bbc = B::vortex_boundary({}, {});
  B::SolverContext bc;
  bc.mesh = &m.bm;
  bc.tables = &bt2;
  bc.bc = &bbc;
  B::CoefficientArray c(4, bt2.n_p, m.bm.n_elements());
  bool threw = false;
  try {
    B::limit(bc, c);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw, "limit at p=2 must throw std::invalid_argument");
  // inadmissible state -> SolverAbort with the reference's message shape
  const R::BasisTables rt = R::build_tables(2);
  const R::BoundaryConditions rbc = R::vortex_boundary({}, {});
  R::SolverContext rc{&m.rm, &rt, {}, &rbc, {}, {}};
  R::CoefficientArray rcf = R::project_initial([&](R::Vec2 x) { return R::vortex_exact(x, {}, {}); }, m.rm, rt, {});
  for (int j = 0; j < rt.n_p; ++j) rcf.at(0, j, 7) = -1.0;  // negative density in element 7
  std::string rmsg, bmsg;
  try {
    R::RhsBuffers rb(4, rt.n_p, m.rm.n_elements());
    R::CoefficientArray d(4, rt.n_p, m.rm.n_elements());
    R::compute_rhs(rc, rcf, 0.0, rb, d);
  } catch (const R::SolverAbort& e) {
    rmsg = e.what();
  }
  try {
    B::RhsBuffers bb;
    B::CoefficientArray d;
    B::compute_rhs(bc, to_b(rcf), 0.0, bb, d);
  } catch (const B::SolverAbort& e) {
    bmsg = e.what();
  }
  std::printf("  reference: %s\n  b200:      %s\n", rmsg.c_str(), bmsg.c_str());
  CHECK(!rmsg.empty() && rmsg == bmsg, "SolverAbort messages differ");
  B::SolverState st;
  st.coeffs = to_b(rcf);
  bc.options.rk_order = 3;
  threw = false;
  try {
    B::rk_step(bc, st, 1e-3);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw, "rk_order 3 must throw std::invalid_argument");
}

static void case_operator_seam_and_checkpoint() {
  std::printf("RhsOperator seam (test_solver.cpp:351-385) and DG2DCKP1 checkpoints (solver.cpp:615-660)\n");
  Pair m = meshes(B::gen_vortex_msh(1));
  const B::BasisTables bt = B::build_tables(3);
  const B::BoundaryConditions bbc = B::vortex_boundary({}, {});
  B::SolverContext bc;
  bc.mesh = &m.bm;
  bc.tables = &bt;
  bc.bc = &bbc;
  B::SolverState a;
  a.coeffs = B::project_initial([](B::Vec2 x) { return B::vortex_exact(x, {}, {}); }, m.bm, bt, {});
  B::SolverState b = a;
  const double dt = B::stable_dt(bc, a.coeffs);
  B::rk_step(bc, a, dt);
  B::RhsOperator op = [&](const B::CoefficientArray& c, double t, B::CoefficientArray& d) {
    B::RhsBuffers bb;
    B::compute_rhs(bc, c, t, bb, d);
  };
  B::rk_step(bc, b, dt, op, false);
  std::vector<double> sc(a.coeffs.data.size());
  for (size_t k = 0; k < sc.size(); ++k) sc[k] = std::fabs(a.coeffs.data[k]);
  const double e = rel(b.coeffs.data, a.coeffs.data, sc, bt.n_p, m.bm.n_elements());
  std::printf("  device rk_step vs host stages around the operator: %.2e\n", e);
  CHECK(e <= 1e-13, "operator seam %.3e", e);
  const std::string path = "/tmp/dg2d_b200_ckpt_test.bin";
  B::save_checkpoint(a, path);
  const R::SolverState r = R::load_checkpoint(path);  // the reference reads our file
  CHECK(r.coeffs.data == a.coeffs.data && r.t == a.t && r.step_count == a.step_count, "checkpoint format");
  const B::SolverState back = B::load_checkpoint(path);
  CHECK(back.coeffs.data == a.coeffs.data, "checkpoint round trip");
}

static bool files_match(const std::string& a, const std::string& b) {
  std::ifstream fa(a), fb(b);
  std::string ta, tb;
  while (true) {
    const bool ra = static_cast<bool>(fa >> ta), rb = static_cast<bool>(fb >> tb);
    if (ra != rb) return false;
    if (!ra) return true;
    if (ta == tb) continue;
    char* ea = nullptr;
    char* eb = nullptr;
    const double va = std::strtod(ta.c_str(), &ea), vb = std::strtod(tb.c_str(), &eb);
    if (*ea || *eb) return false;  // differing non-numeric tokens
    if (std::fabs(va - vb) > 1e-11 * std::fabs(vb)) return false;
  }
}

static void case_output() {
  std::printf("export_vtk / export_csv (output.cpp:30-81)\n");
  Pair m = meshes(B::gen_vortex_msh(1));
  const R::BasisTables rt = R::build_tables(2);
  const B::BasisTables bt = B::build_tables(2);
  const B::BoundaryConditions bbc = B::vortex_boundary({}, {});
  B::SolverContext bc;
  bc.mesh = &m.bm;
  bc.tables = &bt;
  bc.bc = &bbc;
  R::CoefficientArray c = R::project_initial([](R::Vec2 x) { return R::vortex_exact(x, {}, {}); }, m.rm, rt, {});
  R::export_vtk(c, m.rm, rt, {}, "/tmp/dg2d_b200_ref.vtk");
  R::export_csv(c, m.rm, rt, {}, "/tmp/dg2d_b200_ref.csv");
  B::export_vtk(bc, to_b(c), "/tmp/dg2d_b200_ours.vtk");
  B::export_csv(bc, to_b(c), "/tmp/dg2d_b200_ours.csv");
  CHECK(files_match("/tmp/dg2d_b200_ours.vtk", "/tmp/dg2d_b200_ref.vtk"), "vtk files differ");
  CHECK(files_match("/tmp/dg2d_b200_ours.csv", "/tmp/dg2d_b200_ref.csv"), "csv files differ");
}

int main() {
  case_connectivity();
  for (int p = 1; p <= 5; ++p) case_rhs(p, 3 + p);
  case_run(2, 4, false, 20);
  case_run(4, 2, false, 10);
  case_run(1, 2, true, 30);
  case_time_dependent_bc(2, 4, 12);
  case_time_dependent_bc(3, 2, 12);
  case_errors();
  case_operator_seam_and_checkpoint();
  case_output();
  std::printf(g_fail ? "FAILED %d check(s)\n" : "ALL PASSED\n", g_fail);
  return g_fail ? 1 : 0;
}
