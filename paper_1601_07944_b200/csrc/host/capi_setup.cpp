// C ABI of the host-side setup (mesh, tables, problem data).  These entry
// points are not the hot path; they exist so a caller without the reference's
// C++ objects (Python tests, bench.py, other FFIs) can produce the same mesh,
// tables and boundary data the reference would.
#include <cmath>
#include <cstring>
#include <new>
#include <string>

#include "../../../include/dg2d_b200/dg2d_b200.h"
#include "capi_common.hpp"
#include "setup.hpp"

struct dgb_mesh {
  dgb::Mesh m;
};
struct dgb_tables {
  dgb::Tables t;
};

namespace dgb {
thread_local std::string g_last_message;
void set_message(const std::string& s) { g_last_message = s; }
}  // namespace dgb

extern "C" const char* dgb_last_message(void) { return dgb::g_last_message.c_str(); }

namespace {

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const dgb::MeshError& e) {
    dgb::set_message(e.what());
    return DGB_ERR_MESH;
  } catch (const std::bad_alloc&) {
    dgb::set_message("out of host memory");
    return DGB_ERR_ARG;
  } catch (const std::exception& e) {
    dgb::set_message(e.what());
    return DGB_ERR_ARG;
  }
}

int copy_text(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf) {
    if (cap < s.size() + 1) {
      dgb::set_message("buffer too small");
      return DGB_ERR_ARG;
    }
    std::memcpy(buf, s.c_str(), s.size() + 1);
  }
  return DGB_OK;
}

}  // namespace

extern "C" {

int dgb_mesh_from_msh(const char* text, size_t len, dgb_mesh** out) {
  return guarded([&] {
    auto* h = new dgb_mesh;
    try {
      h->m = dgb::build_connectivity(dgb::parse_msh(text, len));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return DGB_OK;
  });
}

int dgb_mesh_generate(int kind, int nx, int ny, const double* params, int n_params, dgb_mesh** out) {
  return guarded([&] {
    auto* h = new dgb_mesh;
    try {
      h->m = dgb::build_connectivity(dgb::generate(kind, nx, ny, params, n_params));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return DGB_OK;
  });
}

int dgb_mesh_generate_text(int kind, int nx, int ny, const double* params, int n_params, char* buf,
                           size_t cap, size_t* needed) {
  return guarded([&] {
    return copy_text(dgb::format_msh(dgb::generate(kind, nx, ny, params, n_params)), buf, cap, needed);
  });
}

int dgb_mesh_get_view(const dgb_mesh* h, dgb_mesh_view* v) {
  if (!h || !v) {
    dgb::set_message("null mesh");
    return DGB_ERR_ARG;
  }
  const dgb::Mesh& m = h->m;
  v->n_vertices = static_cast<int32_t>(m.vx.size());
  v->vx = m.vx.data();
  v->vy = m.vy.data();
  v->n_elements = m.n_elem;
  v->elem_v = m.elem_v.data();
  v->elem_edge = m.elem_edge.data();
  v->det_jac = m.det.data();
  v->tau = m.tau.data();
  v->inradius = m.inradius.data();
  v->n_edges = m.n_edges;
  v->n_boundary_edges = m.n_boundary;
  v->edge_v0 = m.ev0.data();
  v->edge_v1 = m.ev1.data();
  v->edge_left = m.eleft.data();
  v->edge_right = m.eright.data();
  v->edge_side_left = m.eside_l.data();
  v->edge_side_right = m.eside_r.data();
  v->edge_nx = m.enx.data();
  v->edge_ny = m.eny.data();
  v->edge_half_length = m.eh.data();
  return DGB_OK;
}

int dgb_mesh_dump_edges(const dgb_mesh* h, char* buf, size_t cap, size_t* needed) {
  return guarded([&] { return copy_text(dgb::dump_edges(h->m), buf, cap, needed); });
}

void dgb_mesh_free(dgb_mesh* h) { delete h; }

int dgb_tables_build(int p, dgb_tables** out) {
  return guarded([&] {
    auto* h = new dgb_tables;
    try {
      h->t = dgb::build_tables(p);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return DGB_OK;
  });
}

int dgb_tables_get_view(const dgb_tables* h, dgb_tables_view* v) {
  if (!h || !v) {
    dgb::set_message("null tables");
    return DGB_ERR_ARG;
  }
  const dgb::Tables& t = h->t;
  v->p = t.p;
  v->n_p = t.n_p;
  v->n_quad = t.n_quad;
  v->n_edge_pts = t.n_edge_pts;
  v->phi_interior = t.phi_interior.data();
  v->dphi_dr_interior = t.dphi_dr.data();
  v->dphi_ds_interior = t.dphi_ds.data();
  v->w_interior = t.w_interior.data();
  v->r_interior = t.r_interior.data();
  v->phi_edge = t.phi_edge.data();
  v->w_edge = t.w_edge.data();
  v->xi_edge = t.xi_edge.data();
  v->phi_edge_mid = t.phi_edge_mid.data();
  return DGB_OK;
}

void dgb_tables_free(dgb_tables* h) { delete h; }

int dgb_eval_basis(int p, int j, double r, double s, double* phi, double* dr, double* ds) {
  return guarded([&] {
    if (phi) *phi = dgb::eval_basis(p, j, r, s);
    if (dr || ds) {
      double a, b;
      dgb::eval_basis_grad(p, j, r, s, a, b);
      if (dr) *dr = a;
      if (ds) *ds = b;
    }
    return DGB_OK;
  });
}

int dgb_interior_points(const dgb_mesh_view* m, const dgb_tables_view* t, double* xy) {
  const int n = m->n_elements, nq = t->n_quad;
  for (int i = 0; i < n; ++i) {
    const int* v = m->elem_v + 3 * i;
    const double ax = m->vx[v[0]], ay = m->vy[v[0]];
    const double bx = m->vx[v[1]], by = m->vy[v[1]];
    const double cx = m->vx[v[2]], cy = m->vy[v[2]];
    for (int k = 0; k < nq; ++k) {
      const double r = t->r_interior[2 * k], s = t->r_interior[2 * k + 1];
      double* o = xy + 2 * (static_cast<size_t>(i) * nq + k);
      o[0] = ax + r * (bx - ax) + s * (cx - ax);
      o[1] = ay + r * (by - ay) + s * (cy - ay);
    }
  }
  return DGB_OK;
}

int dgb_boundary_points(const dgb_mesh_view* m, const dgb_tables_view* t, double* xy) {
  const int nk = t->n_edge_pts;
  for (int e = 0; e < m->n_boundary_edges; ++e) {
    const double ax = m->vx[m->edge_v0[e]], ay = m->vy[m->edge_v0[e]];
    const double bx = m->vx[m->edge_v1[e]], by = m->vy[m->edge_v1[e]];
    for (int k = 0; k < nk; ++k) {
      const double xi = t->xi_edge[k];
      const double wa = 0.5 * (1.0 - xi), wb = 0.5 * (1.0 + xi);
      double* o = xy + 2 * (static_cast<size_t>(e) * nk + k);
      o[0] = wa * ax + wb * bx;
      o[1] = wa * ay + wb * by;
    }
  }
  return DGB_OK;
}

int dgb_project(const dgb_mesh_view* m, const dgb_tables_view* t, double gamma, const double* ps,
                double* coeffs) {
  const int n = m->n_elements, nq = t->n_quad, np = t->n_p;
  std::memset(coeffs, 0, sizeof(double) * 4 * np * static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < nq; ++k) {
      const double* u = ps + 4 * (static_cast<size_t>(i) * nq + k);
      const double pr = (gamma - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]);
      if (!(u[0] > 0.0 && pr > 0.0)) {
        dgb::set_message("project_initial: inadmissible state at id " + std::to_string(i) + ", point " +
                         std::to_string(k) + " (rho=" + std::to_string(u[0]) + ", p=" + std::to_string(pr) +
                         ")");
        return DGB_ERR_INADMISSIBLE;
      }
      const double w = t->w_interior[k];
      for (int j = 0; j < np; ++j) {
        const double wphi = w * t->phi_interior[k * np + j];
        for (int mm = 0; mm < 4; ++mm) coeffs[(static_cast<size_t>(mm) * np + j) * n + i] += wphi * u[mm];
      }
    }
  }
  return DGB_OK;
}

int dgb_vortex_exact(const double* xy, int64_t n, double r_inner, double r_outer, double mach_inner,
                     double rho_inner, double c_inner, double gamma, double* states) {
  return guarded([&] {
    for (int64_t i = 0; i < n; ++i)
      dgb::vortex_exact(xy[2 * i], xy[2 * i + 1], r_inner, r_outer, mach_inner, rho_inner, c_inner, gamma,
                        states + 4 * i);
    return DGB_OK;
  });
}

int dgb_rankine_hugoniot_post(const double* pre, double mach, double nx, double ny, double gamma,
                              double* post) {
  dgb::rankine_hugoniot_post(pre, mach, nx, ny, gamma, post);
  return DGB_OK;
}

int dgb_isentropic_vortex(const double* xy, int64_t n, double xc, double yc, double beta, double u_inf,
                          double v_inf, double width, double height, double t, double gamma,
                          double* states) {
  for (int64_t i = 0; i < n; ++i)
    dgb::isentropic_vortex(xy[2 * i], xy[2 * i + 1], xc, yc, beta, u_inf, v_inf, width, height, t, gamma,
                           states + 4 * i);
  return DGB_OK;
}

}  // extern "C"
