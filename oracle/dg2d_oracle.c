/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle (see dg2d_oracle.h).  Serial C
 * restatement of the reference hot path; every function names the
 * reference lines it restates.
 */
#include "dg2d_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define EQ 4

typedef struct {
  double u[EQ];
} St;

/* euler.hpp:29-31 */
static double pressure(const double* u, double g) { return (g - 1.0) * (u[3] - 0.5 * (u[1] * u[1] + u[2] * u[2]) / u[0]); }
/* euler.hpp:33-35 */
static int admissible(const double* u, double g) { return u[0] > 0.0 && pressure(u, g) > 0.0; }
/* euler.hpp:43-50 */
static void euler_flux(const double* u, double g, double* f1, double* f2) {
  double inv = 1.0 / u[0], vx = u[1] * inv, vy = u[2] * inv, p = pressure(u, g);
  f1[0] = u[1];
  f1[1] = u[1] * vx + p;
  f1[2] = u[2] * vx;
  f1[3] = vx * (u[3] + p);
  f2[0] = u[2];
  f2[1] = u[1] * vy;
  f2[2] = u[2] * vy + p;
  f2[3] = vy * (u[3] + p);
}
/* euler.hpp:52-55 */
static double wave_speed(const double* u, double nx, double ny, double g) {
  double vn = (u[1] * nx + u[2] * ny) / u[0];
  return fabs(vn) + sqrt(g * pressure(u, g) / u[0]);
}
/* euler.hpp:59-71 (local Lax-Friedrichs) */
static void llf(const double* ul, const double* ur, double nx, double ny, double g, double* f) {
  double f1l[EQ], f2l[EQ], f1r[EQ], f2r[EQ];
  euler_flux(ul, g, f1l, f2l);
  euler_flux(ur, g, f1r, f2r);
  double sl = wave_speed(ul, nx, ny, g), sr = wave_speed(ur, nx, ny, g);
  double s = sl > sr ? sl : sr;
  for (int m = 0; m < EQ; ++m) f[m] = 0.5 * (nx * (f1l[m] + f1r[m]) + ny * (f2l[m] + f2r[m])) - 0.5 * s * (ur[m] - ul[m]);
}
/* Roe flux with Harten's entropy fix on the acoustic waves (delta = 0.1 c~).  NOT in the
 * reference ("Roe is new"; SPEC.md:265 lists it as a non-goal);
 * BASELINE.json's north star asks for "Lax-Friedrichs or Roe".  Restated from Roe (1981),
 * J. Comput. Phys. 43:357-372, in the rotated (normal/tangential) wave decomposition;
 * parity unpinned by the reference, pinned by its defining properties in
 * tests/test_oracle.py (consistency, conservation, rotation, upwinding). */
static void roe(const double* ul, const double* ur, double nx, double ny, double g, double* f) {
  double f1l[EQ], f2l[EQ], f1r[EQ], f2r[EQ];
  euler_flux(ul, g, f1l, f2l);
  euler_flux(ur, g, f1r, f2r);
  const double rl = ul[0], rr = ur[0];
  const double uL = ul[1] / rl, vL = ul[2] / rl, uR = ur[1] / rr, vR = ur[2] / rr;
  const double pL = pressure(ul, g), pR = pressure(ur, g);
  const double HL = (ul[3] + pL) / rl, HR = (ur[3] + pR) / rr;
  const double sl = sqrt(rl), sr = sqrt(rr), isum = 1.0 / (sl + sr);
  const double u = (sl * uL + sr * uR) * isum, v = (sl * vL + sr * vR) * isum, H = (sl * HL + sr * HR) * isum;
  const double q2 = u * u + v * v;
  const double c = sqrt((g - 1.0) * (H - 0.5 * q2)), rho = sl * sr;
  const double qn = u * nx + v * ny;
  const double du = uR - uL, dv = vR - vL, dqn = du * nx + dv * ny;
  const double dut = du - dqn * nx, dvt = dv - dqn * ny; /* tangential velocity jump */
  const double dr = rr - rl, dp = pR - pL;
  const double a1 = (dp - rho * c * dqn) / (2.0 * c * c), a2 = dr - dp / (c * c), a3 = (dp + rho * c * dqn) / (2.0 * c * c);
  double l1 = fabs(qn - c), l2 = fabs(qn), l3 = fabs(qn + c);
  const double d = 0.1 * c;
  if (l1 < d) l1 = (l1 * l1 + d * d) / (2.0 * d);
  if (l3 < d) l3 = (l3 * l3 + d * d) / (2.0 * d);
  double D[EQ];
  D[0] = l1 * a1 + l2 * a2 + l3 * a3;
  D[1] = l1 * a1 * (u - c * nx) + l2 * a2 * u + l3 * a3 * (u + c * nx) + l2 * rho * dut;
  D[2] = l1 * a1 * (v - c * ny) + l2 * a2 * v + l3 * a3 * (v + c * ny) + l2 * rho * dvt;
  D[3] = l1 * a1 * (H - qn * c) + l2 * a2 * 0.5 * q2 + l3 * a3 * (H + qn * c) + l2 * rho * (u * dut + v * dvt);
  for (int m = 0; m < EQ; ++m) f[m] = 0.5 * (nx * (f1l[m] + f1r[m]) + ny * (f2l[m] + f2r[m])) - 0.5 * D[m];
}

static void num_flux(const or_problem* P, const double* ul, const double* ur, double nx, double ny, double* f) {
  if (P->flux == 1)
    roe(ul, ur, nx, ny, P->gamma, f);
  else
    llf(ul, ur, nx, ny, P->gamma, f);
}

/* euler.hpp:75-78 */
static void reflect(const double* u, double nx, double ny, double* g) {
  double mn = 2.0 * (u[1] * nx + u[2] * ny);
  g[0] = u[0];
  g[1] = u[1] - mn * nx;
  g[2] = u[2] - mn * ny;
  g[3] = u[3];
}

static size_t cidx(int np, int n, int m, int j, int i) { return ((size_t)m * np + j) * n + i; }

static void fail_rec(or_fail* f, int pass, int64_t id, int point, const double* u, double g) {
  if (!f) return;
  if (f->pass == 0 || id < f->id) { /* AbortRecord: lowest id wins (solver.cpp:44-55) */
    f->pass = pass;
    f->id = id;
    f->point = point;
    f->rho = u[0];
    f->p = pressure(u, g);
  }
}

/* ghost_state, euler.hpp:118-140, closures as per-point tables */
static int ghost(const or_problem* P, const double* ul, int code, int e, int k, double t, double nx, double ny,
                 double* ur) {
  const dgb_bc_view* bc = P->bc;
  const int K = P->tables->n_edge_pts;
  const size_t pk = (size_t)e * K + k;
  switch (code) {
    case -1:
      reflect(ul, nx, ny, ur);
      return 0;
    case -2:
      if (!bc || !bc->wall_normal) return -1;
      reflect(ul, bc->wall_normal[2 * pk], bc->wall_normal[2 * pk + 1], ur);
      return 0;
    case -3:
      if (bc && bc->dirichlet_state)
        memcpy(ur, bc->dirichlet_state + 4 * pk, 4 * sizeof(double));
      else if (bc)
        memcpy(ur, bc->inflow_state, 4 * sizeof(double));
      else
        memset(ur, 0, 4 * sizeof(double));
      return 0;
    case -4:
      memcpy(ur, ul, 4 * sizeof(double));
      return 0;
    case -5: {
      if (!bc || !bc->has_shock) return -1;
      const dgb_mesh_view* M = P->mesh;
      double xi = P->tables->xi_edge[k];
      int v0 = M->edge_v0[e], v1 = M->edge_v1[e];
      /* solver.cpp:198 */
      double x = 0.5 * (1.0 - xi) * M->vx[v0] + 0.5 * (1.0 + xi) * M->vx[v1];
      double y = 0.5 * (1.0 - xi) * M->vy[v0] + 0.5 * (1.0 + xi) * M->vy[v1];
      double rad = bc->shock_angle_deg * M_PI / 180.0; /* euler.hpp:97-100 */
      double front = bc->shock_x0 + (y * cos(rad) + bc->shock_speed * t) / sin(rad);
      memcpy(ur, x < front ? bc->shock_post : bc->shock_pre, 4 * sizeof(double));
      return 0;
    }
    default:
      return -1;
  }
}

/* eval_volume_pass, solver.cpp:99-158 */
int or_volume(const or_problem* P, const double* c, double* vol, or_fail* f) {
  const dgb_mesh_view* M = P->mesh;
  const dgb_tables_view* T = P->tables;
  const int n = M->n_elements, np = T->n_p, nq = T->n_quad;
  const double g = P->gamma;
  int bad = 0;
  memset(vol, 0, sizeof(double) * EQ * np * (size_t)n);
  for (int i = 0; i < n; ++i) {
    const double* tau = M->tau + 4 * (size_t)i;
    for (int k = 0; k < nq; ++k) {
      double u[EQ];
      for (int m = 0; m < EQ; ++m) {
        double s = 0.0;
        for (int j = 0; j < np; ++j) s += T->phi_interior[k * np + j] * c[cidx(np, n, m, j, i)];
        u[m] = s;
      }
      if (!admissible(u, g)) {
        fail_rec(f, 1, i, k, u, g);
        bad = 1;
        u[0] = 1.0; u[1] = 0.0; u[2] = 0.0; u[3] = 2.5;
      }
      double f1[EQ], f2[EQ];
      euler_flux(u, g, f1, f2);
      const double w = T->w_interior[k];
      for (int j = 0; j < np; ++j) {
        const double gr = T->dphi_dr_interior[k * np + j], gs = T->dphi_ds_interior[k * np + j];
        const double tx = tau[0] * gr + tau[2] * gs, ty = tau[1] * gr + tau[3] * gs;
        for (int m = 0; m < EQ; ++m) vol[cidx(np, n, m, j, i)] += w * (f1[m] * tx + f2[m] * ty);
      }
    }
  }
  return bad;
}

/* eval_surface_pass, solver.cpp:160-251; slots: RhsBuffers::slot (solver.hpp:59-61) */
int or_surface(const or_problem* P, const double* c, double t, double* sl, double* sr, or_fail* f) {
  const dgb_mesh_view* M = P->mesh;
  const dgb_tables_view* T = P->tables;
  const int n = M->n_elements, np = T->n_p, nk = T->n_edge_pts;
  const double g = P->gamma;
  int bad = 0;
  double* accl = malloc(sizeof(double) * EQ * np);
  double* accr = malloc(sizeof(double) * EQ * np);
  for (int e = 0; e < M->n_edges; ++e) {
    const int L = M->edge_left[e], R = M->edge_right[e], bnd = R < 0;
    const int qs = M->edge_side_left[e] - 1, qr = M->edge_side_right[e] - 1;
    const double nx = M->edge_nx[e], ny = M->edge_ny[e], h = M->edge_half_length[e];
    memset(accl, 0, sizeof(double) * EQ * np);
    memset(accr, 0, sizeof(double) * EQ * np);
    for (int k = 0; k < nk; ++k) {
      double ul[EQ], ur[EQ];
      for (int m = 0; m < EQ; ++m) {
        double s = 0.0;
        for (int j = 0; j < np; ++j) s += c[cidx(np, n, m, j, L)] * T->phi_edge[(qs * nk + k) * np + j];
        ul[m] = s;
      }
      const int kr = nk - 1 - k; /* opposite traversal, solver.cpp:213 */
      if (bnd) {
        if (!admissible(ul, g)) {
          fail_rec(f, 2, e, k, ul, g);
          bad = 1;
          continue;
        }
        if (ghost(P, ul, R, e, k, t, nx, ny, ur)) {
          bad = 2;
          continue;
        }
      } else {
        for (int m = 0; m < EQ; ++m) {
          double s = 0.0;
          for (int j = 0; j < np; ++j) s += c[cidx(np, n, m, j, R)] * T->phi_edge[(qr * nk + kr) * np + j];
          ur[m] = s;
        }
      }
      if (!admissible(ul, g) || !admissible(ur, g)) {
        fail_rec(f, 2, e, k, admissible(ul, g) ? ur : ul, g);
        bad = 1;
        continue;
      }
      double fn[EQ];
      num_flux(P, ul, ur, nx, ny, fn);
      const double wl = h * T->w_edge[k];
      for (int j = 0; j < np; ++j) {
        const double pl = T->phi_edge[(qs * nk + k) * np + j];
        for (int m = 0; m < EQ; ++m) accl[m * np + j] -= wl * fn[m] * pl;
        if (!bnd) {
          const double pr = T->phi_edge[(qr * nk + kr) * np + j];
          for (int m = 0; m < EQ; ++m) accr[m * np + j] += wl * fn[m] * pr;
        }
      }
    }
    for (int m = 0; m < EQ; ++m)
      for (int j = 0; j < np; ++j) {
        sl[(((size_t)qs * EQ + m) * np + j) * n + L] = accl[m * np + j];
        if (!bnd) sr[(((size_t)qr * EQ + m) * np + j) * n + R] = accr[m * np + j];
      }
  }
  free(accl);
  free(accr);
  return bad;
}

/* eval_rhs_pass, solver.cpp:253-277 */
void or_gather(const or_problem* P, const double* vol, const double* sl, const double* sr, double* deriv) {
  const dgb_mesh_view* M = P->mesh;
  const int n = M->n_elements, np = P->tables->n_p;
  for (int i = 0; i < n; ++i) {
    const double inv_det = 1.0 / M->det_jac[i];
    int from_left[3];
    for (int q = 0; q < 3; ++q) from_left[q] = M->edge_left[M->elem_edge[3 * i + q]] == i;
    for (int m = 0; m < EQ; ++m)
      for (int j = 0; j < np; ++j) {
        double acc = vol[cidx(np, n, m, j, i)];
        for (int q = 0; q < 3; ++q) {
          const size_t s = (((size_t)q * EQ + m) * np + j) * n + i;
          acc += from_left[q] ? sl[s] : sr[s];
        }
        deriv[cidx(np, n, m, j, i)] = acc * inv_det;
      }
  }
}

/* compute_rhs, solver.cpp:279-284 (volume failures are reported first) */
int or_rhs(const or_problem* P, const double* c, double t, double* deriv, or_fail* f) {
  const size_t sz = (size_t)EQ * P->tables->n_p * P->mesh->n_elements;
  double* vol = malloc(sizeof(double) * sz);
  double* sl = calloc(3 * sz, sizeof(double));
  double* sr = calloc(3 * sz, sizeof(double));
  int rc = or_volume(P, c, vol, f);
  if (!rc) rc = or_surface(P, c, t, sl, sr, f);
  if (!rc) or_gather(P, vol, sl, sr, deriv);
  free(vol);
  free(sl);
  free(sr);
  return rc;
}

static double clamp01(double a) { return a < 0.0 ? 0.0 : (a > 1.0 ? 1.0 : a); }

/* limit, solver.cpp:286-425 (Barth-Jespersen + positivity guard), p = 1 */
int or_limit(const or_problem* P, double* c) {
  const dgb_mesh_view* M = P->mesh;
  const dgb_tables_view* T = P->tables;
  if (T->p != 1) return -1;
  const int n = M->n_elements, nk = T->n_edge_pts, np = 3;
  const double sqrt2 = sqrt(2.0), g = P->gamma;
  double phi1[64], phi2[64], max1 = 0.0, max2 = 0.0;
  int idx = 0;
  for (int k = 0; k < T->n_quad; ++k, ++idx) {
    phi1[idx] = T->phi_interior[k * np + 1];
    phi2[idx] = T->phi_interior[k * np + 2];
  }
  for (int q = 0; q < 3; ++q)
    for (int k = 0; k < nk; ++k, ++idx) {
      phi1[idx] = T->phi_edge[(q * nk + k) * np + 1];
      phi2[idx] = T->phi_edge[(q * nk + k) * np + 2];
    }
  for (int q = 0; q < 3; ++q, ++idx) {
    phi1[idx] = T->phi_edge_mid[q * np + 1];
    phi2[idx] = T->phi_edge_mid[q * np + 2];
  }
  const int n_pts = idx, eb = T->n_quad;
  for (int k = 0; k < n_pts; ++k) {
    if (fabs(phi1[k]) > max1) max1 = fabs(phi1[k]);
    if (fabs(phi2[k]) > max2) max2 = fabs(phi2[k]);
  }
  for (int i = 0; i < n; ++i) {
    double c0[EQ], c1[EQ], c2[EQ];
    for (int m = 0; m < EQ; ++m) {
      c0[m] = c[cidx(np, n, m, 0, i)];
      c1[m] = c[cidx(np, n, m, 1, i)];
      c2[m] = c[cidx(np, n, m, 2, i)];
    }
    int nb[3];
    for (int q = 0; q < 3; ++q) { /* Mesh::neighbor, mesh.hpp:56-59 */
      const int e = M->elem_edge[3 * i + q];
      nb[q] = M->edge_left[e] == i ? M->edge_right[e] : M->edge_left[e];
    }
    for (int m = 0; m < EQ; ++m) {
      const double uc = c0[m] * sqrt2;
      double umax = uc, umin = uc;
      for (int q = 0; q < 3; ++q) {
        if (nb[q] < 0) continue;
        const double un = c[cidx(np, n, m, 0, nb[q])] * sqrt2;
        if (un > umax) umax = un;
        if (un < umin) umin = un;
      }
      const double tol = 1e-13 * (fabs(uc) + (umax - umin));
      double alpha = 1.0;
      for (int k = eb; k < eb + 3 * nk; ++k) {
        const double d = c1[m] * phi1[k] + c2[m] * phi2[k];
        double a = 1.0;
        if (d > tol)
          a = (umax - uc) / d;
        else if (d < -tol)
          a = (umin - uc) / d;
        a = clamp01(a);
        if (a < alpha) alpha = a;
      }
      c1[m] *= alpha;
      c2[m] *= alpha;
    }
    double mean[EQ] = {c0[0] * sqrt2, c0[1] * sqrt2, c0[2] * sqrt2, c0[3] * sqrt2};
    const double p_mean = pressure(mean, g);
    if (mean[0] > 0.0 && p_mean > 0.0) {
      const double eps_rho = 1e-8 * mean[0], eps_p = 1e-8 * p_mean;
      double dev[EQ];
      for (int m = 0; m < EQ; ++m) dev[m] = fabs(c1[m]) * max1 + fabs(c2[m]) * max2;
      const double rho_floor = mean[0] - dev[0];
      int safe = rho_floor > eps_rho;
      if (safe) {
        const double mxp = fabs(mean[1]) + dev[1], myp = fabs(mean[2]) + dev[2];
        const double p_floor = (g - 1.0) * (mean[3] - dev[3] - 0.5 * (mxp * mxp + myp * myp) / rho_floor);
        safe = p_floor > eps_p;
      }
      if (!safe) {
        double rho_min = mean[0];
        for (int k = 0; k < n_pts; ++k) {
          const double v = c0[0] * sqrt2 + c1[0] * phi1[k] + c2[0] * phi2[k];
          if (v < rho_min) rho_min = v;
        }
        if (rho_min < eps_rho) {
          const double th = clamp01((mean[0] - eps_rho) / (mean[0] - rho_min));
          c1[0] *= th;
          c2[0] *= th;
        }
        double th_p = 1.0;
        for (int k = 0; k < n_pts; ++k) {
          double u[EQ];
          for (int m = 0; m < EQ; ++m) u[m] = c0[m] * sqrt2 + c1[m] * phi1[k] + c2[m] * phi2[k];
          if (u[0] <= 0.0) {
            th_p = 0.0;
            break;
          }
          const double pk = pressure(u, g);
          if (pk < eps_p) {
            const double r = (p_mean - eps_p) / (p_mean - pk);
            if (r < th_p) th_p = r;
          }
        }
        if (th_p < 1.0) {
          if (th_p < 0.0) th_p = 0.0;
          for (int m = 0; m < EQ; ++m) {
            c1[m] *= th_p;
            c2[m] *= th_p;
          }
        }
      }
    }
    for (int m = 0; m < EQ; ++m) {
      c[cidx(np, n, m, 1, i)] = c1[m];
      c[cidx(np, n, m, 2, i)] = c2[m];
    }
  }
  return 0;
}

/* stable_dt, solver.cpp:427-461 */
int or_stable_dt(const or_problem* P, const double* c, double cfl, double* dt, or_fail* f) {
  const dgb_mesh_view* M = P->mesh;
  const dgb_tables_view* T = P->tables;
  const int n = M->n_elements, np = T->n_p;
  const double g = P->gamma;
  double dt_min = 1.79769313486231570815e+308;
  int bad = 0;
  for (int i = 0; i < n; ++i) {
    double lambda = 0.0;
    for (int q = 1; q <= 3; ++q) {
      double u[EQ];
      for (int m = 0; m < EQ; ++m) {
        double s = 0.0;
        for (int j = 0; j < np; ++j) s += c[cidx(np, n, m, j, i)] * T->phi_edge_mid[(q - 1) * np + j];
        u[m] = s;
      }
      if (!admissible(u, g)) {
        fail_rec(f, 3, i, q, u, g);
        bad = 1;
        continue;
      }
      const int e = M->elem_edge[3 * i + q - 1];
      const double sign = M->edge_left[e] == i ? 1.0 : -1.0;
      const double s = wave_speed(u, sign * M->edge_nx[e], sign * M->edge_ny[e], g);
      if (s > lambda) lambda = s;
    }
    const double d = 2.0 * M->inradius[i] / ((2.0 * T->p + 1.0) * lambda);
    if (d < dt_min) dt_min = d;
  }
  *dt = cfl * dt_min;
  return bad;
}

/* rk_step_ws (solver.cpp:506-541) for schemes 2 and 4, plus SSP-RK2/RK3 as
 * compositions of the same operator (not in the reference). */
int or_step(const or_problem* P, double* c, double* t, double dt, int scheme, int limiting, double* resid, or_fail* f) {
  const size_t sz = (size_t)EQ * P->tables->n_p * P->mesh->n_elements;
  double *k1 = malloc(sizeof(double) * sz), *k2 = malloc(sizeof(double) * sz), *k3 = malloc(sizeof(double) * sz),
         *k4 = malloc(sizeof(double) * sz), *s = malloc(sizeof(double) * sz), *s2 = malloc(sizeof(double) * sz);
  const double t0 = *t;
  int rc = 0;
#define RHS(in, tt, out) \
  do {                   \
    rc = or_rhs(P, in, tt, out, f); \
    if (rc) goto done;   \
  } while (0)
#define LIM(x) \
  if (limiting) or_limit(P, x)
  if (scheme == 2) {
    RHS(c, t0, k1);
    for (size_t i = 0; i < sz; ++i) s[i] = c[i] + 0.5 * dt * k1[i];
    LIM(s);
    RHS(s, t0 + 0.5 * dt, k2);
    for (size_t i = 0; i < sz; ++i) s[i] = c[i] + dt * k2[i];
  } else if (scheme == 4) {
    RHS(c, t0, k1);
    for (size_t i = 0; i < sz; ++i) s[i] = c[i] + 0.5 * dt * k1[i];
    LIM(s);
    RHS(s, t0 + 0.5 * dt, k2);
    for (size_t i = 0; i < sz; ++i) s[i] = c[i] + 0.5 * dt * k2[i];
    LIM(s);
    RHS(s, t0 + 0.5 * dt, k3);
    for (size_t i = 0; i < sz; ++i) s[i] = c[i] + dt * k3[i];
    LIM(s);
    RHS(s, t0 + dt, k4);
    for (size_t i = 0; i < sz; ++i) s[i] = c[i] + dt / 6.0 * (k1[i] + 2.0 * k2[i] + 2.0 * k3[i] + k4[i]);
  } else if (scheme == 102) {
    RHS(c, t0, k1);
    for (size_t i = 0; i < sz; ++i) s2[i] = c[i] + dt * k1[i];
    LIM(s2);
    RHS(s2, t0 + dt, k2);
    for (size_t i = 0; i < sz; ++i) s[i] = 0.5 * c[i] + 0.5 * s2[i] + 0.5 * dt * k2[i];
  } else if (scheme == 103) {
    RHS(c, t0, k1);
    for (size_t i = 0; i < sz; ++i) s2[i] = c[i] + dt * k1[i];
    LIM(s2);
    RHS(s2, t0 + dt, k2);
    for (size_t i = 0; i < sz; ++i) s[i] = 0.75 * c[i] + 0.25 * s2[i] + 0.25 * dt * k2[i];
    LIM(s);
    RHS(s, t0 + 0.5 * dt, k3);
    for (size_t i = 0; i < sz; ++i) s[i] = (1.0 / 3.0) * c[i] + (2.0 / 3.0) * s[i] + (2.0 / 3.0) * dt * k3[i];
  } else {
    rc = -1;
    goto done;
  }
  LIM(s);
  {
    double r = 0.0; /* max_abs_diff, solver.cpp:672-678 */
    for (size_t i = 0; i < sz; ++i) {
      const double d = fabs(c[i] - s[i]);
      if (d > r) r = d;
    }
    *resid = r;
  }
  memcpy(c, s, sizeof(double) * sz);
  *t = t0 + dt;
done:
  free(k1);
  free(k2);
  free(k3);
  free(k4);
  free(s);
  free(s2);
  return rc;
#undef RHS
#undef LIM
}

/* run_fixed_steps, solver.cpp:600-613 */
int or_run_fixed_steps(const or_problem* P, double* c, double* t, int64_t n, int scheme, double cfl, int limiting,
                       double* resid, double* hist, or_fail* f) {
  *resid = 0.0;
  for (int64_t s = 0; s < n; ++s) {
    double dt;
    int rc = or_stable_dt(P, c, cfl, &dt, f);
    if (rc) return rc;
    rc = or_step(P, c, t, dt, scheme, limiting, resid, f);
    if (rc) return rc;
    if (hist) hist[s] = *resid;
  }
  return 0;
}

/* KAT hooks for tests/test_oracle.py: the physics primitives on their own. */
double or_pressure(const double* u, double gamma) { return pressure(u, gamma); }
void or_euler_flux(const double* u, double gamma, double* f1, double* f2) { euler_flux(u, gamma, f1, f2); }
void or_roe(const double* ul, const double* ur, double nx, double ny, double gamma, double* f) {
  roe(ul, ur, nx, ny, gamma, f);
}

void or_llf(const double* ul, const double* ur, double nx, double ny, double gamma, double* f) {
  llf(ul, ur, nx, ny, gamma, f);
}
double or_wave_speed(const double* u, double nx, double ny, double gamma) { return wave_speed(u, nx, ny, gamma); }
