// Problem data evaluated on the host (libm), following proj/src/problems.cpp:
// the supersonic-vortex exact solution (problems.cpp:44-66), the
// Rankine-Hugoniot post-shock state (problems.cpp:79-94), plus the periodic
// isentropic vortex that BASELINE.json's configs name (not in the reference).
#include <cmath>
#include <stdexcept>
#include <string>

#include "setup.hpp"

namespace dgb {

void vortex_exact(double x, double y, double r_inner, double r_outer, double mach_inner,
                  double rho_inner, double c_inner, double g, double* u) {
  const double r = std::sqrt(x * x + y * y);
  const double margin = 0.05 * (r_outer - r_inner);
  if (r < r_inner - margin || r > r_outer + margin)
    throw std::domain_error("point at radius " + std::to_string(r) + " is outside the annulus");
  const double ri = r_inner, mi = mach_inner;
  const double rho =
      rho_inner * std::pow(1.0 + 0.5 * (g - 1.0) * mi * mi * (1.0 - ri * ri / (r * r)), 1.0 / (g - 1.0));
  const double vt = c_inner * mi * ri / r;
  const double p_inner = rho_inner * c_inner * c_inner / g;
  const double p = p_inner * std::pow(rho / rho_inner, g);
  const double tx = -y / r, ty = x / r;
  u[0] = rho;
  u[1] = rho * vt * tx;
  u[2] = rho * vt * ty;
  u[3] = p / (g - 1.0) + 0.5 * rho * vt * vt;
}

void rankine_hugoniot_post(const double* pre, double mach, double nx, double ny, double g, double* post) {
  const double p1 = (g - 1.0) * (pre[3] - 0.5 * (pre[1] * pre[1] + pre[2] * pre[2]) / pre[0]);
  const double c1 = std::sqrt(g * p1 / pre[0]);
  const double m2 = mach * mach;
  const double rho2 = pre[0] * ((g + 1.0) * m2) / ((g - 1.0) * m2 + 2.0);
  const double p2 = p1 * (2.0 * g * m2 - (g - 1.0)) / (g + 1.0);
  const double vn = 2.0 * (m2 - 1.0) / ((g + 1.0) * mach) * c1;
  post[0] = rho2;
  post[1] = rho2 * vn * nx;
  post[2] = rho2 * vn * ny;
  post[3] = p2 / (g - 1.0) + 0.5 * rho2 * vn * vn;
}

void isentropic_vortex(double x, double y, double xc, double yc, double beta, double u_inf,
                       double v_inf, double width, double height, double t, double g, double* u) {
  // centre advected with the mean flow, nearest periodic image
  double dx = x - (xc + u_inf * t);
  double dy = y - (yc + v_inf * t);
  if (width > 0.0) dx -= width * std::floor(dx / width + 0.5);
  if (height > 0.0) dy -= height * std::floor(dy / height + 0.5);
  const double r2 = dx * dx + dy * dy;
  const double e = std::exp(0.5 * (1.0 - r2));
  const double du = -beta / (2.0 * M_PI) * e * dy;
  const double dv = beta / (2.0 * M_PI) * e * dx;
  const double temp = 1.0 - (g - 1.0) * beta * beta / (8.0 * g * M_PI * M_PI) * e * e;
  const double rho = std::pow(temp, 1.0 / (g - 1.0));
  const double p = rho * temp;
  const double vx = u_inf + du, vy = v_inf + dv;
  u[0] = rho;
  u[1] = rho * vx;
  u[2] = rho * vy;
  u[3] = p / (g - 1.0) + 0.5 * rho * (vx * vx + vy * vy);
}

}  // namespace dgb
