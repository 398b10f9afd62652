// Host-side setup for the B200 path: basis tables, mesh connectivity and problem
// data.  These run once per run and produce exactly the data the reference's
// builders produce (basis.cpp, mesh.cpp, problems.cpp under /root/reference/proj),
// laid out as plain arrays ready for the device upload.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace dgb {

struct MeshError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

constexpr int kMaxDegree = 5;
constexpr int kEq = 4;
inline constexpr int basis_count(int p) { return (p + 1) * (p + 2) / 2; }

// ------------------------------------------------------------------ basis
// Orthonormal Koornwinder-Dubiner basis on the canonical triangle
// (0,0),(1,0),(0,1); mode order by total degree then ascending k
// (basis.cpp:63-73).
double eval_basis(int p, int j, double r, double s);
void eval_basis_grad(int p, int j, double r, double s, double& dr, double& ds);

struct Rule2D {
  std::vector<double> r, s, w;  // weights sum to 1/2
};
Rule2D interior_rule(int p);  // Dunavant, exact to degree 2p (basis.cpp:85-108)
void gauss_legendre(int n, std::vector<double>& nodes, std::vector<double>& weights);
void side_point(int q, double xi, double& r, double& s);  // q = 1..3 (basis.cpp:194-199)

struct Tables {
  int p = 0, n_p = 0, n_quad = 0, n_edge_pts = 0;
  std::vector<double> phi_interior, dphi_dr, dphi_ds, w_interior, r_interior;  // r_interior: (r,s)
  std::vector<double> phi_edge, w_edge, xi_edge, phi_edge_mid;
};
Tables build_tables(int p);

// ------------------------------------------------------------------ mesh
struct Precursor {
  std::vector<double> vx, vy;
  std::vector<std::array<int, 3>> tris;
  struct Line {
    int v0, v1, tag;
  };
  std::vector<Line> lines;
  // Optional periodic identification: vertex -> representative used to pair
  // edges (empty = identity).  Geometry always uses the real vertex.
  std::vector<int> key_of;
};

Precursor parse_msh(const char* text, std::size_t len);

// SoA mesh, same content as the reference Mesh (mesh.hpp:46-63).
struct Mesh {
  std::vector<double> vx, vy;
  int n_elem = 0;
  std::vector<int32_t> elem_v, elem_edge;  // [3*n]
  std::vector<double> det, tau, inradius;  // [n], [4n], [n]
  int n_edges = 0, n_boundary = 0;
  std::vector<int32_t> ev0, ev1, eleft, eright, eside_l, eside_r;
  std::vector<double> enx, eny, eh;
};
Mesh build_connectivity(const Precursor& pre);

enum MeshKind { kBox = 0, kShearedBox = 1, kDoubleMach = 2, kVortex = 3, kPeriodicBox = 4 };
Precursor generate(int kind, int nx, int ny, const double* params, int n_params);
std::string format_msh(const Precursor& pre);
std::string dump_edges(const Mesh& m);

// ------------------------------------------------------------------ problems
void vortex_exact(double x, double y, double r_inner, double r_outer, double mach_inner,
                  double rho_inner, double c_inner, double gamma, double* u);
void rankine_hugoniot_post(const double* pre, double mach, double nx, double ny, double gamma,
                           double* post);
void isentropic_vortex(double x, double y, double xc, double yc, double beta, double u_inf,
                       double v_inf, double width, double height, double t, double gamma,
                       double* u);

}  // namespace dgb
