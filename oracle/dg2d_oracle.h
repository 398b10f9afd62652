/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the modal-DG Euler RHS + RK stage.
 *
 * A plain-C, serial restatement of the reference's hot path
 * (/root/reference/proj/src/solver.cpp and include/dg2d/euler.hpp), used as
 * the checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg.  It is never linked into or called by the product path.
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * real reference compiled from its sources (oracle/_ref, see Makefile) and
 * against the committed golden vectors in tests/golden/ (generated from the
 * reference by tests/golden/make_golden.py).
 *
 * The mesh / tables / boundary views are layout-compatible with
 * include/dg2d_b200/dg2d_b200.h so the same arrays feed both sides.
 */
#ifndef DG2D_ORACLE_H
#define DG2D_ORACLE_H

#include <stdint.h>

#include "../include/dg2d_b200/dg2d_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct or_problem {
  const dgb_mesh_view* mesh;
  const dgb_tables_view* tables;
  const dgb_bc_view* bc;
  double gamma;
  int flux; /* 0 local Lax-Friedrichs (euler.hpp:59-71), 1 Roe (not in the reference) */
} or_problem;

/* failure record: pass 0 none, 1 eval_volume, 2 eval_surface, 3 stable_dt */
typedef struct or_fail {
  int pass;
  int64_t id;
  int point;
  double rho, p;
} or_fail;

int or_volume(const or_problem* P, const double* c, double* vol, or_fail* f);
int or_surface(const or_problem* P, const double* c, double t, double* sl, double* sr, or_fail* f);
void or_gather(const or_problem* P, const double* vol, const double* sl, const double* sr, double* deriv);
int or_rhs(const or_problem* P, const double* c, double t, double* deriv, or_fail* f);
int or_limit(const or_problem* P, double* c);
int or_stable_dt(const or_problem* P, const double* c, double cfl, double* dt, or_fail* f);
/* one step of scheme 2 (midpoint), 4 (classic), 102 (SSP2), 103 (SSP3) */
int or_step(const or_problem* P, double* c, double* t, double dt, int scheme, int limiting, double* resid, or_fail* f);
int or_run_fixed_steps(const or_problem* P, double* c, double* t, int64_t n, int scheme, double cfl, int limiting,
                       double* resid, double* hist, or_fail* f);

/* physics primitives (KAT hooks) */
double or_pressure(const double* u, double gamma);
void or_euler_flux(const double* u, double gamma, double* f1, double* f2);
void or_llf(const double* ul, const double* ur, double nx, double ny, double gamma, double* f);
void or_roe(const double* ul, const double* ur, double nx, double ny, double gamma, double* f);
double or_wave_speed(const double* u, double nx, double ny, double gamma);

#ifdef __cplusplus
}
#endif
#endif
