/*
 * dg2d_b200 — C ABI of the B200-native modal-DG Euler right-hand side and RK stage.
 *
 * This is the drop-in boundary for the hot path of the reference solver
 * (`/root/reference/proj`, namespace `dg2d`).  Every entry point below names
 * the reference interface it replaces (file:line under proj/).  The ABI uses
 * plain pointers, sizes and status codes only: no C++ types, no exceptions,
 * no std::function, no torch types.  The C++ wrapper `dg2d_b200/dg2d.hpp`
 * re-raises the reference's exception types from the status codes.
 *
 * Array conventions (identical to the reference):
 *   coefficients  double[4][n_p][n_elem]        CoefficientArray, solver.hpp:20-38
 *                 index ((m*n_p)+j)*n_elem + i
 *   surface slots double[3][4][n_p][n_elem]     RhsBuffers::surface_left/right,
 *                 index ((q*4+m)*n_p+j)*n_elem+i solver.hpp:46-62
 *   element / edge ids are the reference ids (mesh.cpp:282-288 edge order).
 *
 * Threading: one context per device, used from one host thread; all device
 * work is enqueued on the context stream (default: a private stream, or the
 * caller's via dgb_set_stream).  Functions that return host values
 * synchronise that stream.  Not thread-safe per context.
 */
#ifndef DG2D_B200_H
#define DG2D_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
enum dgb_status {
  DGB_OK = 0,
  DGB_ERR_INADMISSIBLE = 1, /* SolverAbort: inadmissible state (solver.cpp:57-62) */
  DGB_ERR_BC = 2,           /* SolverAbort from a boundary condition (solver.cpp:203-211, 249) */
  DGB_ERR_ARG = 3,          /* std::invalid_argument (solver.cpp:290, 533) */
  DGB_ERR_CUDA = 4,         /* CUDA runtime failure or no device */
  DGB_ERR_MESH = 5,         /* MeshError (mesh.hpp:15-17) */
  DGB_ERR_NOT_REACHED = 6,  /* SolverAbort "t_end not reached within N steps" (solver.cpp:590-591) */
  DGB_ERR_IO = 7            /* checkpoint / file errors (solver.cpp:619, 637-658) */
};

/* Human-readable message of the last failure on this thread (any handle). */
const char* dgb_last_message(void);

/* ---------------------------------------------------------------- views */
/* SoA view of a reference `Mesh` (mesh.hpp:21-63).  All pointers are host
 * pointers owned by the caller; they are only read during dgb_create. */
typedef struct dgb_mesh_view {
  int32_t n_vertices;
  const double* vx;          /* [n_vertices]  Mesh::vertices[].x */
  const double* vy;          /* [n_vertices]  Mesh::vertices[].y */
  int32_t n_elements;
  const int32_t* elem_v;     /* [3*n_elements] Element::v (CCW), row-major */
  const int32_t* elem_edge;  /* [3*n_elements] Element::edge */
  const double* det_jac;     /* [n_elements]  Element::det_jac */
  const double* tau;         /* [4*n_elements] Element::tau, row-major */
  const double* inradius;    /* [n_elements]  Element::inradius */
  int32_t n_edges;
  int32_t n_boundary_edges;  /* Mesh::n_boundary_edges; boundary edges are [0, n) */
  const int32_t* edge_v0, *edge_v1, *edge_left, *edge_right; /* [n_edges] */
  const int32_t* edge_side_left, *edge_side_right;          /* [n_edges] 1..3 (0 boundary) */
  const double* edge_nx, *edge_ny, *edge_half_length;        /* [n_edges] */
} dgb_mesh_view;

/* View of a reference `BasisTables` (basis.hpp:48-82). */
typedef struct dgb_tables_view {
  int32_t p, n_p, n_quad, n_edge_pts;
  const double* phi_interior;      /* [n_quad*n_p] */
  const double* dphi_dr_interior;  /* [n_quad*n_p] */
  const double* dphi_ds_interior;  /* [n_quad*n_p] */
  const double* w_interior;        /* [n_quad]     */
  const double* r_interior;        /* [2*n_quad]  (r,s) pairs */
  const double* phi_edge;          /* [3*n_edge_pts*n_p] */
  const double* w_edge;            /* [n_edge_pts] */
  const double* xi_edge;           /* [n_edge_pts] */
  const double* phi_edge_mid;      /* [3*n_p] */
} dgb_tables_view;

/* Boundary data replacing the host closures of `BoundaryConditions`
 * (euler.hpp:104-111).  The closures are evaluated by the caller once at every
 * boundary Gauss point (dgb_boundary_points gives the coordinates, computed as
 * solver.cpp:198 does); the moving shock (euler.hpp:91-102) stays analytic. */
typedef struct dgb_bc_view {
  double inflow_state[4];          /* BoundaryConditions::inflow_state */
  const double* dirichlet_state;   /* [n_boundary_edges*n_edge_pts*4] or NULL -> inflow_state */
  const double* wall_normal;       /* [n_boundary_edges*n_edge_pts*2] or NULL (code -2 then fails) */
  int32_t has_shock;               /* BoundaryConditions::shock engaged */
  double shock_x0, shock_angle_deg, shock_speed;
  double shock_post[4], shock_pre[4];
} dgb_bc_view;

/* ---------------------------------------------------------------- context */
typedef struct dgb_ctx dgb_ctx;

/* SolverContext (solver.hpp:80-87) + device upload of mesh, tables, BC data.
 * gamma = GasModel::gamma.  device = CUDA ordinal. */
int dgb_create(const dgb_mesh_view* mesh, const dgb_tables_view* tables, const dgb_bc_view* bc,
               double gamma, int device, dgb_ctx** out);
int dgb_destroy(dgb_ctx* ctx);
/* Enqueue all work on a caller stream (cudaStream_t passed as void*); NULL = private stream. */
int dgb_set_stream(dgb_ctx* ctx, void* cuda_stream);
/* Numerical flux at the edges: the reference's local Lax-Friedrichs (riemann_solver,
 * euler.hpp:59-71; the default) or Roe with Harten's entropy fix (not in the reference,
 * asked for by BASELINE.json's north star; oracle/dg2d_oracle.c roe()). */
enum dgb_flux { DGB_FLUX_LLF = 0, DGB_FLUX_ROE = 1 };
int dgb_set_flux(dgb_ctx* ctx, int flux);
/* Limiting runs at p = 1 (whole-mesh contexts): 1 = each RK stage and its limit (solver.cpp:517-535)
 * in ONE persistent launch, the limiter trailing the stage tile by tile through L2; 0 = a stage
 * kernel followed by a limiter kernel; -1 (default; env DGB_FUSED_LIMIT=0/1 fixes it at creation) =
 * the fused launch on meshes up to 400K triangles, where it saves a launch per stage, the two
 * kernels above (measured).  All give bit-identical results. */
int dgb_set_fused_limiter(dgb_ctx* ctx, int enable);
/* Trace buffers (no reference counterpart: a data-layout choice of the device step loop).  With
 * enable = 1, the stages of a run at p >= 2 without limiting write the edge
 * traces of their output and the next stage reads its own and its neighbours' traces instead of
 * interpolating them from the coefficient columns; 0 interpolates every stage.  Default from
 * env DGB_TRACE_BUF at creation.  Both give bit-identical results. */
int dgb_set_trace_buffers(dgb_ctx* ctx, int enable);
/* Launch forms for small meshes (no reference counterpart: the CPU has no launch shape).  A p <= 2
 * stage launch of at most stage_max_n elements, and a limiter launch of at most limit_max_n, take
 * the four-lanes-per-element latency form instead of one thread per element; -1 = the built-in
 * size (env DGB_G4_MAXN / DGB_LIM4_MAXN), 0 = never.  Both forms give bit-identical results. */
int dgb_set_latency_forms(dgb_ctx* ctx, int stage_max_n, int limit_max_n);
/* Replace the Dirichlet table (time-dependent BCs): same layout as dgb_bc_view. */
int dgb_set_dirichlet(dgb_ctx* ctx, const double* dirichlet_state);
/* Time-dependent boundary data inside the step (the reference evaluates its Dirichlet closure at
 * every stage time, solver.cpp:198-211): n_tables (1..8) tables laid out as dgb_bc_view's, table k
 * holding the closure at the time of stage k of the next step (t + c_k dt, dgb_scheme_stage_times);
 * a stage beyond the last table reads the last one.  Kept until replaced; dgb_set_dirichlet
 * returns to one table for every stage. */
int dgb_set_dirichlet_stages(dgb_ctx* ctx, int n_tables, const double* tables);
/* Stage-time coefficients c_k of a scheme (stage k runs at t + c_k dt) and the stage count. */
int dgb_scheme_stage_times(int scheme, double* tcoef, int* n_stages);

/* Coefficient slots living on the device, reference layout at the boundary. */
enum dgb_slot {
  DGB_SLOT_STATE = 0,  /* SolverState::coeffs (time-stepped by the drivers) */
  DGB_SLOT_INPUT = 1,  /* a free input array (compute_rhs / pass-level calls) */
  DGB_SLOT_VOLUME = 2, /* RhsBuffers::volume */
  DGB_SLOT_DERIV = 3   /* compute_rhs output */
};
int dgb_upload(dgb_ctx* ctx, int slot, const double* host_coeffs);
int dgb_download(dgb_ctx* ctx, int slot, double* host_coeffs);
/* Asynchronous forms of dgb_upload / dgb_download (no reference counterpart: the
 * reference's arrays live in host memory).  They return once the copy is enqueued;
 * `host_coeffs` should be pinned (cudaHostAlloc) and must stay untouched until
 * dgb_sync.  Each direction has its own copy stream and staging buffer, so a result's
 * device->host copy overlaps the next input's host->device copy; later calls on the
 * context are ordered after them on the device. */
int dgb_upload_async(dgb_ctx* ctx, int slot, const double* host_coeffs);
/* dgb_upload_async in two halves, so the next request's host->device copy can run while
 * the current request computes: dgb_stage_input_async enqueues the copy into the
 * context's input staging buffer (after the previous staged input was committed);
 * dgb_commit_input(slot) orders, on the compute stream, the permutation of the staged
 * input into `slot` after everything enqueued so far.  DGB_ERR_ARG if nothing is staged. */
int dgb_stage_input_async(dgb_ctx* ctx, const double* host_coeffs);
int dgb_commit_input(dgb_ctx* ctx, int slot);
int dgb_download_async(dgb_ctx* ctx, int slot, double* host_coeffs);
/* Wait for every copy and kernel the context has enqueued. */
int dgb_sync(dgb_ctx* ctx);
/* Device-resident copies (no host round trip): dst <- src. */
int dgb_copy_slot(dgb_ctx* ctx, int dst, int src);

/* ---------------------------------------------------------------- passes */
/* eval_volume_pass (solver.cpp:99-158): VOLUME <- volume integral of `in_slot`. */
int dgb_eval_volume_pass(dgb_ctx* ctx, int in_slot);
/* eval_surface_pass (solver.cpp:160-251): fills the per-side slot buffer. */
int dgb_eval_surface_pass(dgb_ctx* ctx, int in_slot, double t);
/* Slot buffer in RhsBuffers layout; a slot not owned by the edge side is left 0. */
int dgb_download_surface(dgb_ctx* ctx, double* surface_left, double* surface_right);
/* Fill the slot buffer from RhsBuffers layout: slot (q,i) is taken from
 * surface_left if element i is the left element of its side-q edge, else from
 * surface_right (the orientation test of solver.cpp:264). */
int dgb_upload_surface(dgb_ctx* ctx, const double* surface_left, const double* surface_right);
/* eval_rhs_pass (solver.cpp:253-277): DERIV <- (VOLUME + slots) / det_jac. */
int dgb_eval_rhs_pass(dgb_ctx* ctx);
/* compute_rhs (solver.cpp:279-284), fused single kernel: out_slot <- L(in_slot, t). */
int dgb_compute_rhs(dgb_ctx* ctx, int in_slot, double t, int out_slot);

/* limit (solver.cpp:286-425), in place; p != 1 -> DGB_ERR_ARG. */
int dgb_limit(dgb_ctx* ctx, int slot);
/* stable_dt (solver.cpp:427-461). */
int dgb_stable_dt(dgb_ctx* ctx, int slot, double cfl, double* dt);

/* ---------------------------------------------------------------- time stepping */
/* Schemes: the reference's rk_order 2 (midpoint) and 4 (classical), solver.cpp:513-531,
 * plus the strong-stability-preserving schemes BASELINE.json asks for (not in the reference). */
enum dgb_scheme {
  DGB_RK2_MIDPOINT = 2,
  DGB_RK4_CLASSIC = 4,
  DGB_SSP_RK2 = 102,
  DGB_SSP_RK3 = 103
};
/* State time / step counter (SolverState::t, step_count). */
int dgb_set_time(dgb_ctx* ctx, double t, int64_t step_count);
int dgb_get_time(dgb_ctx* ctx, double* t, int64_t* step_count);
/* rk_step (solver.cpp:545-557) on STATE with a given dt; returns max|c_new - c_old|. */
int dgb_rk_step(dgb_ctx* ctx, int scheme, double dt, int limiting, double* residual);
/* run_fixed_steps (solver.cpp:600-613): stable dt every step, state stays on device.
 * residual_hist (optional, [n_steps]) receives the per-step residual (on_step). */
int dgb_run_fixed_steps(dgb_ctx* ctx, int scheme, double cfl, int limiting, int64_t n_steps,
                        double* residual, double* residual_hist);
/* run_to_time (solver.cpp:581-598): last step clipped to t_end. */
int dgb_run_to_time(dgb_ctx* ctx, int scheme, double cfl, int limiting, double t_end,
                    int64_t max_steps, double* residual, int64_t* steps_taken,
                    double* residual_hist, int64_t hist_cap);
/* run_to_steady (solver.cpp:559-579). */
int dgb_run_to_steady(dgb_ctx* ctx, int scheme, double cfl, int limiting, double tol,
                      int64_t max_steps, int64_t* steps, double* residual, int* converged,
                      double* residual_hist, int64_t hist_cap);

/* ---------------------------------------------------------------- reductions, diagnostics */
/* total_mass (solver.cpp:662-670), serial-order sum on the host for determinism. */
int dgb_total_mass(dgb_ctx* ctx, int slot, double* mass);
/* compute_l2_error (runner.cpp:127-150): L2 norm of the density error against exact values
 * given at every interior quadrature point, exact_rho[n_elem][n_quad] (reference order, points
 * from dgb_interior_points).  Per-element partials on the device, summed on the host in element
 * order.  For a partitioned context: the rank's partial sum of squares (exact_rho over its owned
 * elements, ascending id); the caller adds the ranks in rank order and takes the square root. */
int dgb_l2_error(dgb_ctx* ctx, int slot, const double* exact_rho, double* l2);
/* project_initial (solver.cpp:74-97) on the device, straight into a coefficient slot:
 * point_states[(i*n_quad + k)*4 + m] at the interior points of every local element (compact
 * order: reference order for a whole-mesh context; owned then halo ids for a partition).
 * DGB_ERR_INADMISSIBLE with the reference's message for an inadmissible point state. */
int dgb_project_slot(dgb_ctx* ctx, int slot, const double* point_states);
/* Output extraction for export_vtk (output.cpp:10-20, 30-65): the conserved state at the three
 * corners (reference coordinates (0,0), (1,0), (0,1)) of every owned element,
 * out[(i*3 + c)*4 + m]; phi_corner[c*n_p + j] = eval_basis(p, j, corner c). */
int dgb_corner_states(dgb_ctx* ctx, int slot, const double* phi_corner, double* out);
/* max_abs_diff (solver.cpp:672-678). */
int dgb_max_abs_diff(dgb_ctx* ctx, int slot_a, int slot_b, double* diff);

/* PassTimers (solver.hpp:64-70); `stage` holds the fused RHS+stage kernels. */
typedef struct dgb_pass_timers {
  double volume, surface, rhs, limiter, other, stage;
} dgb_pass_timers;
int dgb_timers(dgb_ctx* ctx, dgb_pass_timers* out);
int dgb_reset_timers(dgb_ctx* ctx);
int dgb_enable_timers(dgb_ctx* ctx, int enable);

/* AbortRecord (solver.cpp:37-63): the failure behind the last DGB_ERR_INADMISSIBLE. */
typedef struct dgb_abort_info {
  char where[32]; /* "eval_volume", "eval_surface", "stable_dt" */
  int64_t id;     /* element or edge id (reference numbering) */
  int32_t point;
  double rho, p;
} dgb_abort_info;
int dgb_last_abort(dgb_ctx* ctx, dgb_abort_info* out);

/* ---------------------------------------------------------------- partitions (multi-GPU)
 * SURVEY.md 8(e); no reference counterpart (the reference is one shared-memory
 * process, solver.cpp OpenMP loops).  Rank r of `world` owns the contiguous
 * reference ids [n*r/world, n*(r+1)/world) ("identical partition indexing").
 * Its context holds the owned elements plus halo columns for the off-rank
 * neighbours.  Coefficient arrays of a partitioned context cross the ABI in
 * "compact" order: dgb_upload takes [4][n_p][n_owned + n_halo] (owned in
 * ascending id, then halo in ascending id, see dgb_part_local_ids), dgb_download
 * returns [4][n_p][n_owned].  Every RK stage the elements a peer needs are
 * written straight into the peer's halo columns by the stage kernel (peer
 * memory over NVLink), then an epoch flag is raised; each rank computes its
 * interior elements while waiting for the peers' flags.  Setup: create on every
 * rank, exchange peer views (same process) or IPC handles (one process per
 * GPU), tell every rank which of its elements each peer needs
 * (dgb_part_set_sends with the peer's halo ids/columns), then dgb_part_finalize.
 * After that the ordinary dgb_run_* / dgb_rk_step calls run the partitioned
 * solve; all ranks must issue the same sequence of calls. */
int dgb_part_create(const dgb_mesh_view* mesh, const dgb_tables_view* tables, const dgb_bc_view* bc,
                    double gamma, int device, int rank, int world, dgb_ctx** out);
typedef struct dgb_part_info {
  int32_t rank, world, lo, hi, n_owned, n_halo, n_interior, ld;
  uint32_t neighbor_mask; /* ranks owning halo elements */
} dgb_part_info;
int dgb_part_get_info(dgb_ctx* ctx, dgb_part_info* out);
/* Host-only plan of rank `rank` (no device needed): counts in *info, then the halo
 * ids (ascending; halo column = n_owned + index) and the boundary element ids
 * (owned elements with an off-rank neighbour, ascending); arrays may be NULL. */
int dgb_part_plan(const dgb_mesh_view* mesh, int rank, int world, dgb_part_info* info, int32_t* halo_ids,
                  int32_t* boundary_ids);
/* Halo columns: reference ids and device columns (a peer feeds these). */
int dgb_part_halo_ids(dgb_ctx* ctx, int32_t* ids, int32_t* cols);
/* Compact local order used by dgb_upload: owned ids then halo ids. */
int dgb_part_local_ids(dgb_ctx* ctx, int32_t* ids);
/* Device addresses a peer writes to (same-process attachment). */
typedef struct dgb_peer_view {
  void* buf[4];  /* rotating coefficient buffers */
  void* flags;   /* [8] epoch flags */
  void* scal;    /* [2][8][4] scalar exchange */
  int32_t ld;
} dgb_peer_view;
int dgb_part_peer_view(dgb_ctx* ctx, dgb_peer_view* out);
int dgb_part_attach_peer(dgb_ctx* ctx, int peer, const dgb_peer_view* view);
/* Cross-process attachment through CUDA IPC: DGB_IPC_BYTES of handles. */
#define DGB_IPC_BYTES (5 * 64)
int dgb_part_ipc_export(dgb_ctx* ctx, void* handles);
int dgb_part_attach_peer_ipc(dgb_ctx* ctx, int peer, const void* handles, int32_t peer_ld);
/* Elements of this rank (reference ids) that `peer` holds as halo, at the peer's columns. */
int dgb_part_set_sends(dgb_ctx* ctx, int peer, int64_t n, const int32_t* ids, const int32_t* peer_cols);
int dgb_part_finalize(dgb_ctx* ctx);
/* Bound on a halo wait before the run fails with DGB_ERR_CUDA (default 60 s). */
int dgb_part_set_timeout(dgb_ctx* ctx, double seconds);

/* Kernel launches issued by this context so far (benchmark evidence). */
int64_t dgb_launch_count(dgb_ctx* ctx);
/* Per-step kernel-only timing helper for the benchmark: device ms of the fused
 * stage kernels since the last reset (CUDA events on the context stream). */
int dgb_stage_kernel_ms(dgb_ctx* ctx, double* ms, int64_t* launches);
/* The individual device durations (ms) behind the timers since the last dgb_reset_timers, one
 * per timed launch of `category` (dgb_pass_timers order: 0 volume, 1 surface, 2 rhs,
 * 3 limiter, 4 other, 5 stage); *n = the count, at most `cap` are copied (benchmark medians). */
int dgb_timer_samples(dgb_ctx* ctx, int category, double* ms, int64_t cap, int64_t* n);

/* Measured FP64 FMA-pipe throughput of `device` (DFMA loop on every SM), TFLOP/s;
 * the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry). */
int dgb_fp64_peak(int device, double* tflops);

/* ---------------------------------------------------------------- host setup (runs once) */
/* Our own builders, bit-compatible with the reference's (not the hot path). */
typedef struct dgb_mesh dgb_mesh;
typedef struct dgb_tables dgb_tables;

/* parse_msh + build_connectivity (mesh.cpp:45-151, 186-306). */
int dgb_mesh_from_msh(const char* text, size_t len, dgb_mesh** out);
/* Direct structured generators, identical to build_connectivity(parse_msh(gen_*_msh(..)))
 * (problems.cpp:123-199) without the text round trip; kinds below. */
enum dgb_mesh_kind {
  DGB_MESH_BOX = 0,          /* params: width, height, tag           (gen_box_msh) */
  DGB_MESH_SHEARED_BOX = 1,  /* params: width, height, shear, tag    (gen_sheared_box_msh) */
  DGB_MESH_DOUBLE_MACH = 2,  /* params: x0                           (gen_double_mach_msh) */
  DGB_MESH_VORTEX = 3,       /* nx = level (any >= 0); params: r_inner, r_outer (gen_vortex_msh) */
  DGB_MESH_PERIODIC_BOX = 4  /* params: width, height; all four sides periodic (new) */
};
int dgb_mesh_generate(int kind, int nx, int ny, const double* params, int n_params,
                      dgb_mesh** out);
/* GMSH v2.2 text of a generator (problems.cpp:11-29 format); buf may be NULL to size. */
int dgb_mesh_generate_text(int kind, int nx, int ny, const double* params, int n_params,
                           char* buf, size_t cap, size_t* needed);
int dgb_mesh_get_view(const dgb_mesh* mesh, dgb_mesh_view* out);
/* dump_edges (mesh.cpp:308-313) text. */
int dgb_mesh_dump_edges(const dgb_mesh* mesh, char* buf, size_t cap, size_t* needed);
void dgb_mesh_free(dgb_mesh* mesh);

/* build_tables (basis.cpp:201-242). */
int dgb_tables_build(int p, dgb_tables** out);
int dgb_tables_get_view(const dgb_tables* tables, dgb_tables_view* out);
void dgb_tables_free(dgb_tables* tables);
/* eval_basis / eval_basis_grad (basis.cpp:136-157). */
int dgb_eval_basis(int p, int j, double r, double s, double* phi, double* dr, double* ds);

/* Physical coordinates of every interior quadrature point [n_elem][n_quad][2]
 * (map_to_physical, solver.cpp:65-70) and boundary Gauss point [n_bnd][K][2]
 * (solver.cpp:198). */
int dgb_interior_points(const dgb_mesh_view* mesh, const dgb_tables_view* tables, double* xy);
int dgb_boundary_points(const dgb_mesh_view* mesh, const dgb_tables_view* tables, double* xy);
/* project_initial (solver.cpp:74-97) from point values [n_elem][n_quad][4]. */
int dgb_project(const dgb_mesh_view* mesh, const dgb_tables_view* tables, double gamma,
                const double* point_states, double* coeffs);

/* Problem data (problems.cpp): evaluated on the host with libm. */
int dgb_vortex_exact(const double* xy, int64_t n, double r_inner, double r_outer,
                     double mach_inner, double rho_inner, double c_inner, double gamma,
                     double* states);
int dgb_rankine_hugoniot_post(const double* pre, double mach, double nx, double ny,
                              double gamma, double* post);
/* Isentropic vortex (Shu) on a periodic box: centre (xc,yc), strength beta, mean flow
 * (u_inf, v_inf), periodic images within (width,height); evaluated at time t. (new) */
int dgb_isentropic_vortex(const double* xy, int64_t n, double xc, double yc, double beta,
                          double u_inf, double v_inf, double width, double height, double t,
                          double gamma, double* states);

#ifdef __cplusplus
}
#endif
#endif /* DG2D_B200_H */
