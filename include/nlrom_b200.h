/*
 * nlrom_b200 — C ABI of the B200-native DAE-subspace Newton-step hot path
 * (arXiv 2102.11026; reference package `nlrom`, /root/reference/pkg).
 *
 * The reference has no FFI ("in-process, no external
 * interfaces"); its drop-in surface is the Python API of `nlrom` (SURVEY.md
 * §8b). Each entry point below is the native body of one reference operation;
 * the Python package `nlrom` (this repo) binds them with ctypes
 * (paper_2102_11026_b200/_lib.py, INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - plain pointers and sizes only; all host arrays C-contiguous float64 / int32;
 *    matrices row-major; multicomplex part stacks are (2^k, dim, batch) with the
 *    bitmask slot layout of mcx.py:1-8 (MCArray layout, mcx.py:294-300);
 *  - the caller owns host arrays (copied in / out); handles own device memory,
 *    streams and CUDA graphs; results never alias inputs;
 *  - every call returns an NLROM_* status; the text of the last error is
 *    available from nlrom_*_last_error();
 *  - a handle must not be used from two threads at once ("one simulation per
 *    thread"); calls on different handles are independent.
 */
#ifndef NLROM_B200_H
#define NLROM_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define NLROM_API __attribute__((visibility("default")))
#else
#define NLROM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (SURVEY.md §8b "errors") */
#define NLROM_OK 0
#define NLROM_ERR_ORDER 1        /* -> nlrom.mcx.OrderError (mcx.py:31-32)            */
#define NLROM_ERR_DIM 2          /* -> ValueError "dimension mismatch"  */
#define NLROM_ERR_NONFINITE 3    /* -> FloatingPointError "non-finite"  */
#define NLROM_ERR_NEWTON 4       /* -> NewtonDivergence with last norm  */
#define NLROM_ERR_CUDA 5         /* -> RuntimeError                                   */
#define NLROM_ERR_ARG 6          /* -> ValueError                                     */
#define NLROM_ERR_NOCACHE 7      /* -> backward without forward         */

/* ------------------------------------------------------------------------- */
/* generic dense network: densenet.forward / densenet.backward                */
/* (LayerSpec kinds SPEC.md:111-116)                         */
/* ------------------------------------------------------------------------- */
#define NLROM_LAYER_FC 0
#define NLROM_LAYER_FILTER 1
#define NLROM_LAYER_SIN 2
#define NLROM_LAYER_SQUARE 3

typedef struct nlrom_net nlrom_net;

typedef struct {
  int kind;           /* NLROM_LAYER_*                                          */
  int in_dim, out_dim;
  const double* W;    /* FC: (out,in) row-major; FILTER: basis U (dim, n_basis) */
  const double* b;    /* FC: (out,)                                             */
  int n_basis;        /* FILTER: n_p                                            */
} nlrom_layer_desc;

/* densenet.DenseNet upload (replaces in-process numpy weights) */
NLROM_API int nlrom_net_create(nlrom_net** out, int device, int n_layers, const nlrom_layer_desc* layers);
NLROM_API void nlrom_net_destroy(nlrom_net* net);
NLROM_API const char* nlrom_net_last_error(const nlrom_net* net);

/* densenet.forward(net, x) over real (order 0) or multicomplex (order 1..3)
 * inputs: parts_in (2^order, in_dim, batch) -> parts_out (2^order, out_dim, batch).
 * True multicomplex arithmetic (recursive sin, mcx.py:63-100). */
NLROM_API int nlrom_net_forward(nlrom_net* net, int order, const double* parts_in, int batch, double* parts_out);

/* densenet.backward(net, x, upstream), order 0 (real) or 1 (complex-step BP,
 * PAPER.md:353-366). x_parts (2^o, in, B), up_parts (2^o, out, B) ->
 * in_cot (2^o, in, B); param_cot (nullable): for each FC layer in order,
 * dW (2^o, out, in) then db (2^o, out), concatenated. */
NLROM_API int nlrom_net_backward(nlrom_net* net, int order, const double* x_parts, const double* up_parts,
                       int batch, double* in_cot, double* param_cot);

/* ------------------------------------------------------------------------- */
/* reduced simulator context: decoder + FE model + cubature                   */
/* (daereduce.ReducedModel, elastic.ElasticModel, neucubature.CubatureModel)  */
/* ------------------------------------------------------------------------- */
typedef struct nlrom_ctx nlrom_ctx;

typedef struct {
  /* dims: N free DOFs, n_p linear (PCA) and n_q nonlinear (DAE) coordinates   */
  int N, n_p, n_q;
  /* decoder D: n_fc FC layers widths[0]=n_q .. widths[n_fc]=N, sin after all
     but the last, then the filter I - U U^T       */
  int n_fc;
  const int* widths;
  const double* const* W;   /* W[l]: (widths[l+1], widths[l]) row-major       */
  const double* const* b;   /* b[l]: (widths[l+1],)                            */
  const double* U;          /* (N, n_p) row-major, orthonormal columns         */
  const double* mass;       /* (N,) lumped, free DOFs                          */
  /* tet mesh (elastic.TetMesh / ElasticModel)                */
  int n_verts, n_tets;
  const int* tets;          /* (T,4)                                           */
  const int* vert_dof;      /* (V,) free-vertex index or -1 if fixed           */
  const double* Dm_inv;     /* (T,3,3) row-major inverse rest edge matrices    */
  const double* vol;        /* (T,)                                            */
  double mu, lambda, alpha; /* StVK Lame parameters, Rayleigh mass damping     */
  /* cubature set C and weight net (neucubature.CubatureModel)
     wnet: N -> wn -> wn -> wn (sin) -> T (square), only rows of C are used    */
  int n_cub;
  const int* cub_elems;     /* (|C|,) element ids, duplicate-free              */
  int wnet_width;
  const double* const* wnet_W; /* 4 layers, (out,in) row-major               */
  const double* const* wnet_b;
  /* number of independent simulations sharing this model, batched through one
     set of kernels (configs[4]: 4096 sims); state arrays are (n_sims, n)      */
  int n_sims;
} nlrom_model_desc;

NLROM_API int nlrom_create(nlrom_ctx** out, int device, const nlrom_model_desc* desc);
NLROM_API void nlrom_destroy(nlrom_ctx* ctx);
NLROM_API const char* nlrom_last_error(const nlrom_ctx* ctx);

/* diffops queries with the reference pass structure.
 * op: one of NLROM_OP_*; vec = v (jvp/hvv/hv/svv) or a (vjp/vhp), may be NULL
 * for value/jacobian. out sizes: VALUE/JVP/HVV N; JACOBIAN/HV/SVV (N,n_q)
 * row-major; VJP n_q; VHP (n_q,n_q) row-major.
 * mode 0: multi-dual arithmetic on eps-scaled slots (eps cancels exactly);
 * mode 1: literal multicomplex CSFD with the given eps (mcx arithmetic). */
#define NLROM_OP_VALUE 0
#define NLROM_OP_JVP 1
#define NLROM_OP_JACOBIAN 2
#define NLROM_OP_HVV 3
#define NLROM_OP_HV 4
#define NLROM_OP_SVV 5
#define NLROM_OP_VJP 6
#define NLROM_OP_VHP 7
NLROM_API int nlrom_diffop(nlrom_ctx* ctx, int op, const double* q, const double* vec, double eps, int mode, double* out);

/* SimConfig */
typedef struct {
  double dt;
  double newton_tol;
  int max_iters;
  int drop_fict;      /* LSD simplification toggle                              */
  int integration;    /* 0 = cubature (C, wnet weights), 1 = exact_sum          */
  int line_search;    /* backtracking halving <= 10          */
  int fixed_iters;    /* > 0: exactly that many Newton steps, no line search    */
} nlrom_simcfg;

typedef struct {
  int iters;
  double res_norm;
  int status;
} nlrom_step_info;

/* The fused per-iteration pieces, each at candidate r with state (r_bar, rdot_bar):
 * rdsim.residual, rdsim.system_jacobian,
 * rdsim.delta_j, rdsim.fictitious_force. */
NLROM_API int nlrom_residual(nlrom_ctx* ctx, const double* r, const double* r_bar, const double* rdot_bar,
                   const double* f_ext, const nlrom_simcfg* cfg, double* phi);
NLROM_API int nlrom_system_jacobian(nlrom_ctx* ctx, const double* r, const double* r_bar, const double* rdot_bar,
                          const double* f_ext, const nlrom_simcfg* cfg, double* S);
NLROM_API int nlrom_delta_j(nlrom_ctx* ctx, const double* q, const double* q_bar, const double* qdot_bar,
                  double dt, int drop_fict, double* dJ);
NLROM_API int nlrom_fictitious_force(nlrom_ctx* ctx, const double* q, const double* q_bar, double* f_fict);

/* neucubature: wnet_forward restricted to C and
 * cubature_integrate: f_red (n), K_red (n,n) row-major,
 * integration 0 = cubature, 1 = exact_sum (C = all elements, w = 1).
 * w_cub holds w_len doubles; w_len must equal |C| (NLROM_ERR_DIM otherwise). */
NLROM_API int nlrom_wnet_forward(nlrom_ctx* ctx, const double* r, double* w_cub, int64_t w_len);
NLROM_API int nlrom_cubature_integrate(nlrom_ctx* ctx, const double* r, int integration, double* f_red, double* K_red);

/* elastic: per-element StVK forces of a full-space displacement u (N,):
 * f_int (N,) assembled (elastic.internal_force) and, if
 * want_K, per-element stiffness K_e (T,12,12) (elastic.stiffness, SPEC.md:336-343;
 * rows/cols vertex-major over the element's 4 vertices, fixed DOFs included). */
NLROM_API int nlrom_element_forces(nlrom_ctx* ctx, const double* u, int want_K, double* f_int, double* K_elems);

/* elastic.element_reduced_force: J~(r)_e^T f_e(u(r)) for a list
 * of elements; out (n_elems, n) row-major. */
NLROM_API int nlrom_element_reduced_forces(nlrom_ctx* ctx, const double* r, const int* elems, int n_elems, double* out);

/* daereduce: u = U p + D(q) (Eq. 9) and J~ = [U, J] (N, n) row-major */
NLROM_API int nlrom_full_displacement(nlrom_ctx* ctx, const double* r, double* u);
NLROM_API int nlrom_jtilde(nlrom_ctx* ctx, const double* q, double* Jt);

/* rdsim.step: host state in / out. In fixed-iteration mode (cfg->fixed_iters
 * > 0) info may be NULL: the final residual of the last iterate (info->res_norm) is then not
 * evaluated (one residual evaluation less per call); the pivot status is always checked. */
NLROM_API int nlrom_step(nlrom_ctx* ctx, const double* r_bar, const double* rdot_bar, const double* f_ext,
               const nlrom_simcfg* cfg, double* r_out, double* rdot_out, nlrom_step_info* info);

/* Device-resident variant for torch tensors: all pointers are device pointers
 * on `stream` (cudaStream_t passed as void*). Fixed-iteration mode only
 * (cfg->fixed_iters > 0), no host synchronisation inside. */
NLROM_API int nlrom_step_device(nlrom_ctx* ctx, const double* r_bar, const double* rdot_bar, const double* f_ext,
                      const nlrom_simcfg* cfg, double* r_out, double* rdot_out, void* stream);

/* Timing hook for bench.py: replays `n_iters` fixed Newton iterations of the
 * captured CUDA graph at the state last set by nlrom_step*, and returns the
 * device time (CUDA events on the graph's stream) of the whole replay, plus the
 * device time of the dominant kernel (last decoder layer), averaged per
 * iteration. */
NLROM_API int nlrom_bench_iterations(nlrom_ctx* ctx, int n_iters, int flush_l2, float* ms_total, float* ms_dominant);

/* Per-replay timing for bench.py: replays the captured one-Newton-iteration graph n_iters
 * times at the current device state (set by nlrom_step* / nlrom_set_iterate), each bracketed
 * by CUDA events on the graph's stream, L2 flushed (256 MB write) before each replay outside
 * the events if flush_l2; ms_each[i] = device ms of replay i. */
NLROM_API int nlrom_bench_replays(nlrom_ctx* ctx, int n_iters, int flush_l2, float* ms_each);

/* The benchmarked graph without timing: n_iters replays of one fixed Newton iteration
 * (E at r, J, LU, r += dr) on the current device state. With nlrom_get_iterate /
 * nlrom_set_iterate this lets bench.py and tests check the exact timed graph against the
 * oracle (r after each iteration, phi at the iterate the iteration started from). */
NLROM_API int nlrom_iterate(nlrom_ctx* ctx, int n_iters);
/* r (n_sims x n) of the current iterate; phi (n_sims x n) and ||phi||_2 (n_sims) as evaluated
 * by the last E phase (any of the pointers may be NULL). */
NLROM_API int nlrom_get_iterate(nlrom_ctx* ctx, double* r, double* phi, double* norm);
/* Overwrite the current iterate r (n_sims x n); r_bar, rdot_bar, f_ext stay as set. */
NLROM_API int nlrom_set_iterate(nlrom_ctx* ctx, const double* r);

/* Device time per stage (CUDA events on the context stream, averaged over n_iters):
 * ms4[0] hidden jet chain, ms4[1] decoder output layer, ms4[2] vhp backward chain,
 * ms4[3] LU solve. Used by bench.py to pick and time the dominant kernel. */
NLROM_API int nlrom_bench_kernels(nlrom_ctx* ctx, int n_iters, int flush_l2, float* ms4);

/* Device time of one cubature launch over the context's cubature set (weighted element forces,
 * stiffness, reduced-force / reduced-stiffness partials) for all sims, L2 flushed before each
 * launch, averaged over n_iters; *bytes = the algorithmic bytes of that launch (SURVEY.md 8d
 * B_cub per sim x n_sims). bench.py reports *bytes / *ms against the HBM peak. */
NLROM_API int nlrom_bench_cubature(nlrom_ctx* ctx, int n_iters, int flush_l2, float* ms, double* bytes);

/* Neural-cubature training set (Eq. 18): for each of n_poses
 * poses rs (n_poses x n, row-major) the per-element reduced forces J~_e(r)^T f_e(u(r)) of ALL
 * T elements into F_out (n_poses x T x n) and, if u_out != NULL, u(r) into u_out (n_poses x N).
 * Replaces per-pose calls of elastic.element_reduced_force over all elements. */
NLROM_API int nlrom_train_forces(nlrom_ctx* ctx, const double* rs, int n_poses, double* F_out, double* u_out);

/* Number of kernel launches of one Newton iteration (for bench "gpu_launches"). */
NLROM_API int nlrom_launches_per_iteration(nlrom_ctx* ctx);

/* Number of decoder hidden layers that run on the tcgen05 kind::i8 Ozaki GEMM (batched
 * contexts; 0 = every layer on fp64 DMMA). bench.py uses it to pick the roofline peak. */
NLROM_API int nlrom_tc_layers(nlrom_ctx* ctx);

/* Which decoder GEMMs of a batched context run on the tcgen05 Ozaki GEMM: out[0] = hidden jet
 * layers, out[1] = output layer (0 / 1), out[2] = shared-real vhp backward layers. */
NLROM_API int nlrom_tc_info(nlrom_ctx* ctx, int* out);

/* Profiling: prefix-graph timing of one Newton iteration. For k = 1..min(cap, launches) the
 * first k launches are captured as a graph and timed over n_iters replays (L2 flushed before
 * each): ms[k-1] - ms[k-2] is launch k's marginal in-graph cost. names receives the kernel
 * names ('\n'-separated); n_launches the number of prefixes timed. */
NLROM_API int nlrom_bench_prefix(nlrom_ctx* ctx, int n_iters, int flush_l2, int cap, float* ms, char* names,
                                 int names_len, int* n_launches);

/* Test hook: fills the shared memory of every SM with NaN bit patterns (one resident
 * max-shared-memory CTA per SM, synchronous), so that a later kernel reading shared memory it
 * never wrote is caught deterministically by the parity tests. No context needed. */
NLROM_API int nlrom_debug_poison_shared_memory(int device);

/* The context's CUDA stream (cudaStream_t) -- every call above is ordered on it; a host
 * that interleaves its own collectives (NCCL) with the coupled phases below uses it. */
NLROM_API int nlrom_stream(nlrom_ctx* ctx, void** stream);

/* ---------------------------------------------------------------------------------------
 * Substructured scene (SURVEY.md §8e, cfg4 puffer ball, PAPER.md:84/580/603). No reference
 * interface exists (the reference has no coupled scenes); the model is
 * oracle/coupled.py. This context's n_sims sims are strings [lo, hi) of a scene of k_total
 * strings sharing the networks, attached to a translating core (3 DOFs) replicated on every
 * rank. One Newton iteration on every rank:
 *   nlrom_coupled_eval(ctx, cfg, 1, partial)          16 doubles into device buffer `partial`
 *   allreduce-sum(partial -> total) over the ranks     (host: NCCL on nlrom_stream; skip at 1 rank)
 *   nlrom_coupled_update(ctx, cfg, total, 1, 1.0, 0)  Schur solve for the core, r_s / c update
 * mode 0: residual norm only (after eval(jacobian=0)); mode 1: direction + apply(t);
 * mode 2: re-apply the last direction with step t (line search). norm_host (optional) receives
 * ||[phi_1 .. phi_k, phi_c]||_2 (synchronises). */
NLROM_API int nlrom_coupled_setup(nlrom_ctx* ctx, const double* R /* n_sims x 3 x 3, string -> world */,
                                  const double* f_world /* n_sims x N */, int k_total, double m_core,
                                  double k_core, const double* f_core /* 3 */);
NLROM_API int nlrom_coupled_begin(nlrom_ctx* ctx, const double* r_bar, const double* rdot_bar,
                                  const double* c_bar /* 3 */, const double* cdot_bar /* 3 */,
                                  const nlrom_simcfg* cfg);
NLROM_API int nlrom_coupled_eval(nlrom_ctx* ctx, const nlrom_simcfg* cfg, int jacobian, double* partial_dev);
NLROM_API int nlrom_coupled_update(nlrom_ctx* ctx, const nlrom_simcfg* cfg, const double* total_dev, int mode,
                                   double t, double* norm_host);
NLROM_API int nlrom_coupled_read(nlrom_ctx* ctx, double dt, double* r, double* rdot, double* core_c,
                                 double* core_cdot);
/* kernel launches of one coupled Newton iteration (eval graph + update) */
NLROM_API int nlrom_coupled_launches(nlrom_ctx* ctx);

/* ---------------------------------------------------------------------------------------
 * Full-space StVK implicit Euler (elastic.fullspace_step; SURVEY.md §8f
 * rank 2: ground truth for trajectory error and the pose generator's integrator,
 * posegen.generate_poses SPEC.md:395-403). One Newton solve per step of
 *   M (v' - v) / dt + (alpha M + beta K(u')) v' + f_int(u') = f_ext,   u' = u + dt v',
 * unknown v'; Newton matrix (1 + alpha dt) M + (beta dt + dt^2) K(u') (dK/du v' dropped:
 * it changes the convergence rate only, not the solution); each linear system by Jacobi-
 * preconditioned CG in one cooperative kernel (deterministic reductions). The mesh data are
 * those of nlrom_model_desc (free-DOF numbering by vert_dof, Dirichlet by elimination). */
typedef struct nlrom_fs nlrom_fs;

typedef struct {
  int n_verts, n_tets;
  const int* tets;          /* (T,4)                                           */
  const int* vert_dof;      /* (V,) free-vertex index or -1 if fixed           */
  const double* Dm_inv;     /* (T,3,3) row-major                               */
  const double* vol;        /* (T,)                                            */
  const double* mass;       /* (N,) lumped, free DOFs                          */
  double mu, lambda, alpha, beta;
} nlrom_fs_desc;

typedef struct {
  double dt;
  double newton_tol;        /* ||residual force||_2 <= newton_tol * max(1, ||f_ext||_2) */
  int max_iters;            /* Newton iterations before NLROM_ERR_NEWTON       */
  double cg_tol;            /* relative CG residual                            */
  int cg_max_iters;
} nlrom_fs_cfg;

typedef struct {
  int iters;                /* Newton iterations                               */
  int cg_iters;             /* CG iterations, all Newton iterations            */
  double res_norm;          /* final ||residual force||_2                      */
  double energy;            /* StVK energy at u'                               */
} nlrom_fs_info;

NLROM_API int nlrom_fs_create(nlrom_fs** out, int device, const nlrom_fs_desc* desc);
NLROM_API void nlrom_fs_destroy(nlrom_fs* fs);
NLROM_API const char* nlrom_fs_last_error(const nlrom_fs* fs);
/* (u, v) -> (u', v'), all (N,) */
NLROM_API int nlrom_fs_step(nlrom_fs* fs, const double* u, const double* v, const double* f_ext,
                            const nlrom_fs_cfg* cfg, double* u_out, double* v_out, nlrom_fs_info* info);
/* StVK energy and internal force at u (f_int nullable) */
NLROM_API int nlrom_fs_energy_force(nlrom_fs* fs, const double* u, double* energy, double* f_int);

#ifdef __cplusplus
}
#endif
#endif /* NLROM_B200_H */
