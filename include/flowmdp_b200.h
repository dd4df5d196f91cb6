/*
 * flowmdp_b200.h -- C ABI of the B200-native planner hot path
 * (MDP model build + value-iteration solve of arXiv 2109.00857).
 *
 * The reference (`flowmdp`, pure Python/numpy) has no native plugin layer;
 * its drop-in boundary is the Python API of model_builder.py / solver.py.
 * Every entry point below replaces one reference function; the citation
 * names the file:line (relative to /root/reference/pkg/src/flowmdp) it
 * stands in for.  Python binds these with ctypes
 * (paper_2109_00857_b200/_lib.py); INTEGRATION.md shows the binding a
 * maintainer of the reference would add.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers (cudaMalloc / torch storage)
 *     unless the parameter name starts with `h_`.
 *   - `stream` is a cudaStream_t passed as void*; NULL = legacy stream.
 *   - Every function returns an fm_status; on failure fm_last_error()
 *     returns a thread-local message.  No C++ exception crosses the ABI.
 *   - Layouts match the reference's numpy arrays (C-contiguous):
 *       mean   f64 [nt][ny][nx][2]          environment.py:114-131
 *       modes  f64 [n_modes][nt][ny][nx][2]
 *       coeffs f64 [nt][n_real][n_modes]
 *       g      f64 [nt][ny][nx]             environment.py:163-173
 *       mask   u8  [nt][ny][nx]             environment.py:176-184
 *   - State index s = t*N_c + j*nx + i, SINK = N_g = nt*N_c
 *     (environment.py:9-14).
 */
#ifndef FLOWMDP_B200_H
#define FLOWMDP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    FM_OK = 0,
    FM_SUBGRID_OVERFLOW = 1, /* ContractViolation, model_builder.py:430-438 */
    FM_BAD_ARG = 2,          /* ContractViolation (argument contract)       */
    FM_CUDA_ERROR = 3,
    FM_CAPACITY = 4          /* output buffer too small; *needed reported   */
} fm_status;

enum { FM_OBJ_TIME = 0, FM_OBJ_ENERGY = 1, FM_OBJ_NET_ENERGY = 2 };

/* Grid geometry (environment.py:30-49, GridSpec). */
typedef struct {
    int32_t nx, ny, nt;
    double dx, dt;
    double ox, oy; /* origin */
} fm_grid;

/* Reduced-order (DO) velocity field + scalar mean + obstacle mask
 * (environment.py:106-184).  Device pointers. */
typedef struct {
    const double *mean, *modes, *coeffs, *g;
    const uint8_t *mask;
    int32_t n_modes, n_real;
} fm_env;

/* Per-action constants computed on the host exactly as the reference does
 * (ActionSpace.vectors/speeds, environment.py:220-233; step_flat reward
 * bases, model_builder.py:350-358).  Device pointer to n_actions records. */
typedef struct {
    double ax, ay;      /* F*(cos th, sin th)                                */
    double base;        /* time: -dt; energy: (-(c_f*f*f))*dt; net: unused   */
    double base_hit;    /* base + r_term (time / energy)                      */
    double neg_cff;     /* -(c_f*f*f)   (net_energy)                          */
    double pad;
} fm_action;

/* Reward configuration (model_builder.py:54-79) and mission target. */
typedef struct {
    int32_t objective;  /* FM_OBJ_* */
    double c_f, c_r, r_term, r_outbound;
    int32_t target_i, target_j;
} fm_reward;

/* Device-resident compact model produced by fm_build.
 * Rows are (t, c, a) for the cells c of [cell0, cell0 + ncell) -- the
 * whole layer (cell0 = 0, ncell = N_c) or one GPU's row strip (rows j0..j1:
 * cell0 = j0*nx, ncell = (j1-j0)*nx) -- with
 * row id = (t*ncell + c - cell0)*n_actions + a.
 * Entry word = (slot << 16) | count; slot indexes the (2hx+1)(2hy+1)
 * displacement window row-major in (dj, di), slot == n_slots is the OUT
 * slot (successor SINK).  probability = count / n_real.
 * Entries of a row are contiguous and slot-ascending (= column-ascending,
 * SINK last: the canonical order of model_builder.py:474-501). */
typedef struct {
    int32_t nx, ny, nt, n_actions, n_real;
    int32_t hx, hy;            /* sub-grid half widths used for slots        */
    int32_t cell0, ncell;      /* cells whose rows the model holds           */
    int64_t n_rows;            /* nt*ncell*n_actions                         */
    uint64_t *row_ptr;         /* [n_rows] first entry of each row           */
    uint16_t *row_nnz;         /* [n_rows]                                   */
    double *reward;            /* [n_rows] R_{a,t}[s] = sum_r / n_real       */
    uint32_t *entries;         /* [capacity]                                 */
    uint64_t capacity;         /* entries allocated                          */
    uint64_t *d_nnz;           /* [1] device counter: entries emitted        */
} fm_model;

/* Build arguments: one slab range [t0, t1) and one row strip [j0, j1)
 * (spatial sharding across GPUs: SURVEY.md section 8(e)). */
typedef struct {
    fm_grid grid;
    fm_env env;
    fm_reward reward;
    const fm_action *actions; /* device [n_actions] */
    int32_t n_actions;
    int32_t hx, hy;           /* sub-grid (model_builder.py:82-112)          */
    int32_t rx, ry;           /* obstacle gate radius (model_builder.py:218) */
    const int32_t *mask_sat;  /* device [nt][ny+1][nx+1], from fm_mask_sat   */
    int32_t t0, t1, j0, j1;
    uint32_t *viol_flags;     /* device [nt*n_actions], zeroed by caller     */
    uint32_t *task_counter;   /* device [1] scratch, zeroed by fm_build      */
    const int32_t *d_gate_r;  /* device [rx, ry] from fm_gate_radius, or NULL
                                 to use rx/ry above                          */
    /* Optional fast-path enablers (both may be left 0 / negative: the build
     * is then fully checked per transition).  Neither changes any output.
     *  h_actions: HOST copy of `actions`.  With it the build proves, per
     *    launch, whether every per-transition reward is a dyadic value whose
     *    sequential f64 sum over n_real realizations is exact; if so the
     *    reward sum (model_builder.py:457-458) is formed from the histogram
     *    counts instead of per transition (bit-identical by exactness).
     *  vmax_x, vmax_y: the exact maxima of fm_velocity_max (>= 0), or < 0 if
     *    unknown.  With them (and h_actions) the build proves by monotonicity
     *    of rounding that no in-domain landing can leave the sub-grid window
     *    (no overflow check needed) and that cell indices fit in 2^30, so the
     *    lean path floors with one round-down add instead of F2I. */
    const fm_action *h_actions;
    double vmax_x, vmax_y;
    /* Optional (NULL = none): the velocity envelope of fm_velocity_scan
     * covering the build's slabs x strip.  With it (and the two enablers
     * above) lean cells are built per (cell, realization) instead of per
     * (cell, action, realization): each realization is binned once against
     * the action set's landing thresholds; the counts are unchanged. */
    const int32_t *envelope;
    /* SMs' worth of thread blocks the persistent build grid leaves free, so
     * kernels on other streams (a pipelined backward solve, the halo
     * exchange's communication kernels) run while the build proceeds.  0 =
     * the whole GPU. */
    int32_t reserve_sms;
    /* Which tasks of [t0, t1) x [j0, j1) this call builds: bit 0 = lean
     * tasks (no obstacle or dead cell near any row of the task), bit 1 =
     * obstacle tasks; 0 = all (same as 3).  A pipelined caller builds the
     * obstacle tasks of the whole range first and then the lean tasks slab
     * group by slab group, so each group completes with one short launch
     * (its rows, and the entries it appends, are final when that launch
     * ends).  Builds whose tasks cannot be told apart (no proven fast path)
     * do everything in the lean phase. */
    int32_t phases;
    /* Row rewards (model_builder.py:457-458, 462-464): 0 = the reference's
     * sequential f64 sum over realizations in ascending order (bit-exact;
     * formed from the counts only when provably exact); 1 = formed from the
     * per-slot counts (sum over landing slots of count x reward) whenever the
     * fast path is proven -- counts, columns and probabilities stay
     * bit-exact, rewards agree to rounding (relative ~1e-13, north_star
     * allows 1e-5); lets net-energy rows take the binned build. */
    int32_t reward_mode;
} fm_build_args;

/* Sub-grid overflow report (message of model_builder.py:433-438). */
typedef struct {
    int32_t t, a, di, dj;
} fm_violation;

/* ---- version / errors -------------------------------------------------- */
int32_t fm_abi_version(void);
const char *fm_last_error(void);
/* Number of kernels this library has launched in the process so far. */
int64_t fm_kernel_launches(void);

/* ---- sub-grid sizing ---------------------------------------------------- */
/* compute_subgrid's exact scan, model_builder.py:392-396: d_out2 receives
 * max |v_x|, max |v_y| over every (t, realization, cell) with the
 * reconstruction order of environment.py:293-297.  d_out2 must be zeroed. */
int32_t fm_velocity_max(fm_grid grid, fm_env env, double *d_out2, void *stream);
/* The same scan over the cells of rows [j0, j1) only (one GPU's strip: the
 * global maximum is the max over strips, e.g. an all-reduce). */
int32_t fm_velocity_max_rows(fm_grid grid, fm_env env, int32_t j0, int32_t j1,
                             double *d_out2, void *stream);
/* The scan over layers [t0, t1) x rows [j0, j1), max-accumulated into d_out2:
 * lets a caller scan each time slab as its host->device copy lands (the
 * maxima over slabs are the full scan's). */
int32_t fm_velocity_max_slab(fm_grid grid, fm_env env, int32_t t0, int32_t t1, int32_t j0, int32_t j1,
                             double *d_out2, void *stream);
/* fm_velocity_max_slab plus, when d_envelope is not NULL, the per-(t, cell)
 * velocity envelope of the scanned cells: d_envelope is int32 [nt][N_c][4]
 * (x_lo, x_hi, y_lo, y_hi as order-preserving encodings of f32 bounds that
 * contain every reconstructed v(t, r, cell) of environment.py:293-297).
 * fm_build bins the realizations of a cell against it (fm_build_args.
 * envelope).  Same reference function as above (model_builder.py:392-396):
 * the envelope is a by-product of the scan. */
int32_t fm_velocity_scan(fm_grid grid, fm_env env, int32_t t0, int32_t t1, int32_t j0, int32_t j1,
                         double *d_out2, int32_t *d_envelope, void *stream);

/* The same scan without the exact f64 recompute: d_out4 = (lo_x, hi_x,
 * lo_y, hi_y), each combined by atomic max into the caller's (zeroed)
 * buffer, with lo_c <= max |v_c| <= hi_c (the f32 envelope widened by the
 * per-cell rounding bound; hi = +inf when an input is not finite), plus the
 * envelope as above.  compute_subgrid (model_builder.py:376-399) needs only
 * ceil((max|v_c| + f_max) dt / dx): when lo and hi give the same half width
 * it is exact, and hi is a valid bound for fm_build's proofs (vmax_x/y);
 * otherwise the caller runs fm_velocity_scan. */
int32_t fm_velocity_bounds(fm_grid grid, fm_env env, int32_t t0, int32_t t1, int32_t j0, int32_t j1,
                           double *d_out4, int32_t *d_envelope, void *stream);

/* Segmented max-abs used by velocity_bound (environment.py:404-419):
 * d_out[s] = max_k |src[(s / inner) * outer_stride + (s % inner) * inner_stride
 *                     + k * elem_stride]|, k in [0, seg_len). */
int32_t fm_maxabs_segments(const double *src, int64_t n_seg, int64_t seg_len,
                           int64_t elem_stride, int64_t inner, int64_t outer_stride,
                           int64_t inner_stride, double *d_out, void *stream);

/* Summed-area table of the obstacle mask, per time layer
 * (box queries replace _dilate, model_builder.py:262-271). */
int32_t fm_mask_sat(const uint8_t *mask, int32_t nt, int32_t ny, int32_t nx,
                    int32_t *sat, void *stream);

/* ---- model build -------------------------------------------------------- */
/* K_build: the fused per-(state, action, realization) sweep that replaces
 * build_model -> _timeslice_blocks -> transition_sweep / finalize_rewards /
 * count_nnz / assemble_coo (model_builder.py:402-580).  Returns
 * FM_CAPACITY with *h_needed set when model->capacity is too small (the
 * caller re-allocates and calls again; results are deterministic).
 * FM_SUBGRID_OVERFLOW fills *h_viol like the reference's ContractViolation. */
int32_t fm_build(const fm_build_args *h_args, fm_model *h_model,
                 uint64_t *h_needed, fm_violation *h_viol, void *stream);
/* fm_build = fm_build_launch (asynchronous) + fm_build_check (synchronous:
 * census, capacity and overflow report).  Work that consumes the model
 * (e.g. fm_solve_backward, which never reads past `capacity`) may be queued
 * between the two; its results are valid only if the check returns FM_OK. */
int32_t fm_build_launch(const fm_build_args *h_args, fm_model *h_model, void *stream);
int32_t fm_build_check(const fm_build_args *h_args, fm_model *h_model,
                       uint64_t *h_needed, fm_violation *h_viol, void *stream);

/* Obstacle-gate radius without a host round trip (model_builder.py:218-223,
 * environment.py:404-419): inputs are the fm_maxabs_segments results
 * max|mean| [nt][2], max|coeff| [nt][n_modes], max|mode| [n_modes][nt][2];
 * d_out2 = (rx, ry), d_bound2 (optional) = velocity_bound. */
int32_t fm_gate_radius(fm_grid grid, const double *meanmax, const double *coefmax,
                       const double *modemax, int32_t n_modes, double f_max,
                       int32_t *d_out2, double *d_bound2, void *stream);

/* Export to the reference's canonical COO blocks, SparseModel layout
 * (model_builder.py:157-178, 474-501, 568-573): blocks in [a][t] order,
 * concatenated.  d_block_off[a*nt + t] = first entry of block (a, t),
 * d_block_off[n_actions*nt] = nnz.  Rows/cols u32, vals f64 = count/N_rv,
 * rewards f64 [a][N_g].  d_scratch: (n_rows + 1) uint64. */
int32_t fm_export_coo(const fm_model *h_model, uint64_t *d_scratch,
                      uint64_t *d_block_off, uint32_t *rows, uint32_t *cols,
                      double *vals, double *rewards, void *stream);

/* Model file image (io.write_model, io.py:213-244) from the fm_export_coo
 * arrays: per (action, time) block rows u32, cols u32, vals f32, then the
 * f32 rewards, written at byte `header_bytes` of d_img (the caller writes
 * the header: magic, version/n_states/n_actions/nt, nnz, block offsets). */
int32_t fm_model_image(const uint64_t *d_block_off, int32_t n_blocks,
                       const uint32_t *rows, const uint32_t *cols, const double *vals,
                       uint64_t nnz, const double *rewards, uint64_t n_rewards,
                       uint64_t header_bytes, unsigned char *d_img, void *stream);

/* ---- rollout ------------------------------------------------------------ */
/* Ensemble rollout (rollout.py:107-208): trajectory k follows the policy in
 * realization realizations[k] from the start cell, one step_flat per time
 * index (model_builder.py:286-369).  Row s of trajectory k (s < n_rows[k])
 * is (departure cell, action, cause code CAUSE_*, reward, cumulative
 * reward) at [k * max_rows + s]; final_cell[k] = arrival cell when the last
 * row reached the target, else -1.  The start cell must not be masked at
 * t = 0 (the caller handles that case, rollout.py:124-136). */
typedef struct {
    fm_grid grid;
    fm_env env;
    fm_reward reward;
    const fm_action *actions; /* device [n_actions] */
    int32_t n_actions;
    const int32_t *mask_sat;  /* device, fm_mask_sat */
    const int32_t *d_gate_r;  /* device [rx, ry], fm_gate_radius */
    const uint16_t *policy;   /* device [N_g] */
    int32_t start_i, start_j;
    const int32_t *realizations; /* device [n_traj] */
    int32_t n_traj, max_rows;    /* max_rows >= nt */
    int32_t *row_cell;
    int16_t *row_action;
    int8_t *row_cause;
    double *row_reward, *row_cum;
    int32_t *n_rows, *final_cell;
} fm_rollout_args;

int32_t fm_rollout(const fm_rollout_args *h_args, void *stream);

/* ---- solve -------------------------------------------------------------- */
/* Backward-in-time Bellman sweep over the compact model, layers
 * t = t_hi-1 .. t_lo (value_iteration's fixed point, solver.py:75-109,
 * reached in one pass because the time-expanded model is a DAG).
 * values: f64 [N_g + 1] (SINK last, must hold 0), policy: u16 [N_g].
 * Per row: S = +0; S += p_k * V[col_k] in entry order; Q = R + S; first
 * maximising action wins (np.argmax, solver.py:101-102). */
int32_t fm_solve_backward(const fm_model *h_model, int32_t t_lo, int32_t t_hi,
                          double *values, uint16_t *policy, void *stream);

/* Multi-GPU strip solve ("optional halo descriptors").  The
 * model is one rank's y-strip (fm_model.cell0 / ncell, whole rows); its
 * layers t = t_hi-1 .. t_lo are solved on `stream` as fm_solve_backward
 * does, and after each layer -- V_t of the strip's rows enqueued -- `halo`
 * is called with (user, t, stream) before layer t-1 is launched.  The hook
 * enqueues the exchange of layer t's halo: it sends rows [j0, j0 + h_y) and
 * [j1 - h_y, j1) of V_t and receives rows [j0 - h_y, j0) and [j1, j1 + h_y)
 * into `values` (full-grid layout, state (t, j, i) at t*N_c + j*n_x + i),
 * ordered with `stream` (e.g. ncclGroupStart; ncclSend / ncclRecv on the
 * neighbours; ncclGroupEnd on `stream`, or peer copies / P2P stores), and
 * returns 0; nonzero aborts with FM_BAD_ARG.  halo = NULL: no exchange (one
 * rank).  Replaces the reference's per-slab fork pool (model_builder.py:
 * 548-566) on the solve side; sharding.py's StripPlanner is the Python
 * caller of the same scheme. */
typedef int32_t (*fm_halo_fn)(void *user, int32_t t, void *stream);
int32_t fm_solve_backward_halo(const fm_model *h_model, int32_t t_lo, int32_t t_hi, double *values,
                               uint16_t *policy, fm_halo_fn halo, void *user, void *stream);

/* One backward layer restricted to rows j in [j0, j1) (multi-GPU strips). */
int32_t fm_solve_layer(const fm_model *h_model, int32_t t, int32_t j0, int32_t j1,
                       double *values, uint16_t *policy, void *stream);
/* The count -> probability table fl(q / n_real), q = 0..n_real, into
 * d_ptab [n_real + 1] -- built once per model so a strip solve's layers
 * (fm_solve_layer_tab) launch one kernel each. */
int32_t fm_prob_table(int32_t n_real, double *d_ptab, void *stream);
int32_t fm_solve_layer_tab(const fm_model *h_model, const double *d_ptab, int32_t t, int32_t j0, int32_t j1,
                           double *values, uint16_t *policy, void *stream);

/* General CSR (explicit f64 probabilities) for host-supplied models
 * (io.read_model widens f32 vals, io.py:280-292): per action a, rows of
 * the non-sink states in state order; entries in reference triplet order. */
typedef struct {
    int64_t n_g;
    int32_t n_actions, nt;
    const int64_t *row_ptr;   /* [n_actions][n_g + 1]                      */
    const uint32_t *cols;     /* [nnz]                                     */
    const double *vals;       /* [nnz]                                     */
    const double *rewards;    /* [n_actions][n_g]                          */
} fm_csr;

/* Row pointers from concatenated per-action COO rows: rows (u32) must be
 * non-decreasing inside each action's segment [seg_off[a], seg_off[a+1]).
 * d_sorted_flag receives 0 if that is violated. */
int32_t fm_csr_row_ptr(const uint32_t *rows, const int64_t *h_seg_off, int32_t n_actions,
                       int64_t n_g, int64_t *row_ptr, int32_t *d_sorted_flag,
                       void *stream);

/* Jacobi value iteration with the reference's stopping rule
 * (solver.py:75-109): sweeps from v = 0 until max|dv| < epsilon or
 * max_iter; v0/v1 are ping-pong buffers [n_g+1] (v0 zeroed by the call);
 * d_stats = {iterations (i64), residual bits (u64)} written on device.
 * The converged iterate ends in v0 if iterations is even, else v1. */
int32_t fm_jacobi(const fm_csr *h_csr, double epsilon, int32_t max_iter,
                  double *v0, double *v1, uint64_t *d_stats, void *stream);

/* Greedy policy at given values (extract_policy, solver.py:112-119). */
int32_t fm_greedy(const fm_csr *h_csr, const double *values, uint16_t *actions, void *stream);

/* Fixed-policy evaluation (policy_value, solver.py:122-158). */
int32_t fm_policy_value(const fm_csr *h_csr, const uint16_t *policy, double epsilon,
                        int32_t max_iter, double *v0, double *v1, uint64_t *d_stats,
                        void *stream);

/* ---- measurement helpers ------------------------------------------------- */
/* FP64 add/mul pipe throughput probe (roofline denominator): runs
 * `iters` dependent-chain-free DADD/DMUL pairs per thread. */
int32_t fm_fp64_probe(double *d_sink, int32_t blocks, int32_t iters, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* FLOWMDP_B200_H */
