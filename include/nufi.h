/*
 * nufi.h -- C-ABI of the B200-native NuFI hot path (libnufi_b200.so).
 *
 * Drop-in boundary for the reference's per-step rho loop
 * (/root/reference/pkg/src/vpflow).  Plain C types only:
 * pointers, sizes, doubles.  No torch types cross this boundary.
 *
 * Every entry point returns an int status:
 *   NUFI_OK (0), NUFI_ERR_USAGE (1) -> vpflow UsageError            errors.py:8-9
 *               NUFI_ERR_NUMERICAL (2) -> NumericalConsistencyError  errors.py:16-17
 *               NUFI_ERR_CONFIG (3) -> ConfigError                   errors.py:12-13
 *               NUFI_ERR_CUDA (4), NUFI_ERR_COMM (5)
 * and nufi_last_error() returns a thread-local message for the last failure.
 *
 * Buffers are caller-owned.  Pointer arguments may be host or device memory
 * (resolved through unified addressing); host outputs are complete when the
 * call returns, device outputs are ordered on the handle's stream.
 * One host thread drives one handle; one handle per GPU / rank.
 */
#ifndef NUFI_H
#define NUFI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NUFI_ABI_VERSION 1

#define NUFI_OK 0
#define NUFI_ERR_USAGE 1
#define NUFI_ERR_NUMERICAL 2
#define NUFI_ERR_CONFIG 3
#define NUFI_ERR_CUDA 4
#define NUFI_ERR_COMM 5

#define NUFI_MAX_CENTERS 4

/* nufi_config.flags */
#define NUFI_FLAG_F32_HISTORY 1 /* PotentialHistory(dtype=float32), spline.py:118-125: every stored
                                   coefficient is rounded to float32 (the trace reads it as double) */

/* nufi_trace modes */
#define NUFI_TRACE_FAST 0   /* production arithmetic (FMA, cell-centred polynomial form) */
#define NUFI_TRACE_PARITY 1 /* reference operation order, no FMA: bit-exact vs kernels.py */

/* One velocity axis of f0: v^power * sum_m weights[m] * N(v; centers[m], 1).
 * Mirrors VelocityProfile, initial.py:25-56 (power in {0, 2}, weights > 0). */
typedef struct nufi_profile {
    int32_t n_centers;
    int32_t power;
    double centers[NUFI_MAX_CENTERS];
    double weights[NUFI_MAX_CENTERS];
} nufi_profile;

/* GridSpec (grids.py:18-59) + InitialCondition (initial.py:72-106) + tau
 * (spline.py:118-120) + the history capacity (PotentialHistory, spline.py:108-155).
 * rho_bar: background density; NaN -> computed on the device with the
 * quadrature of background_density (initial.py:187-208).
 * v_blocks: fixed number B of velocity blocks whose partial sums are combined
 * in a fixed order (0 -> default); a rank traces blocks [block_lo, block_hi). */
typedef struct nufi_config {
    int32_t d;
    int32_t Nx;
    int32_t Nv;
    int32_t n_max; /* largest step index; history capacity n_max + 1 slabs */
    double L;
    double vmax;
    double tau;
    double alpha;
    double k;
    double rho_bar;
    nufi_profile profiles[3];
    int32_t v_blocks;
    int32_t block_lo;
    int32_t block_hi;
    int32_t flags; /* NUFI_FLAG_* */
} nufi_config;

typedef struct nufi_handle nufi_handle;

/* ---- lifecycle ----------------------------------------------------------- */

/* Validates cfg like GridSpec.__post_init__ (grids.py:28-34),
 * VelocityProfile.__post_init__ (initial.py:33-39),
 * InitialCondition.__post_init__ (initial.py:89-106), PotentialHistory
 * (spline.py:119-120) and fit_spline's Nx >= 4 (spline.py:73-74); allocates the
 * device-resident history.  stream: a cudaStream_t, or NULL for a private one. */
int nufi_create(const nufi_config *cfg, int device, void *stream, nufi_handle **out);
int nufi_destroy(nufi_handle *h);
const char *nufi_last_error(void);
int nufi_abi_version(void);
int nufi_sync(nufi_handle *h);
/* background density actually used (FlowContext.rho_bar, flow.py:36-39) */
int nufi_rho_bar(nufi_handle *h, double *out);
/* Install the initial condition of cfg (alpha, k, profiles, rho_bar; the grid
 * fields must match the handle) -- binding a FlowContext to a history. */
int nufi_set_initial_condition(nufi_handle *h, const nufi_config *cfg);
/* Grow the history capacity to at least `slabs` (PotentialHistory's doubling
 * growth, spline.py:136-139; stored rows are preserved). */
int nufi_reserve(nufi_handle *h, int64_t slabs);
int64_t nufi_capacity(nufi_handle *h);

/* ---- history (PotentialHistory, spline.py:108-155) ----------------------- */

int nufi_history_len(nufi_handle *h, int64_t *len);
/* Replace the history by `count` coefficient slabs (count, Nx^d) row-major. */
int nufi_load_history(nufi_handle *h, const double *coeffs, int64_t count);
/* Copy slabs [first, first+count) out, (count, Nx^d) row-major. */
int nufi_get_history(nufi_handle *h, double *coeffs, int64_t first, int64_t count);
/* PotentialHistory.append(SplineField) (spline.py:132-142): one fitted slab. */
int nufi_append_coeffs(nufi_handle *h, const double *coeffs);
/* Drop slabs so that len == count (count <= len). */
int nufi_truncate_history(nufi_handle *h, int64_t count);

/* ---- the hot path -------------------------------------------------------- */

/* compute_rho (density.py:72-91) for a single rank: traces every quadrature
 * point of the grid with Psi-tilde through history rows 0..n-1 (needs
 * len >= n, else NUFI_ERR_USAGE like _require_history, flow.py:55-62),
 * evaluates f0 at the foot point and reduces over v.
 * rho_out: Nx^d doubles (neutralised); stats3 = {neutralization, f_min, f_max};
 * evals (optional) += Nx^d * Nv^d * n (FlowContext.field_evals, flow.py:89). */
int nufi_rho(nufi_handle *h, int64_t n, double *rho_out, double *stats3, int64_t *evals);

/* Multi-rank split of nufi_rho.  partials: DEVICE buffer of v_blocks * (Nx^d + 2)
 * doubles: rows [b][Nx^d] of per-block v-sums followed by v_blocks (min, max)
 * pairs.  This rank writes its blocks [block_lo, block_hi) and zeros elsewhere, so an
 * elementwise SUM allreduce of the ranks' buffers is exact (one nonzero
 * contributor per element) and the combine is rank-count independent. */
int nufi_rho_partials(nufi_handle *h, int64_t n, double *partials, int64_t *evals);
/* Multi-rank step tail: combine the (allreduced) block partials, neutralise,
 * then exactly nufi_field_update's work, appending slab n (requires len == n).
 * Every rank runs it redundantly and so holds the full history. */
int nufi_step_finish(nufi_handle *h, int64_t n, const double *partials, double *rho_out, double *E_out,
                     double *W_out, double *stats3);
/* Stream-ordered variant of nufi_step_finish for a host loop that enqueues a whole
 * run ahead (trace -> allreduce -> finish per step, no host synchronisation):
 * outputs must be DEVICE buffers (or NULL); a failing step (non-neutral rho) sets
 * a device flag that makes every later field update a no-op.  Call
 * nufi_check_status() at the end: NUFI_ERR_NUMERICAL if any step failed (the
 * history length is then reset to the fields actually appended). */
int nufi_step_finish_async(nufi_handle *h, int64_t n, const double *partials, double *rho_out, double *E_out,
                           double *W_out, double *stats3);
int nufi_check_status(nufi_handle *h);
/* Multi-rank d = 1 runs with the exchange FUSED into the persistent kernel (no NCCL,
 * no host loop): every rank's kernel stores its block sums straight into every peer's
 * exchange table over NVLink (CUDA IPC peer memory), raises one arrival flag per peer
 * (release, system scope) and waits for all peers' flags, then runs the identical tail.
 * nufi_mg_setup: the handle's block range must be rank's share of B (B % world == 0);
 * writes this rank's IPC handle (nufi_mg_handle_size() bytes) to ipc_handle_out.
 * emulate != 0: all `world` ranks are CTA groups of ONE cooperative launch on this device
 * (handle covers all blocks) -- the same protocol, for testing on one GPU.
 * nufi_mg_connect: the world x nufi_mg_handle_size() bytes of all ranks' handles
 * (e.g. all-gathered); afterwards nufi_run runs the fused multi-rank kernel.  A rank
 * that never arrives trips a 4 s watchdog: nufi_run returns NUFI_ERR_COMM. */
int nufi_mg_setup(nufi_handle *h, int world, int rank, int emulate, void *ipc_handle_out);
int nufi_mg_connect(nufi_handle *h, const void *ipc_handles);
int nufi_mg_handle_size(void);
/* Leave multi-rank mode (frees the exchange buffers, closes the peers' IPC mappings); the
 * handle then runs single-rank kernels again (e.g. after the ranks agreed to fall back to
 * the per-step NCCL loop). */
int nufi_mg_teardown(nufi_handle *h);

/* Multi-rank d = 2, 3 step with the exchange FUSED into the block reduce (no NCCL):
 * after nufi_mg_setup / nufi_mg_connect on a d >= 2 handle, one call enqueues step n
 * (n == history length): trace of this rank's blocks -> block sums STORED into every
 * rank's exchange table over peer memory + system-scope arrival counters -> the step
 * tail, which waits for every peer's counters (4 s watchdog: NUFI_ERR_COMM from
 * nufi_check_status).  Outputs are device buffers (any may be NULL); no host sync.
 * Emulated handles (emulate != 0) run every virtual rank's exchange on this device. */
int nufi_mg_step_async(nufi_handle *h, int64_t n, double *rho_out, double *E_out, double *W_out,
                       double *stats3);

/* Fixed-order combine of the (allreduced) block partials -> rho, stats3. */
int nufi_rho_finish(nufi_handle *h, const double *partials, double *rho_out, double *stats3);
int64_t nufi_partials_len(nufi_handle *h); /* v_blocks * (Nx^d + 2) */

/* solve_poisson (poisson.py:90-112) + fit_spline (spline.py:71-86) +
 * PotentialHistory.append (spline.py:132-142) + electric_energy
 * (poisson.py:115-120) + E at the nodes (SplineField.eval_E_many at
 * x_node_matrix, spline.py:50-52 / kernels.py:102-123), on the device.
 * rho: Nx^d neutral densities.  Outputs (optional, NULL to skip):
 * W_out (1), E_out (Nx^d * d, row-major (node, axis)), coeffs_out (Nx^d).
 * Returns NUFI_ERR_NUMERICAL (history unchanged) if |mean rho| > 1e-8 max|rho|. */
int nufi_field_update(nufi_handle *h, const double *rho, double *W_out, double *E_out,
                      double *coeffs_out);

/* The tail's reference operations one by one (Nx^d doubles, host or device buffers):
 * solve_poisson (poisson.py:90-112): phi nodal values, the phi spectrum
 * fftn(rho)/N^d/k^2 (zero and Nyquist modes dropped; spec_re / spec_im optional) and the
 * electric energy (poisson.py:115-120, optional); NUFI_ERR_NUMERICAL if |mean rho| >
 * 1e-8 max|rho|.  fit_spline (spline.py:71-86): periodic cubic B-spline coefficients
 * of nodal values.  Neither touches the history. */
int nufi_solve_poisson(nufi_handle *h, const double *rho, double *phi_out, double *spec_re, double *spec_im,
                       double *W_out);
int nufi_fit_spline(nufi_handle *h, const double *phi, double *coeffs_out);
/* transform_values / forward_transform (poisson.py:72-83): spectrum = fftn(values) / N^d
 * (numpy FFT layout, real and imaginary parts, Nx^d each).  inverse_transform
 * (poisson.py:85-87): values = Re ifftn(spectrum * N^d). */
int nufi_transform_values(nufi_handle *h, const double *values, double *spec_re, double *spec_im);
int nufi_inverse_transform(nufi_handle *h, const double *spec_re, const double *spec_im, double *values_out);

/* Stream-ordered forms of the per-step drop-in pair (compute_rho + the tail), for a host
 * loop that must not wait on every call.  nufi_async_slots allocates a ring of `slots`
 * pinned host entries; an entry holds [rho (Nx^d) | stats3 | W | status (int32 in a
 * double slot) | pad | E (Nx^d*d) | coeffs (Nx^d)]; the kernels write it directly (mapped
 * pinned memory), so no copy is enqueued on the common path.  nufi_rho_async enqueues compute_rho of step n (same checks as
 * nufi_rho) and its rho / stats copies into entry `slot`; nufi_field_update_async enqueues
 * the tail (rho: host / device Nx^d values, or NULL = the density the last nufi_rho_async
 * left on the device -- no copy) and its W / E / coeffs copies into entry `slot`, and
 * advances the history length provisionally.  Neither waits.  nufi_async_wait blocks until
 * the entry's copies are complete and returns a pointer to it (valid until the slot is
 * reused); a non-neutral density in any enqueued tail makes it return NUFI_ERR_NUMERICAL
 * (history length reset to the fields actually appended, later tails skipped). */
int nufi_async_slots(nufi_handle *h, int slots);
int nufi_rho_async(nufi_handle *h, int64_t n, int slot, int64_t *evals, int *speculative);
/* When n == history length (the loop's next step), nufi_rho_async runs the WHOLE step in
 * one launch -- the tail writes slot n without committing it -- and sets *speculative = 1;
 * nufi_commit_async(h, n) then appends it (history length n + 1) with no further work.
 * Any other call that writes the history or changes f0 discards the speculation. */
int nufi_commit_async(nufi_handle *h, int64_t n);
int nufi_field_update_async(nufi_handle *h, const double *rho, int slot);
int nufi_async_wait(nufi_handle *h, int slot, double **entry);
/* The ring as one contiguous pinned block: *base = entry 0, entry q at *base + q * *slot_elems
 * (a host binding can map it once instead of per entry; an entry is complete once its event
 * -- or the handle's stream (nufi_sync) -- has been waited for). */
int nufi_async_ring(nufi_handle *h, double **base, int64_t *slot_elems);

/* One full step n (requires len == n): nufi_rho + nufi_field_update, all on
 * the device.  Outputs optional. */
int nufi_step(nufi_handle *h, int64_t n, double *rho_out, double *E_out, double *W_out,
              double *stats3, int64_t *evals);

/* The run driver: steps len .. n_last inclusive.
 * Per-step outputs are written at row (step - first_step) of
 * rho_hist (Nx^d), E_hist (Nx^d*d), W_hist (1), stats_hist (3); any may be NULL.
 * Host outputs are copied once at the end. */
int nufi_run(nufi_handle *h, int64_t n_last, double *rho_hist, double *E_hist, double *W_hist,
             double *stats_hist, int64_t *evals);

/* trace_backward (kernels.py:390-412) on caller points, in place.
 * X, V: (M, d) row-major float64 (host or device).  half_kick: Psi (needs
 * len >= n + 1) vs Psi-tilde (len >= n).  mode: NUFI_TRACE_FAST / _PARITY.
 * evals (optional) += M * (n + half_kick) for n > 0. */
int nufi_trace(nufi_handle *h, int64_t n, double *X, double *V, int64_t M, int half_kick, int mode,
               int64_t *evals);

/* FlowContext.install_field(step, UniformField(E0)) (flow.py:44-47, spline.py:55-68):
 * a spatially constant field E0 (d values) overrides stored field `step` for the
 * point-level trace; E0 == NULL removes the override, nufi_clear_fields removes all.
 * While any override is installed, nufi_trace follows the reference's generic path
 * (flow.py:65-82: numpy operation order, UniformField or the stored spline's
 * eval_E_many per slot; a slot needs a stored or installed field), and the density /
 * run entry points (nufi_rho*, nufi_step*, nufi_run, nufi_moments) return
 * NUFI_ERR_USAGE. */
int nufi_set_uniform_field(nufi_handle *h, int64_t step, const double *E0);
/* FlowContext.install_field(step, SplineField) (flow.py:44-47): the spline with coefficient
 * slab `coeffs` (Nx^d, row-major; host or device, copied) overrides stored field `step` for
 * the point-level trace, evaluated like SplineField.eval_E_many (kernels.py:102-123);
 * NULL removes it.  Same rules as nufi_set_uniform_field. */
int nufi_set_spline_field(nufi_handle *h, int64_t step, const double *coeffs);
int nufi_clear_fields(nufi_handle *h);

/* Observable sweep at step n (density.quadrature_sweep_many, density.py:94-120,
 * for the conserved-quantity weights of SPEC.md:403-406): every quadrature
 * point of this handle's velocity blocks is traced with Psi (needs len >= n+1
 * for n > 0, else NUFI_ERR_USAGE like flow.py:106-112), f = f0(foot), and
 *   out[0] = hx^d hv^d sum f          out[1] = hx^d hv^d sum f^2
 *   out[2] = hx^d hv^d sum f ln f     out[3] = hx^d hv^d sum |v|^2 f / 2
 *   out[4 + a] = hx^d hv^d sum v_a f  (a < d)
 *   out[4 + d] = min f,  out[5 + d] = max f
 * with weights taken at the untraced quadrature point (density.py:57-60).
 * out: 6 + d doubles.  evals (optional) += points * (n + 1) for n > 0. */
int nufi_moments(nufi_handle *h, int64_t n, double *out, int64_t *evals);

/* SplineField.eval_phi_many / eval_E_many (spline.py:46-52, kernels.py:84-123) of
 * stored field `slot` at caller points X (M, d): phi_out (M) and E_out (M, d) = minus
 * the spline gradient, each optional; host or device buffers.  The numpy twin's
 * operation order, no FMA: bit-identical to the reference. */
int nufi_eval_field(nufi_handle *h, int64_t slot, const double *X, int64_t M, double *phi_out, double *E_out);

/* kernels.bspline_weights / bspline_dweights (kernels.py:62-81): the cubic B-spline stencil
 * weights of M cell fractions t, w_out / dw_out (4, M) row-major (either may be NULL); numpy's
 * operation order, no FMA (bit-identical). */
int nufi_bspline_weights(nufi_handle *h, const double *t, int64_t M, double *w_out, double *dw_out);

/* f0 at caller points (eval_f0, initial.py:165-180): F[M]. */
int nufi_eval_f0(nufi_handle *h, const double *X, const double *V, int64_t M, double *F);

/* ---- measurement ---------------------------------------------------------- */

/* Per-launch CUDA-event timing of the library's kernels on the handle stream.
 * enable != 0 starts (and zeroes) accumulation; nufi_profiling_read fills
 * out[8] = {trace_ms, trace_launches, reduce_ms, reduce_launches,
 *           field_ms, field_launches, trace_point_steps, 0}. */
int nufi_profiling(nufi_handle *h, int enable);
int nufi_profiling_read(nufi_handle *h, double *out8);
/* FP64 vector (DFMA) peak of `device`, measured by a DFMA-chain kernel. */
int nufi_fp64_peak(int device, double *tflops, double *ms);

#ifdef __cplusplus
}
#endif

#endif /* NUFI_H */
