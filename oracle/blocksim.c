/*
 * oracle/blocksim.c — O-2, the plain CPU block simulator.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
 * `--impl reference`) may load or call this library.  It shares no source, header,
 * table or helper with the CUDA path in paper_2410_17876_b200/, and neither side
 * includes or links the other.
 *
 * Every function follows PAPER.md §2 step by step, in the paper's notation:
 *   qudits q_0..q_{n-1}, q_0 least significant, D = prod d_i
 *   block size b_i = prod_{t<i} d_t, repetitions r_i = prod_{t>i} d_t
 *   an equivalence class = the d_i basis states that differ only in q_i (PAPER.md:198,
 *     Table tab:eq_classes); its members are rep*d_i*b_i + j*b_i + off
 *   the basis state with q_i = j transforms by column j of U; the new class amplitudes
 *     are sum_j x_j * U[:, j], stored back in place
 *   control condition floor(i/b_k) mod d_k = v_k, checked by brute force
 *   phase gates scale block j by U(j,j)
 *   X_{+a} rotates the d_i blocks of every group by a
 *
 * Amplitudes are interleaved (re, im) doubles; U is d*d complex, row-major, interleaved.
 * No fusion, no blocking, no fast-math.  OpenMP only splits the independent classes
 * across threads ("parallelism across blocks").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Block sizes b_k and total dimension D.  Returns -1 on overflow. */
int orc_strides(int n, const int *dims, uint64_t *b, uint64_t *D)
{
    uint64_t p = 1;
    for (int k = 0; k < n; ++k) {
        if (dims[k] < 2) return -1;
        b[k] = p;
        if (p > UINT64_MAX / (uint64_t)dims[k]) return -1;
        p *= (uint64_t)dims[k];
    }
    *D = p;
    return 0;
}

/* floor(i / b_k) mod d_k == v_k for every control. */
static int controls_hold(uint64_t i, int nctrl, const int *ctrl, const int *vals,
                         const uint64_t *b, const int *dims)
{
    for (int m = 0; m < nctrl; ++m) {
        int c = ctrl[m];
        if ((int)((i / b[c]) % (uint64_t)dims[c]) != vals[m]) return 0;
    }
    return 1;
}

/* Superposition (general) gate, §2.3, with the brute-force control filter of §2.4. */
int orc_apply(double *psi, int n, const int *dims, int target, int nctrl,
              const int *ctrl, const int *vals, const double *U)
{
    uint64_t b[64], D;
    if (n < 1 || n > 64 || orc_strides(n, dims, b, &D)) return -1;
    const int d = dims[target];
    const uint64_t bs = b[target];            /* block size  prod_{t<i} d_t  */
    const uint64_t reps = D / (bs * (uint64_t)d);   /* repetitions prod_{t>i} d_t */

    #pragma omp parallel for collapse(2) schedule(static)
    for (uint64_t rep = 0; rep < reps; ++rep) {
        for (uint64_t off = 0; off < bs; ++off) {
            const uint64_t base = rep * (uint64_t)d * bs + off;   /* class member j=0 */
            if (!controls_hold(base, nctrl, ctrl, vals, b, dims)) continue;
            double xr[16], xi[16];
            for (int j = 0; j < d; ++j) {                      /* gather the class */
                xr[j] = psi[2 * (base + (uint64_t)j * bs)];
                xi[j] = psi[2 * (base + (uint64_t)j * bs) + 1];
            }
            double yr[16], yi[16];
            for (int k = 0; k < d; ++k) { yr[k] = 0.0; yi[k] = 0.0; }
            for (int j = 0; j < d; ++j) {                      /* sum_j x_j * U[:, j] */
                for (int k = 0; k < d; ++k) {
                    const double ur = U[2 * (k * d + j)], ui = U[2 * (k * d + j) + 1];
                    yr[k] += ur * xr[j] - ui * xi[j];
                    yi[k] += ur * xi[j] + ui * xr[j];
                }
            }
            for (int k = 0; k < d; ++k) {                      /* store back in place */
                psi[2 * (base + (uint64_t)k * bs)] = yr[k];
                psi[2 * (base + (uint64_t)k * bs) + 1] = yi[k];
            }
        }
    }
    return 0;
}

/* Phase gate, §2.1: block j of every group is multiplied by the scalar U(j,j).
 * diag holds the d diagonal entries (interleaved).  Controls as in §2.4. */
int orc_apply_phase(double *psi, int n, const int *dims, int target, int nctrl,
                    const int *ctrl, const int *vals, const double *diag)
{
    uint64_t b[64], D;
    if (n < 1 || n > 64 || orc_strides(n, dims, b, &D)) return -1;
    const int d = dims[target];
    const uint64_t bs = b[target];
    const uint64_t reps = D / (bs * (uint64_t)d);

    #pragma omp parallel for schedule(static)
    for (uint64_t rep = 0; rep < reps; ++rep) {
        for (int j = 0; j < d; ++j) {
            const double ur = diag[2 * j], ui = diag[2 * j + 1];
            for (uint64_t off = 0; off < bs; ++off) {
                const uint64_t i = rep * (uint64_t)d * bs + (uint64_t)j * bs + off;
                if (!controls_hold(i, nctrl, ctrl, vals, b, dims)) continue;
                const double xr = psi[2 * i], xi = psi[2 * i + 1];
                psi[2 * i] = ur * xr - ui * xi;
                psi[2 * i + 1] = ur * xi + ui * xr;
            }
        }
    }
    return 0;
}

/* Permutation gate X_{+a}, §2.2: block k of every group moves to block (k+a) mod d — a
 * cyclic rotation of the d blocks by a steps.  Controls as in §2.4 (checked per class). */
int orc_apply_shift(double *psi, int n, const int *dims, int target, int nctrl,
                    const int *ctrl, const int *vals, int a)
{
    uint64_t b[64], D;
    if (n < 1 || n > 64 || orc_strides(n, dims, b, &D)) return -1;
    const int d = dims[target];
    const uint64_t bs = b[target];
    const uint64_t reps = D / (bs * (uint64_t)d);
    a = ((a % d) + d) % d;

    #pragma omp parallel for collapse(2) schedule(static)
    for (uint64_t rep = 0; rep < reps; ++rep) {
        for (uint64_t off = 0; off < bs; ++off) {
            const uint64_t base = rep * (uint64_t)d * bs + off;
            if (!controls_hold(base, nctrl, ctrl, vals, b, dims)) continue;
            double tr[16], ti[16];
            for (int k = 0; k < d; ++k) {
                tr[k] = psi[2 * (base + (uint64_t)k * bs)];
                ti[k] = psi[2 * (base + (uint64_t)k * bs) + 1];
            }
            for (int k = 0; k < d; ++k) {
                const uint64_t dst = base + (uint64_t)((k + a) % d) * bs;
                psi[2 * dst] = tr[k];
                psi[2 * dst + 1] = ti[k];
            }
        }
    }
    return 0;
}

/* Apply a whole circuit gate by gate (one gate at a time).
 * ctrl_flat / vals_flat hold the controls of all gates back to back; U_flat holds the
 * d_t*d_t complex matrices back to back. */
int orc_run(double *psi, int n, const int *dims, int64_t ngates, const int *targets,
            const int *nctrls, const int *ctrl_flat, const int *vals_flat, const double *U_flat)
{
    int64_t co = 0, uo = 0;
    for (int64_t g = 0; g < ngates; ++g) {
        const int t = targets[g];
        if (t < 0 || t >= n) return -1;
        if (orc_apply(psi, n, dims, t, nctrls[g], ctrl_flat + co, vals_flat + co, U_flat + uo))
            return -1;
        co += nctrls[g];
        uo += 2 * (int64_t)dims[t] * dims[t];
    }
    return 0;
}

/* sqrt(sum_i |alpha_i|^2), plain left-to-right sum per thread, partials added in order. */
double orc_norm(const double *psi, uint64_t D)
{
    int nt = 1;
#ifdef _OPENMP
    nt = omp_get_max_threads();
#endif
    double *part = (double *)calloc((size_t)nt, sizeof(double));
    #pragma omp parallel
    {
        int id = 0;
#ifdef _OPENMP
        id = omp_get_thread_num();
#endif
        double s = 0.0;
        #pragma omp for schedule(static)
        for (uint64_t i = 0; i < D; ++i)
            s += psi[2 * i] * psi[2 * i] + psi[2 * i + 1] * psi[2 * i + 1];
        part[id] = s;
    }
    double s = 0.0;
    for (int t = 0; t < nt; ++t) s += part[t];
    free(part);
    return sqrt(s);
}

/* The index-labelled input state: Re = i+1, Im = -(i+1)/2. */
static void label(uint64_t i, double *re, double *im)
{
    *re = (double)i + 1.0;
    *im = -((double)i + 1.0) / 2.0;
}

/* One output amplitude of one gate applied to the labelled state, for sampled full-size
 * checks.  Index i is a member of the class with representative i - v*b (v = digit of q_i,
 * PAPER.md:235); if the controls hold, its new amplitude is row v of U times the class
 * vector, else it is unchanged. */
int orc_gate_output_labelled(int n, const int *dims, int target, int nctrl, const int *ctrl,
                             const int *vals, const double *U, const uint64_t *idx,
                             int64_t count, double *out)
{
    uint64_t b[64], D;
    if (n < 1 || n > 64 || orc_strides(n, dims, b, &D)) return -1;
    const int d = dims[target];
    const uint64_t bs = b[target];
    #pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < count; ++s) {
        const uint64_t i = idx[s];
        double yr, yi;
        if (!controls_hold(i, nctrl, ctrl, vals, b, dims)) {
            label(i, &yr, &yi);
        } else {
            const int v = (int)((i / bs) % (uint64_t)d);
            const uint64_t base = i - (uint64_t)v * bs;
            yr = 0.0; yi = 0.0;
            for (int j = 0; j < d; ++j) {
                double xr, xi;
                label(base + (uint64_t)j * bs, &xr, &xi);
                const double ur = U[2 * (v * d + j)], ui = U[2 * (v * d + j) + 1];
                yr += ur * xr - ui * xi;
                yi += ur * xi + ui * xr;
            }
        }
        out[2 * s] = yr;
        out[2 * s + 1] = yi;
    }
    return 0;
}

/* One output amplitude of a short circuit g_1..g_G applied to the labelled state, for sampled
 * full-size checks of multi-gate passes.  Gate by gate from the last one back (PAPER.md:256
 * applies them in order, so the amplitude after g_k at index i is fixed by the amplitudes
 * after g_{k-1}): if g_k's controls hold at i, it is row v of U_k times the
 * class vector of i after g_{k-1} (v = digit of i in q_t), else the amplitude
 * after g_{k-1} at i.  Cost prod_k d_k evaluations per index: short circuits. */
static void circuit_value(uint64_t i, int64_t k, const int *dims, const uint64_t *b,
                          const int *targets, const int *nctrls, const int64_t *coff,
                          const int *ctrl_flat, const int *vals_flat, const int64_t *uoff,
                          const double *U_flat, double *re, double *im)
{
    if (k == 0) { label(i, re, im); return; }
    const int64_t g = k - 1;
    const int t = targets[g];
    if (!controls_hold(i, nctrls[g], ctrl_flat + coff[g], vals_flat + coff[g], b, dims)) {
        circuit_value(i, k - 1, dims, b, targets, nctrls, coff, ctrl_flat, vals_flat, uoff, U_flat, re, im);
        return;
    }
    const int d = dims[t];
    const uint64_t bs = b[t];
    const int v = (int)((i / bs) % (uint64_t)d);
    const uint64_t base = i - (uint64_t)v * bs;
    const double *U = U_flat + uoff[g];
    double yr = 0.0, yi = 0.0;
    for (int j = 0; j < d; ++j) {
        double xr, xi;
        circuit_value(base + (uint64_t)j * bs, k - 1, dims, b, targets, nctrls, coff, ctrl_flat,
                      vals_flat, uoff, U_flat, &xr, &xi);
        const double ur = U[2 * (v * d + j)], ui = U[2 * (v * d + j) + 1];
        yr += ur * xr - ui * xi;
        yi += ur * xi + ui * xr;
    }
    *re = yr;
    *im = yi;
}

int orc_circuit_output_labelled(int n, const int *dims, int64_t ngates, const int *targets,
                                const int *nctrls, const int *ctrl_flat, const int *vals_flat,
                                const double *U_flat, const uint64_t *idx, int64_t count, double *out)
{
    uint64_t b[64], D;
    if (n < 1 || n > 64 || ngates < 0 || ngates > 8 || orc_strides(n, dims, b, &D)) return -1;
    int64_t coff[8], uoff[8], co = 0, uo = 0;
    for (int64_t g = 0; g < ngates; ++g) {
        if (targets[g] < 0 || targets[g] >= n) return -1;
        coff[g] = co;
        uoff[g] = uo;
        co += nctrls[g];
        uo += 2 * (int64_t)dims[targets[g]] * dims[targets[g]];
    }
    #pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < count; ++s)
        circuit_value(idx[s], ngates, dims, b, targets, nctrls, coff, ctrl_flat, vals_flat, uoff, U_flat,
                      &out[2 * s], &out[2 * s + 1]);
    return 0;
}

/* OpenMP thread count of later calls (the bench's 1-thread baseline run); n < 1 keeps it. */
void orc_set_threads(int n)
{
#ifdef _OPENMP
    if (n >= 1) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
