/*
 * conv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU oracle for the operator that
 * arXiv 2008.03602 tunes: the "2D convolution" DNN operator
 * (section "DNN Autotuning Systems"), inference only,
 * followed by the optional bias + "RELU operator" epilogue.
 * The paper states that tuning does not change the operator's output
 * ("the output of the inference remains the same"), so the oracle
 * is the plain definition of conv2d written out:
 *
 *   acc[n,k,p,q] = sum_{c'<Cg} sum_{r<R} sum_{s<S}
 *                    x[n, c0+c', p*sh - ph + r*dh, q*sw - pw + s*dw] * w[k, c', r, s]
 *                  (out-of-range spatial index contributes 0;  c0 = (k / Kg) * Cg)
 *   y[n,k,p,q]   = relu?( acc + (bias ? b[k] : 0) )
 *   P = floor((H + 2 ph - dh (R-1) - 1) / sh) + 1,  Q likewise.
 *
 * Readings of the silent paper: C1 cross-correlation
 * (no filter flip), C2 symmetric zero padding, C3 floor output formula,
 * C4 dilation >= 1 supported here, C5 groups in {1..C} with C % g == 0,
 * K % g == 0, C9 bias then ReLU.
 *
 * Layout: logical NCHW for x, KCRS (K, C/g, R, S) for w, NKPQ for y,
 * all dense row-major, fp64.  The oracle shares NO code with the CUDA path
 * (paper_2008_03602_b200/csrc); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC (no -ffast-math).
 */
#include <stdint.h>
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t n, c, h, w, k, r, s;
    int32_t stride_h, stride_w, pad_h, pad_w, dil_h, dil_w, groups;
    int32_t has_bias, relu;
} oracle_desc;

/* Output extent along one spatial axis, SURVEY 8(c) C3. Returns <1 when the
 * window does not fit (caller treats that as an invalid shape). */
int oracle_out_dim(int32_t in, int32_t k, int32_t stride, int32_t pad, int32_t dil)
{
    int32_t span = in + 2 * pad - dil * (k - 1) - 1;
    if (span < 0 || stride < 1) return 0;
    return span / stride + 1;
}

static int check_desc(const oracle_desc* d)
{
    if (d->n < 1 || d->c < 1 || d->h < 1 || d->w < 1 || d->k < 1 || d->r < 1 || d->s < 1) return 1;
    if (d->stride_h < 1 || d->stride_w < 1 || d->dil_h < 1 || d->dil_w < 1) return 1;
    if (d->pad_h < 0 || d->pad_w < 0 || d->groups < 1) return 1;
    if (d->c % d->groups != 0 || d->k % d->groups != 0) return 1;
    if (oracle_out_dim(d->h, d->r, d->stride_h, d->pad_h, d->dil_h) < 1) return 1;
    if (oracle_out_dim(d->w, d->s, d->stride_w, d->pad_w, d->dil_w) < 1) return 1;
    return 0;
}

/* One output element, straight from the definition above. */
static double conv_point(const oracle_desc* d, const double* x, const double* w,
                         const double* b, int32_t P, int32_t Q,
                         int32_t n, int32_t k, int32_t p, int32_t q)
{
    (void)P; (void)Q;
    const int32_t Cg = d->c / d->groups;
    const int32_t Kg = d->k / d->groups;
    const int32_t c0 = (k / Kg) * Cg;
    double acc = 0.0;
    for (int32_t cc = 0; cc < Cg; ++cc) {
        for (int32_t r = 0; r < d->r; ++r) {
            const int32_t hi = p * d->stride_h - d->pad_h + r * d->dil_h;
            if (hi < 0 || hi >= d->h) continue;
            for (int32_t s = 0; s < d->s; ++s) {
                const int32_t wi = q * d->stride_w - d->pad_w + s * d->dil_w;
                if (wi < 0 || wi >= d->w) continue;
                const double xv = x[(((int64_t)n * d->c + (c0 + cc)) * d->h + hi) * d->w + wi];
                const double wv = w[(((int64_t)k * Cg + cc) * d->r + r) * d->s + s];
                acc += xv * wv;
            }
        }
    }
    if (d->has_bias) acc += b[k];
    if (d->relu && acc < 0.0) acc = 0.0;
    return acc;
}

/* Full output tensor y[N][K][P][Q].  OpenMP over (n, k); nthreads <= 0 means
 * "runtime default".  Returns 0 on success, 1 on an invalid descriptor. */
int oracle_conv2d_f64(const oracle_desc* d, const double* x, const double* w,
                      const double* b, double* y, int32_t nthreads)
{
    if (check_desc(d)) return 1;
    const int32_t P = oracle_out_dim(d->h, d->r, d->stride_h, d->pad_h, d->dil_h);
    const int32_t Q = oracle_out_dim(d->w, d->s, d->stride_w, d->pad_w, d->dil_w);
    const int64_t NK = (int64_t)d->n * d->k;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#else
    (void)nthreads;
#endif
    for (int64_t nk = 0; nk < NK; ++nk) {
        const int32_t n = (int32_t)(nk / d->k), k = (int32_t)(nk % d->k);
        double* yo = y + nk * (int64_t)P * Q;
        for (int32_t p = 0; p < P; ++p)
            for (int32_t q = 0; q < Q; ++q)
                yo[(int64_t)p * Q + q] = conv_point(d, x, w, b, P, Q, n, k, p, q);
    }
    return 0;
}

/* Selected outputs only: idx[i] is a flat NKPQ index.  Used for sampled
 * parity at full size (the 4096-point correctness gate of SURVEY 8(a) a10). */
int oracle_conv2d_points_f64(const oracle_desc* d, const double* x, const double* w,
                             const double* b, const int64_t* idx, int64_t npts,
                             double* out, int32_t nthreads)
{
    if (check_desc(d)) return 1;
    const int32_t P = oracle_out_dim(d->h, d->r, d->stride_h, d->pad_h, d->dil_h);
    const int32_t Q = oracle_out_dim(d->w, d->s, d->stride_w, d->pad_w, d->dil_w);
    const int64_t total = (int64_t)d->n * d->k * P * Q;
    for (int64_t i = 0; i < npts; ++i)
        if (idx[i] < 0 || idx[i] >= total) return 2;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#else
    (void)nthreads;
#endif
    for (int64_t i = 0; i < npts; ++i) {
        int64_t t = idx[i];
        const int32_t q = (int32_t)(t % Q); t /= Q;
        const int32_t p = (int32_t)(t % P); t /= P;
        const int32_t k = (int32_t)(t % d->k); t /= d->k;
        const int32_t n = (int32_t)t;
        out[i] = conv_point(d, x, w, b, P, Q, n, k, p, q);
    }
    return 0;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
