// FireCaffe CPU oracle — TEST INFRASTRUCTURE ONLY.
//
// Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
// `--impl reference`) may load this library. The product path
// (paper_1511_00175_b200/) never links, imports or calls it, and this file
// shares no code, header, constant or helper with the CUDA path.
//
// Plain, slow, obviously-correct host C++ of what the data-parallel hot path
// computes (PAPER.md = /root/reference/PAPER.md, cited as P:line):
//
//   * oracle_tree_sum  — element-wise sum of the p per-worker gradient vectors
//     through a k-nomial reduction tree rooted at rank 0 (§6.2
//     "binomial reduction tree", Fig. P:312-315).  The floating-point
//     association is the tree's own (reading R1): at step s = k^l,
//     node r (r mod k·s == 0) absorbs r + j·s for j = 1..k-1 in ascending order.
//   * oracle_ps_sum    — the parameter server of §6.1:
//     one node sums every worker's gradient, ascending rank, sequentially
//     (the tree of height 1 and branching factor p).  Reading R4.
//   * oracle_sgd       — one SGD step with momentum and weight decay
//     (rule not written in the paper -> Caffe convention,
//     reading R6): g = S·fl(1/B) (inputs are per-worker SUMS of ∇W, P:235-236,
//     reading R7), d = fma(wd, w, g), v' = fma(mu, v, fl(lr·d)), w' = w − v'.
//   * oracle_sum_f64 / oracle_sgd_f64 — float64 left-to-right references used
//     for the "1e-6 relative vs float64" tolerance in north_star.
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -shared -fPIC.
// -ffp-contract=off matters: a contracted a*b+c would change the rounding
// sequence the oracle defines.  std::fma is a true fused multiply-add
// (one rounding), emulation through double is NOT (SURVEY.md §0 finding 6).
// x86-64 evaluates float arithmetic in float (SSE, FLT_EVAL_METHOD == 0), so
// every `+`, `*`, `-` below is one IEEE round-to-nearest-even fp32 operation.
// No FTZ/DAZ (MXCSR default).  liboracle.so (the correctness oracle) is
// single-threaded.  The element loops of oracle_tree_sum and oracle_sgd carry
// `#pragma omp` directives that the plain build ignores; the -fopenmp build of
// this same file (liboracle_omp.so, bench.py's all-cores CPU baseline,
// SURVEY §8(d)) splits ELEMENTS over the host cores.  Every element's
// arithmetic and association is unchanged, so both builds give identical bits
// (tests/test_oracle.py checks it).

#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

extern "C" {

// Version tag so tests can check they loaded the intended build.
int oracle_version(void) { return 1; }

#ifdef _OPENMP
#include <omp.h>
int oracle_threads(void) { return omp_get_max_threads(); }
void oracle_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }
#else
int oracle_threads(void) { return 1; }
void oracle_set_threads(int) {}
#endif

// ---------------------------------------------------------------------------
// Reduction tree sum (Eq. 4; Fig. P:312-315).
//
// g   : p*n floats, row-major (g[r*n + i] = worker r's gradient element i)
// out : n floats, the tree's root value (what every rank ends with after the
//       broadcast "back down the tree").
// k   : branching factor, 2 <= k; k >= p gives the one-level tree = PS order.
//
// Per element i (elements are independent, "element-wise addition"):
//   part[r] = g[r][i]
//   step = 1
//   while step < p:
//     for r = 0, k*step, 2*k*step, ... < p:
//       for j = 1 .. k-1:                  (children in ascending rank)
//         c = r + j*step
//         if c < p: part[r] = fl32(part[r] + part[c])
//     step *= k
//   out[i] = part[0]
// ---------------------------------------------------------------------------
int oracle_tree_sum(const float* g, int p, int64_t n, int k, float* out) {
    if (p < 1 || n < 0 || k < 2 || (n > 0 && (!g || !out))) return 1;
#pragma omp parallel
    {
    std::vector<float> part((size_t)p);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        for (int r = 0; r < p; ++r) part[(size_t)r] = g[(int64_t)r * n + i];
        int64_t step = 1;
        while (step < p) {
            for (int64_t r = 0; r < p; r += (int64_t)k * step) {
                for (int j = 1; j <= k - 1; ++j) {
                    int64_t c = r + (int64_t)j * step;
                    if (c < p) {
                        part[(size_t)r] = part[(size_t)r] + part[(size_t)c];
                    }
                }
            }
            step *= k;
        }
        out[i] = part[0];
    }
    }
    return 0;
}

// ---------------------------------------------------------------------------
// Parameter-server sum: the server adds the workers'
// gradients one after another, ascending rank: ((g0+g1)+g2)+...+g_{p-1}.
// Written out on its own (not by calling the tree with k=p) so that the
// "k=p tree == PS" identity is a test, not a tautology.
// ---------------------------------------------------------------------------
int oracle_ps_sum(const float* g, int p, int64_t n, float* out) {
    if (p < 1 || n < 0 || (n > 0 && (!g || !out))) return 1;
    for (int64_t i = 0; i < n; ++i) {
        float acc = g[i];
        for (int r = 1; r < p; ++r) {
            acc = acc + g[(int64_t)r * n + i];
        }
        out[i] = acc;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// SGD with momentum and weight decay, in place (μ, wd P:358, P:363;
// lr P:413; Caffe convention per SPEC S:86 and reading R6).
//   inv_b = fl32(1 / (float)B)          (global batch B, reading R7)
//   g  = fl32(S · inv_b)
//   d  = fma(wd, w, g)                  (g + wd·w, one rounding)
//   t  = fl32(lr · d)
//   v' = fma(mu, v, t)                  (mu·v + lr·d, one rounding)
//   w' = fl32(w − v')
// ---------------------------------------------------------------------------
int oracle_sgd(float* w, float* v, const float* S, int64_t n, float lr, float mu,
               float wd, int64_t batch) {
    if (n < 0 || batch < 1 || (n > 0 && (!w || !v || !S))) return 1;
    const float inv_b = 1.0f / (float)batch;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const float g = S[i] * inv_b;
        const float d = std::fma(wd, w[i], g);
        const float t = lr * d;
        const float vn = std::fma(mu, v[i], t);
        const float wn = w[i] - vn;
        v[i] = vn;
        w[i] = wn;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// SGD with Caffe per-blob multipliers ("consistent with
// the Caffe configuration files", P:357-358 per-layer settings).  The flat
// parameter vector is a concatenation of blobs; blob s covers
// [begin[s], begin[s+1]) (the last one up to n) and carries lr_mult[s],
// decay_mult[s] (Caffe ParamSpec).  Per element (reading R20):
//   local_lr = fl(lr · lr_mult),  local_wd = fl(wd · decay_mult)
//   then the oracle_sgd rule with (local_lr, local_wd).
// With every multiplier 1 this is bit-identical to oracle_sgd.
// ---------------------------------------------------------------------------
int oracle_sgd_segments(float* w, float* v, const float* S, int64_t n, float lr, float mu,
                        float wd, int64_t batch, const int64_t* begin, const float* lr_mult,
                        const float* decay_mult, int nseg) {
    if (n < 0 || batch < 1 || nseg < 1 || !begin || !lr_mult || !decay_mult) return 1;
    if (n > 0 && (!w || !v || !S)) return 1;
    if (begin[0] != 0) return 1;
    for (int s = 1; s < nseg; ++s)
        if (begin[s] <= begin[s - 1] || begin[s] >= n) return 1;
    const float inv_b = 1.0f / (float)batch;
    int s = 0;
    for (int64_t i = 0; i < n; ++i) {
        while (s + 1 < nseg && begin[s + 1] <= i) ++s;  // blob containing element i
        const float local_lr = lr * lr_mult[s];
        const float local_wd = wd * decay_mult[s];
        const float g = S[i] * inv_b;
        const float d = std::fma(local_wd, w[i], g);
        const float t = local_lr * d;
        const float vn = std::fma(mu, v[i], t);
        const float wn = w[i] - vn;
        v[i] = vn;
        w[i] = wn;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// Learning-rate schedules of the paper:
//   policy 0 fixed      : base_lr
//   policy 1 step       : base_lr · gamma^floor(iter / stepsize)
//   policy 2 multistep  : base_lr · gamma^#{k : steps[k] <= iter}   ("reduce this by
//                          a factor of 10x twice")
//   policy 3 poly       : base_lr · (1 − it/max_iter)^power,  it = min(iter, max_iter)
//                          (power 0.5; past max_iter training has ended and
//                          the schedule stays at its end value — reading R21)
// Evaluated in double (std::pow), rounded once to fp32 (reading R21).  Domain:
// base_lr > 0, gamma > 0, power >= 0 (all finite), stepsize >= 1, max_iter >= 1,
// iter >= 0; returns -1 otherwise.
// ---------------------------------------------------------------------------
float oracle_lr_at(int policy, float base_lr, int64_t iter, float gamma, int64_t stepsize,
                   const int64_t* steps, int nsteps, float power, int64_t max_iter) {
    if (iter < 0 || !(base_lr > 0.0f) || !std::isfinite(base_lr)) return -1.0f;
    double f = 1.0;
    if (policy == 0) {
        f = 1.0;
    } else if (policy == 1) {
        if (stepsize < 1 || !(gamma > 0.0f) || !std::isfinite(gamma)) return -1.0f;
        f = std::pow((double)gamma, (double)(iter / stepsize));
    } else if (policy == 2) {
        if (nsteps < 0 || (nsteps > 0 && !steps) || !(gamma > 0.0f) || !std::isfinite(gamma))
            return -1.0f;
        int k = 0;
        for (int j = 0; j < nsteps; ++j)
            if (steps[j] <= iter) ++k;
        f = std::pow((double)gamma, (double)k);
    } else if (policy == 3) {
        if (max_iter < 1 || !(power >= 0.0f) || !std::isfinite(power)) return -1.0f;
        const int64_t it = iter < max_iter ? iter : max_iter;
        f = std::pow(1.0 - (double)it / (double)max_iter, (double)power);
    } else {
        return -1.0f;
    }
    return (float)((double)base_lr * f);
}

// ---------------------------------------------------------------------------
// float64 references (north_star: "within 1e-6 relative error (fp32) against
// a naive left-to-right float64 sum").
// ---------------------------------------------------------------------------
int oracle_sum_f64(const float* g, int p, int64_t n, double* out) {
    if (p < 1 || n < 0 || (n > 0 && (!g || !out))) return 1;
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int r = 0; r < p; ++r) acc += (double)g[(int64_t)r * n + i];
        out[i] = acc;
    }
    return 0;
}

// Σ_r |g_r[i]| in float64: the scale the summation error bound is stated in.
int oracle_abs_sum_f64(const float* g, int p, int64_t n, double* out) {
    if (p < 1 || n < 0 || (n > 0 && (!g || !out))) return 1;
    for (int64_t i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int r = 0; r < p; ++r) acc += std::fabs((double)g[(int64_t)r * n + i]);
        out[i] = acc;
    }
    return 0;
}

// Same SGD rule in float64 (fp32 hyper-parameters promoted); S64 is the
// float64 gradient sum.  w64, v64 are in/out.
int oracle_sgd_f64(double* w64, double* v64, const double* S64, int64_t n, float lr,
                   float mu, float wd, int64_t batch) {
    if (n < 0 || batch < 1 || (n > 0 && (!w64 || !v64 || !S64))) return 1;
    for (int64_t i = 0; i < n; ++i) {
        double g = S64[i] / (double)batch;
        double d = g + (double)wd * w64[i];
        double vn = (double)mu * v64[i] + (double)lr * d;
        v64[i] = vn;
        w64[i] = w64[i] - vn;
    }
    return 0;
}

// ---------------------------------------------------------------------------
// The reduce phase of the tree as a communication plan (SPEC S:367-375
// `plan_topology`): every (level, sender -> receiver) edge in the
// order the oracle's loop visits them.  Returns the number of edges written
// (at most cap); edges[3*e+0..2] = level, sender (child), receiver (parent).
// ---------------------------------------------------------------------------
int oracle_tree_plan(int p, int k, int* edges, int cap) {
    if (p < 1 || k < 2) return -1;
    int e = 0;
    int level = 0;
    int64_t step = 1;
    while (step < p) {
        for (int64_t r = 0; r < p; r += (int64_t)k * step) {
            for (int j = 1; j <= k - 1; ++j) {
                int64_t c = r + (int64_t)j * step;
                if (c < p) {
                    if (e < cap && edges) {
                        edges[3 * e + 0] = level;
                        edges[3 * e + 1] = (int)c;
                        edges[3 * e + 2] = (int)r;
                    }
                    ++e;
                }
            }
        }
        step *= k;
        ++level;
    }
    return e;
}

}  // extern "C"
