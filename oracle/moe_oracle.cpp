// oracle/moe_oracle.cpp -- fp64 CPU ORACLE for the Mixtral-8x7B sparse-MoE block.
//
// TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library. The product path
// (paper_2408_00008_b200/, libmoe.so) never calls, links or includes anything
// here, and this file includes nothing from the product tree: no shared headers,
// helpers, tables or constants. It decodes bf16 with its own bit shift.
//
// What it computes (the plain definition, written out; no blocking, fusion or
// reordering):
//   PAPER.md is silent on the MoE math. P:123 (Sec. 4.1, "We mainly focus on
//   optimizing the Mixture of Experts [jiang2024mixtral] LLMs") and P:172 (Sec. 5,
//   "We select Mistral 8x7B [jiang2024mixtral]") name Mixtral-8x7B, whose sparse
//   MoE layer is (reading R1):
//       l      = x W_g^T                                  (router logits, no bias)
//       S      = indices of the top-k logits              (R3: ties -> lower index)
//       p      = softmax(l) over all E experts
//       w_j    = p_{S_j} / sum_{j'} p_{S_j'}              (renormalised, R2)
//       h      = silu(x W1_e^T) * (x W3_e^T),  silu(z) = z / (1 + exp(-z))
//       o_e    = h W2_e^T
//       y      = sum_j w_j o_{S_j}
//   BASELINE.json north_star: "router GEMM, softmax, top-2 expert selection with
//   renormalised gate weights, token permutation by expert, grouped SwiGLU
//   expert GEMMs (w1/w3 then w2) and a weighted scatter-combine back to token
//   order".
//
// Everything is accumulated in double, sequentially, in index order.
// Weight layout is HuggingFace nn.Linear [out, in] row-major (R9):
//   x [T, d], W_g [E, d], W1 [E, f, d], W3 [E, f, d], W2 [E, d, f].
//
// Parity pins: see tests/test_oracle.py (every function below is pinned there;
// DESIGN.md "Oracle pins" lists which test pins which function).

#include <cstdint>
#include <cstring>
#include <cmath>
#include <omp.h>
#include <vector>
#include <algorithm>

namespace {

// ---- element decoders (own implementation; bf16 = top 16 bits of an IEEE fp32) ----
inline double dec(const uint16_t* p, size_t i) {
    uint32_t u = static_cast<uint32_t>(p[i]) << 16;
    float f;
    std::memcpy(&f, &u, sizeof(f));
    return static_cast<double>(f);
}
inline double dec(const float* p, size_t i) { return static_cast<double>(p[i]); }
inline double dec(const double* p, size_t i) { return p[i]; }

// ---- step 2: router logits l[t,e] = sum_c x[t,c] * W_g[e,c] (sequential fp64 sum) ----
template <typename Tin>
void router_logits(const Tin* x, const Tin* wg, int64_t t, int d, int E, double* l) {
    for (int e = 0; e < E; ++e) {
        double s = 0.0;
        for (int c = 0; c < d; ++c)
            s += dec(x, (size_t)t * d + c) * dec(wg, (size_t)e * d + c);
        l[e] = s;
    }
}

// ---- step 3: order experts by (logit desc, index asc); S = first k (reading R3) ----
void order_experts(const double* l, int E, std::vector<int>& order) {
    order.resize(E);
    for (int e = 0; e < E; ++e) order[e] = e;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        if (l[a] != l[b]) return l[a] > l[b];
        return a < b;
    });
}

// ---- step 4: softmax over all E, then renormalise over the selected k (R2) ----
void gates(const double* l, int E, const int* S, int k, double* w) {
    double lmax = l[0];
    for (int e = 1; e < E; ++e) lmax = std::max(lmax, l[e]);
    std::vector<double> p(E);
    double Z = 0.0;
    for (int e = 0; e < E; ++e) { p[e] = std::exp(l[e] - lmax); Z += p[e]; }
    for (int e = 0; e < E; ++e) p[e] /= Z;
    double s = 0.0;
    for (int j = 0; j < k; ++j) s += p[S[j]];
    for (int j = 0; j < k; ++j) w[j] = p[S[j]] / s;
}

inline double silu(double z) { return z / (1.0 + std::exp(-z)); }

// ---- step 5: one SwiGLU expert on one token: o = W2_e (silu(W1_e x) * (W3_e x)) ----
// If f_lo/f_hi restrict the ffn index range, only that slice of h contributes
// (used by the TP partition emulation; the full expert is f_lo=0, f_hi=f).
template <typename Tin>
void expert(const Tin* x, const Tin* w1, const Tin* w3, const Tin* w2, int64_t t, int e,
            int d, int f, int f_lo, int f_hi, double* o /*[d]*/) {
    std::vector<double> h(f, 0.0);
    for (int i = f_lo; i < f_hi; ++i) {
        double a = 0.0, b = 0.0;
        for (int c = 0; c < d; ++c) {
            double xc = dec(x, (size_t)t * d + c);
            a += dec(w1, ((size_t)e * f + i) * d + c) * xc;
            b += dec(w3, ((size_t)e * f + i) * d + c) * xc;
        }
        h[i] = silu(a) * b;
    }
    for (int r = 0; r < d; ++r) {
        double s = 0.0;
        for (int i = f_lo; i < f_hi; ++i) s += dec(w2, ((size_t)e * d + r) * f + i) * h[i];
        o[r] = s;
    }
}

template <typename Tin>
int router_impl(const Tin* x, const Tin* wg, int64_t T, int d, int E, int k,
                double* logits, int32_t* idx, double* w, double* m12, double* m23) {
    if (T < 0 || d <= 0 || E <= 0 || k <= 0 || k > E) return 1;
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < T; ++t) {
        std::vector<double> l(E);
        std::vector<int> order;
        router_logits(x, wg, t, d, E, l.data());
        order_experts(l.data(), E, order);
        std::vector<double> wt(k);
        gates(l.data(), E, order.data(), k, wt.data());
        for (int e = 0; e < E; ++e) if (logits) logits[t * E + e] = l[e];
        for (int j = 0; j < k; ++j) {
            if (idx) idx[t * k + j] = order[j];
            if (w) w[t * k + j] = wt[j];
        }
        // margins (reading R4): m12 = l(1)-l(2), m23 = l(2)-l(3) (inf when absent)
        if (m12) m12[t] = (E >= 2) ? l[order[0]] - l[order[1]] : INFINITY;
        if (m23) m23[t] = (E >= 3) ? l[order[1]] - l[order[2]] : INFINITY;
    }
    return 0;
}

// Full block forward for a list of tokens (all tokens when tok_list == nullptr).
// forced_idx [T,k] (nullable): steps 4-6 with an externally supplied S (step 8,
// "forced routing"); gates are still the renormalised softmax of the logits at S.
// y [n, d] row i is token tok_list[i] (or i).
template <typename Tin>
int forward_impl(const Tin* x, const Tin* wg, const Tin* w1, const Tin* w3, const Tin* w2,
                 int64_t T, int d, int f, int E, int k, const int32_t* forced_idx,
                 const int64_t* tok_list, int64_t n_list, int add_residual, double* y) {
    if (T < 0 || d <= 0 || f <= 0 || E <= 0 || k <= 0 || k > E) return 1;
    int64_t n = tok_list ? n_list : T;
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = tok_list ? tok_list[i] : i;
        if (t < 0 || t >= T) return 2;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = tok_list ? tok_list[i] : i;
        std::vector<double> l(E), wt(k), o(d), acc(d, 0.0);
        std::vector<int> order, S(k);
        router_logits(x, wg, t, d, E, l.data());
        order_experts(l.data(), E, order);
        for (int j = 0; j < k; ++j) S[j] = forced_idx ? forced_idx[t * k + j] : order[j];
        gates(l.data(), E, S.data(), k, wt.data());
        for (int j = 0; j < k; ++j) {
            expert(x, w1, w3, w2, t, S[j], d, f, 0, f, o.data());
            for (int r = 0; r < d; ++r) acc[r] += wt[j] * o[r];
        }
        // C5 stack composition x_{l+1} = x_l + MoE_l(x_l) (reading R12)
        if (add_residual)
            for (int r = 0; r < d; ++r) acc[r] += dec(x, (size_t)t * d + r);
        for (int r = 0; r < d; ++r) y[i * d + r] = acc[r];
    }
    return 0;
}

// EP / TP partition emulation (step 9). For G ranks:
//   EP: rank r owns experts [r*E/G, (r+1)*E/G); partial_r(t) = sum_{j: S_j owned by r} w_j o_{S_j}(t)
//   TP: rank r owns ffn slice [r*f/G, (r+1)*f/G) of every expert;
//       partial_r(t) = sum_j w_j W2_{S_j}[:, slice] h_{S_j}[slice]
// Output partials [G, n, d]. The sum over r must equal the full forward.
template <typename Tin>
int partition_impl(const Tin* x, const Tin* wg, const Tin* w1, const Tin* w3, const Tin* w2,
                   int64_t T, int d, int f, int E, int k, int G, int mode,
                   const int64_t* tok_list, int64_t n_list, double* partials) {
    if (G <= 0) return 1;
    if (mode == 1 && E % G) return 1;
    if (mode == 2 && f % G) return 1;
    int64_t n = tok_list ? n_list : T;
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = tok_list ? tok_list[i] : i;
        if (t < 0 || t >= T) return 2;
    }
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = tok_list ? tok_list[i] : i;
        std::vector<double> l(E), wt(k), o(d);
        std::vector<int> order;
        router_logits(x, wg, t, d, E, l.data());
        order_experts(l.data(), E, order);
        gates(l.data(), E, order.data(), k, wt.data());
        for (int r = 0; r < G; ++r) {
            double* P = partials + ((size_t)r * n + i) * d;
            for (int c = 0; c < d; ++c) P[c] = 0.0;
            for (int j = 0; j < k; ++j) {
                int e = order[j];
                if (mode == 1) {
                    if (e / (E / G) != r) continue;
                    expert(x, w1, w3, w2, t, e, d, f, 0, f, o.data());
                } else {
                    expert(x, w1, w3, w2, t, e, d, f, r * (f / G), (r + 1) * (f / G), o.data());
                }
                for (int c = 0; c < d; ++c) P[c] += wt[j] * o[c];
            }
        }
    }
    return 0;
}

}  // namespace

extern "C" {

// dtype codes: 0 = bf16 (uint16 bit patterns), 1 = fp32, 2 = fp64.
#define ORACLE_DISPATCH(dtype, CALL_BF16, CALL_F32, CALL_F64) \
    switch (dtype) {                                           \
        case 0: return CALL_BF16;                              \
        case 1: return CALL_F32;                               \
        case 2: return CALL_F64;                               \
        default: return 3;                                     \
    }

int oracle_router(int dtype, const void* x, const void* wg, int64_t T, int d, int E, int k,
                  double* logits, int32_t* idx, double* w, double* m12, double* m23) {
    ORACLE_DISPATCH(dtype,
        router_impl((const uint16_t*)x, (const uint16_t*)wg, T, d, E, k, logits, idx, w, m12, m23),
        router_impl((const float*)x, (const float*)wg, T, d, E, k, logits, idx, w, m12, m23),
        router_impl((const double*)x, (const double*)wg, T, d, E, k, logits, idx, w, m12, m23))
}

int oracle_moe_forward(int dtype, const void* x, const void* wg, const void* w1, const void* w3,
                       const void* w2, int64_t T, int d, int f, int E, int k,
                       const int32_t* forced_idx, const int64_t* tok_list, int64_t n_list,
                       int add_residual, double* y) {
    ORACLE_DISPATCH(dtype,
        forward_impl((const uint16_t*)x, (const uint16_t*)wg, (const uint16_t*)w1, (const uint16_t*)w3,
                     (const uint16_t*)w2, T, d, f, E, k, forced_idx, tok_list, n_list,
                     add_residual, y),
        forward_impl((const float*)x, (const float*)wg, (const float*)w1, (const float*)w3,
                     (const float*)w2, T, d, f, E, k, forced_idx, tok_list, n_list,
                     add_residual, y),
        forward_impl((const double*)x, (const double*)wg, (const double*)w1, (const double*)w3,
                     (const double*)w2, T, d, f, E, k, forced_idx, tok_list, n_list,
                     add_residual, y))
}

int oracle_partition(int dtype, const void* x, const void* wg, const void* w1, const void* w3,
                     const void* w2, int64_t T, int d, int f, int E, int k, int G, int mode,
                     const int64_t* tok_list, int64_t n_list, double* partials) {
    ORACLE_DISPATCH(dtype,
        partition_impl((const uint16_t*)x, (const uint16_t*)wg, (const uint16_t*)w1, (const uint16_t*)w3,
                       (const uint16_t*)w2, T, d, f, E, k, G, mode, tok_list, n_list, partials),
        partition_impl((const float*)x, (const float*)wg, (const float*)w1, (const float*)w3,
                       (const float*)w2, T, d, f, E, k, G, mode, tok_list, n_list, partials),
        partition_impl((const double*)x, (const double*)wg, (const double*)w1, (const double*)w3,
                       (const double*)w2, T, d, f, E, k, G, mode, tok_list, n_list, partials))
}

// Step 7, permutation reference (BASELINE.json north_star: "a histogram, an
// exclusive scan and a scatter into per-expert contiguous tiles"). Given a
// routing idx [T,k]:
//   counts[e]    = #{(t,j) : idx[t,j] == e}
//   offsets[0]   = 0, offsets[e+1] = offsets[e] + roundup(counts[e], align)
//   pos[t,j]     = offsets[e] + #{t' < t : token t' routed to e}   (stable by token index)
// Returns 1 on an out-of-range expert index or a token routed twice to one expert.
int oracle_permutation(const int32_t* idx, int64_t T, int k, int E, int align,
                       int32_t* counts, int64_t* offsets, int64_t* pos) {
    if (T < 0 || k <= 0 || E <= 0 || align <= 0) return 1;
    for (int e = 0; e < E; ++e) counts[e] = 0;
    for (int64_t t = 0; t < T; ++t)
        for (int j = 0; j < k; ++j) {
            int e = idx[t * k + j];
            if (e < 0 || e >= E) return 1;
            for (int j2 = 0; j2 < j; ++j2) if (idx[t * k + j2] == e) return 1;
            counts[e] += 1;
        }
    offsets[0] = 0;
    for (int e = 0; e < E; ++e)
        offsets[e + 1] = offsets[e] + ((int64_t)(counts[e] + align - 1) / align) * align;
    std::vector<int64_t> seen(E, 0);
    for (int64_t t = 0; t < T; ++t)
        for (int j = 0; j < k; ++j) {
            int e = idx[t * k + j];
            pos[t * k + j] = offsets[e] + seen[e];
            seen[e] += 1;
        }
    return 0;
}

// Host-thread count of the OpenMP loops (bench.py times the oracle both with all
// cores and single-threaded, BASELINE.md "CPU baseline plan"); returns the previous
// setting. Does not touch the arithmetic: every token is computed the same way.
int oracle_set_threads(int n) {
    const int prev = omp_get_max_threads();
    if (n > 0) omp_set_num_threads(n);
    return prev;
}

}  // extern "C"
