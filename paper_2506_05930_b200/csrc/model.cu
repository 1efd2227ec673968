// model.cu -- FP32 encoder / MLP (parity path), training gradients with the
// fixed-point hash-grid scatter, fused dense Adam, and the fp16 shadow refresh
// (SURVEY table K: K1 parity mode, K3, K4).
//
// Reference routines (under /root/reference/pkg/src/viscache):
//   encode_batch hashgrid.py:117-131, grad_from_ctx :140-151,
//   forward mlp.py:110-140, l2_loss :143-149, backward_l2 :152-183,
//   adam_step :203-218, VisibilityCache.train_step cache.py:60-73.
#include <algorithm>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace nvc {
// A per-device side stream (highest priority) and events that let the small
// MLP-gradient kernels run beside the grid kernels of the same step: the
// per-block partial reduce beside the hash-grid scatter, the MLP Adam beside
// the grid Adam.  Both pairs touch disjoint memory; the caller's stream waits
// for the side stream before each entry point returns, so its ordering
// contract is unchanged.  NVC_NO_SIDE_STREAM=1 serialises them (A/B).
struct SideStream {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};
inline SideStream* side_stream() {
    if (getenv("NVC_NO_SIDE_STREAM")) return nullptr;
    static thread_local SideStream per_dev[64];   // per host thread: the fork/join events are never shared
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    SideStream& ss = per_dev[dev];
    if (!ss.s) {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        if (cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            ss.s = nullptr;
            return nullptr;
        }
    }
    return &ss;
}

static thread_local char g_err[512];

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return NVC_ERR_CUDA;
    }
    return NVC_OK;
}

namespace {

#ifndef NVC_TRAIN_ROWS
#define NVC_TRAIN_ROWS 32
#endif
constexpr int kRows = NVC_TRAIN_ROWS;   // rows per block in the SIMT MLP kernels
constexpr int kRPT = kRows >= 32 ? 2 : 1;   // rows per thread tile in k_train3 (keeps 256 threads busy)
constexpr int kThreads = 256;

struct Net {
    int n_layers;
    int dims[NVC_MAX_LAYERS + 1];
    int64_t woff[NVC_MAX_LAYERS];   // offset of w_i in params (after the grid)
    int64_t boff[NVC_MAX_LAYERS];
    int64_t grid_count;             // L*T*F
    int64_t mlp_count;
    float alpha;
    int out_sigmoid;
};

Net net_of(const nvc_model* m) {
    Net n;
    n.n_layers = m->n_layers;
    for (int i = 0; i <= m->n_layers; ++i) n.dims[i] = m->dims[i];
    n.grid_count = (int64_t)m->levels * m->table_size * m->features;
    int64_t o = n.grid_count;
    for (int i = 0; i < m->n_layers; ++i) {
        n.woff[i] = o;
        o += (int64_t)m->dims[i + 1] * m->dims[i];
        n.boff[i] = o;
        o += m->dims[i + 1];
    }
    n.mlp_count = o - n.grid_count;
    n.alpha = m->alpha;
    n.out_sigmoid = m->out_sigmoid;
    return n;
}

// Where gradients accumulate: the dense int64 grad_fx (param order), or the
// compact mode (nvc.h): entry e -> slot rank(e) of the batch's sorted entry set.
struct GradSink {
    int64_t* dense;
    const uint32_t* bits;
    const int32_t* off;
    int64_t* comp;
    int64_t comp_entries;
    int F;
    int64_t grid_count;
};

GradSink sink_of(const nvc_model* m) {
    GradSink gs;
    gs.dense = m->grad_c ? nullptr : m->grad_fx;
    gs.bits = m->touch_bits;
    gs.off = m->touch_off;
    gs.comp = m->grad_c;
    gs.comp_entries = m->grad_c_entries;
    gs.F = m->features;
    gs.grid_count = (int64_t)m->levels * m->table_size * m->features;
    return gs;
}

__device__ __forceinline__ bool grid_touched(const GradSink& gs, int64_t e) { return (gs.bits[e >> 5] >> (e & 31)) & 1u; }
// gradient slot (feature 0) of table entry e; in compact mode e must be marked
__device__ __forceinline__ int64_t* grid_grad(const GradSink& gs, int64_t e) {
    if (gs.comp) {
        const uint32_t w = gs.bits[e >> 5];
        const int32_t r = gs.off[e >> 5] + __popc(w & ((1u << (e & 31)) - 1u));
        return gs.comp + (int64_t)r * gs.F;
    }
    return gs.dense + e * gs.F;
}
__device__ __forceinline__ int64_t* mlp_grad(const GradSink& gs, int64_t j) {
    return gs.comp ? gs.comp + gs.comp_entries * gs.F + j : gs.dense + gs.grid_count + j;
}

int validate(const nvc_model* m) {
    NVC_REQUIRE(m, "null model");
    NVC_REQUIRE(m->levels >= 1 && m->levels <= NVC_MAX_LEVELS, "levels out of range");
    NVC_REQUIRE(m->features >= 1 && m->features <= 8, "features out of range");
    NVC_REQUIRE(m->table_size >= 1 && (m->table_size & (m->table_size - 1)) == 0 && m->table_size <= (1ll << 30),
                "table_size must be a power of two <= 2^30");
    NVC_REQUIRE(m->n_layers >= 1 && m->n_layers <= NVC_MAX_LAYERS, "n_layers out of range");
    NVC_REQUIRE(m->dims[0] == m->levels * m->features, "dims[0] must equal levels*features");
    for (int i = 0; i <= m->n_layers; ++i) NVC_REQUIRE(m->dims[i] >= 1 && m->dims[i] <= 256, "layer width out of range");
    NVC_REQUIRE(m->params, "params not bound");
    return NVC_OK;
}

inline int grid1(int64_t n, int bs) { return (int)((n + bs - 1) / bs); }

// ---------------------------------------------------------------------------
// encoder, exact reference op order on the f32 master table
// ---------------------------------------------------------------------------
__device__ __forceinline__ void encode_level_f32(const GridDev& g, const float* __restrict__ table,
                                                 const double q[3], int l, float* out,
                                                 int32_t* idx_out, double* w_out) {
    int c0[3];
    double f[3];
    cell(g.res[l], q, c0, f);
    float acc[8];
    for (int k = 0; k < g.F; ++k) acc[k] = 0.0f;
    const float* tl = table + (int64_t)l * g.T * g.F;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t idx = corner_index(g, l, c0, (c >> 2) & 1, (c >> 1) & 1, c & 1);
        const double w = corner_weight(f, c);
        const float wf = (float)w;
        if (idx_out) idx_out[c] = (int32_t)idx;
        if (w_out) w_out[c] = w;
        for (int k = 0; k < g.F; ++k) acc[k] = __fadd_rn(acc[k], __fmul_rn(wf, __ldg(tl + (int64_t)idx * g.F + k)));
    }
    for (int k = 0; k < g.F; ++k) out[k] = acc[k];
}

__global__ void k_encode(GridDev g, const float* __restrict__ table, const double* __restrict__ pos, int64_t n,
                         float* __restrict__ feats, int32_t* __restrict__ idx_out, double* __restrict__ w_out) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t i = t / g.L;
    const int l = (int)(t - i * g.L);
    if (i >= n) return;
    const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
    double q[3];
    normalize(g, p, q);
    encode_level_f32(g, table, q, l, feats + i * g.L * g.F + l * g.F,
                     idx_out ? idx_out + (i * g.L + l) * 8 : nullptr, w_out ? w_out + (i * g.L + l) * 8 : nullptr);
}

// ---------------------------------------------------------------------------
// SIMT fp32 MLP over a tile of kRows rows (forward; backward when training)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float leaky(float z, float a) { return z >= 0.0f ? z : __fmul_rn(a, z); }

__device__ __forceinline__ float sigmoid_ref(float z) {  // mlp.py:101-107
    if (z >= 0.0f) return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-z)));
    const float e = expf(z);
    return __fdiv_rn(e, __fadd_rn(1.0f, e));
}

// z[r][n] = sum_k a[r][k] * W[n][k] + b[n] for R rows
__device__ __forceinline__ void dense_fwd(const float* __restrict__ W, const float* __restrict__ bias,
                                          const float* a, int K, int N, float* z) {
    for (int e = threadIdx.x; e < kRows * N; e += blockDim.x) {
        const int r = e / N, n = e - r * N;
        const float* w = W + (int64_t)n * K;
        const float* ar = a + r * K;
        float acc = 0.0f;
        for (int k = 0; k < K; ++k) acc = fmaf(ar[k], __ldg(w + k), acc);
        z[e] = acc + __ldg(bias + n);
    }
}

struct TileLayout {   // smem offsets (floats) of per-layer buffers
    int act[NVC_MAX_LAYERS + 1];   // act[i] = input of layer i (act[0] = features), act[n] = output
    int z[NVC_MAX_LAYERS];
    int scratch;                    // two dz buffers of the max width
    int wmax;
    int total;
};

__host__ __device__ inline TileLayout tile_layout(const Net& net) {
    TileLayout t;
    int o = 0, wmax = 0;
    for (int i = 0; i <= net.n_layers; ++i) {
        t.act[i] = o;
        o += kRows * net.dims[i];
        if (net.dims[i] > wmax) wmax = net.dims[i];
    }
    for (int i = 0; i < net.n_layers; ++i) {
        t.z[i] = o;
        o += kRows * net.dims[i + 1];
    }
    t.scratch = o;
    t.wmax = wmax;
    o += 2 * kRows * wmax;
    t.total = o;
    return t;
}

// Forward (and backward when `train`) for rows [row0, row0+kRows) of the
// caller's row range [lo, hi).
template <bool kTrain>
__global__ void __launch_bounds__(kThreads) k_mlp(GridDev g, Net net, const float* __restrict__ params,
                                                 const double* __restrict__ pos, int64_t b_max,
                                                 const int64_t* __restrict__ b_dev, int shard, int n_shards,
                                                 const float* __restrict__ tgt, const float* __restrict__ mask,
                                                 float* __restrict__ out, GradSink gs,
                                                 float* __restrict__ part_w, double* __restrict__ part_loss) {
    extern __shared__ float sm[];
    const TileLayout tl = tile_layout(net);
    const int64_t b = b_dev ? *b_dev : b_max;
    int64_t lo, hi;
    shard_range(b, shard, n_shards, lo, hi);
    const int64_t row0 = lo + (int64_t)blockIdx.x * kRows;
    const int nr = (int)max((int64_t)0, min((int64_t)kRows, hi - row0));
    const int D0 = net.dims[0];
    const int K = net.dims[net.n_layers];

    // ---- encode rows into act[0] (zero rows past the end) ----
    for (int e = threadIdx.x; e < kRows * g.L; e += blockDim.x) {
        const int r = e / g.L, l = e - r * g.L;
        float* dst = sm + tl.act[0] + r * D0 + l * g.F;
        if (r < nr) {
            const int64_t i = row0 + r;
            const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            double q[3];
            normalize(g, p, q);
            encode_level_f32(g, params, q, l, dst, nullptr, nullptr);
        } else {
            for (int k = 0; k < g.F; ++k) dst[k] = 0.0f;
        }
    }
    __syncthreads();

    // ---- forward ----
    for (int i = 0; i < net.n_layers; ++i) {
        const int Kin = net.dims[i], N = net.dims[i + 1];
        dense_fwd(params + net.woff[i], params + net.boff[i], sm + tl.act[i], Kin, N, sm + tl.z[i]);
        __syncthreads();
        const bool last = i == net.n_layers - 1;
        for (int e = threadIdx.x; e < kRows * N; e += blockDim.x) {
            const float z = sm[tl.z[i] + e];
            sm[tl.act[i + 1] + e] = (last && net.out_sigmoid) ? sigmoid_ref(z) : leaky(z, net.alpha);
        }
        __syncthreads();
    }

    if (!kTrain) {
        for (int e = threadIdx.x; e < nr * K; e += blockDim.x) {
            const float v = sm[tl.act[net.n_layers] + e];
            out[(row0 - lo) * K + e] = net.out_sigmoid ? fminf(fmaxf(v, 1e-6f), 0.999999f) : v;
        }
        return;
    }

    // ---- loss + d_out (mlp.py:143-149, 160-168) ----
    float* dz = sm + tl.scratch;
    const float inv_bk = (float)(b * K);
    double lsum = 0.0;
    for (int e = threadIdx.x; e < kRows * K; e += blockDim.x) {
        const int r = e / K;
        float d = 0.0f;
        if (r < nr) {
            const int64_t li = (row0 - lo) * K + e;   // shard-local
            const float s = sm[tl.act[net.n_layers] + e];
            const float outc = net.out_sigmoid ? fminf(fmaxf(s, 1e-6f), 0.999999f) : s;
            const float t = tgt[li];
            const float mk = mask ? mask[li] : 1.0f;
            float dd = __fsub_rn(outc, t);
            if (mask) dd = __fmul_rn(dd, mk);
            lsum += (double)__fmul_rn(dd, dd);
            float dout = __fdiv_rn(__fmul_rn(2.0f, __fsub_rn(s, t)), inv_bk);
            if (mask) dout = __fmul_rn(dout, mk);
            d = net.out_sigmoid ? __fmul_rn(__fmul_rn(dout, s), __fsub_rn(1.0f, s))
                                : (sm[tl.z[net.n_layers - 1] + e] >= 0.0f ? dout : __fmul_rn(dout, net.alpha));
        }
        dz[e] = d;
    }
    // block reduce of the loss (fixed order: warp shuffles then warps in order)
    {
        __shared__ double s_l[kThreads / 32];
        for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if ((threadIdx.x & 31) == 0) s_l[threadIdx.x >> 5] = lsum;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_l[w];
            part_loss[blockIdx.x] = t / (double)K;
        }
    }
    __syncthreads();

    // ---- backward (mlp.py:170-183) ----
    float* part = part_w + (int64_t)blockIdx.x * net.mlp_count;
    float* dz_cur = dz;
    float* dz_nxt = dz + kRows * tl.wmax;   // scratch holds two max-width buffers
    for (int i = net.n_layers - 1; i >= 0; --i) {
        const int Kin = net.dims[i], N = net.dims[i + 1];
        const float* a = sm + tl.act[i];
        // g_W[n][k] = sum_r dz[r][n] a[r][k]; g_b[n] = sum_r dz[r][n]
        float* gw = part + (net.woff[i] - net.grid_count);
        for (int e = threadIdx.x; e < N * Kin; e += blockDim.x) {
            const int n = e / Kin, k = e - n * Kin;
            float acc = 0.0f;
            for (int r = 0; r < kRows; ++r) acc = fmaf(dz_cur[r * N + n], a[r * Kin + k], acc);
            gw[e] = acc;
        }
        float* gb = part + (net.boff[i] - net.grid_count);
        for (int n = threadIdx.x; n < N; n += blockDim.x) {
            float acc = 0.0f;
            for (int r = 0; r < kRows; ++r) acc += dz_cur[r * N + n];
            gb[n] = acc;
        }
        // da[r][k] = sum_n dz[r][n] W[n][k], then through leaky'(z_{i-1})
        const float* W = params + net.woff[i];
        for (int e = threadIdx.x; e < kRows * Kin; e += blockDim.x) {
            const int r = e / Kin, k = e - r * Kin;
            float acc = 0.0f;
            for (int n = 0; n < N; ++n) acc = fmaf(dz_cur[r * N + n], __ldg(W + (int64_t)n * Kin + k), acc);
            if (i > 0) acc = sm[tl.z[i - 1] + e] >= 0.0f ? acc : __fmul_rn(acc, net.alpha);
            dz_nxt[e] = acc;
        }
        __syncthreads();
        float* t = dz_cur;
        dz_cur = dz_nxt;
        dz_nxt = t;
    }

    // ---- hash-grid scatter (hashgrid.py:140-151), fixed point, deterministic ----
    for (int e = threadIdx.x; e < nr * g.L; e += blockDim.x) {
        const int r = e / g.L, l = e - r * g.L;
        const int64_t i = row0 + r;
        const double p[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        double q[3];
        normalize(g, p, q);
        int c0[3];
        double f[3];
        cell(g.res[l], q, c0, f);
        const float* up = dz_cur + r * D0 + l * g.F;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t idx = corner_index(g, l, c0, (c >> 2) & 1, (c >> 1) & 1, c & 1);
            const double w = corner_weight(f, c);
            int64_t* gp = grid_grad(gs, (int64_t)l * g.T + idx);
            for (int k = 0; k < g.F; ++k) {
                const float contrib = (float)__dmul_rn(w, (double)up[k]);   // (w * g).astype(f32)
                red_add_fx(gp + k, to_fx((double)contrib));
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Split training step (default when every width is a multiple of 4):
//   k_tr_encode   one thread per (row, level): exact f32 features -> act0
//   k_train3      one block per kRows rows: SIMT fp32 forward / loss /
//                 backward with only W in shared memory (row stride Ki+4, so
//                 both the n-strided forward reads and the k-contiguous
//                 backward reads are bank-conflict free); writes dL/dact0
//   k_tr_scatter  one thread per (row, level): fixed-point hash-grid scatter
// Same arithmetic and the same kRows row partition as k_mlp<true> (so the
// per-block MLP partials, and hence the reduced gradients, are unchanged);
// the phases that were latency-bound inside one block (gathers, atomics)
// now run at full-GPU parallelism.
// ---------------------------------------------------------------------------
struct T3Layout {
    int w[NVC_MAX_LAYERS], ws[NVC_MAX_LAYERS];   // float offset and row stride of W_l [N][Ki+4]
    int bias[NVC_MAX_LAYERS];
    int act[NVC_MAX_LAYERS + 1];                 // act_l [kRows][D_l]
    int dz0, dz1;                                // two [kRows][Dmax] buffers
    int total;
    int rbits;    // diagnostics (NVC_T3_BITS): GEMM operands rounded to this many significant bits; 0 = off
    int rwhat;    // which operands (NVC_T3_WHAT bits): 1 weights, 2 activations, 4 deltas
};

// round to m significant bits, nearest-even (the precision study behind the
// tensor-core step's operand split)
__device__ __forceinline__ float round_bits(float x, int m) {
    const int d = 24 - m;
    uint32_t u = __float_as_uint(x);
    u += (1u << (d - 1)) - 1u + ((u >> d) & 1u);
    return __uint_as_float(u & ~((1u << d) - 1u));
}

// with_w = false: the layout for MLPs too wide for every W + the activations in
// shared memory (C4: 3x128): one W buffer sized for the largest layer, which
// k_train3<true> refills with the layer it is about to use (forward and the
// backward's dL/dact); same padded row stride Ki+4
__host__ __device__ inline T3Layout t3_layout(const Net& net, bool with_w = true) {
    T3Layout t;
    t.rbits = 0;
    t.rwhat = 7;
    int o = 0, dmax = 0, wmax = 0;
    for (int l = 0; l < net.n_layers; ++l) {
        t.w[l] = o;
        t.ws[l] = net.dims[l] + 4;
        if (with_w) o += net.dims[l + 1] * t.ws[l];
        else if (net.dims[l + 1] * t.ws[l] > wmax) wmax = net.dims[l + 1] * t.ws[l];
        t.bias[l] = o;
        o += (net.dims[l + 1] + 3) / 4 * 4;
    }
    if (!with_w) {   // the shared W buffer
        for (int l = 0; l < net.n_layers; ++l) t.w[l] = o;
        o += wmax;
    }
    for (int l = 0; l <= net.n_layers; ++l) {
        t.act[l] = o;
        o += kRows * net.dims[l];
        if (net.dims[l] > dmax) dmax = net.dims[l];
    }
    t.dz0 = o;
    o += kRows * dmax;
    t.dz1 = o;
    o += kRows * dmax;
    t.total = o;
    return t;
}

struct ShardRows {
    int64_t lo, hi;
};
__device__ __forceinline__ ShardRows shard_rows(int64_t b_max, const int64_t* b_dev, int shard, int n_shards) {
    const int64_t b = b_dev ? *b_dev : b_max;
    ShardRows r;
    shard_range(b, shard, n_shards, r.lo, r.hi);
    return r;
}

__global__ void __launch_bounds__(128) k_tr_encode(GridDev g, const float* __restrict__ params,
                                                   const double* __restrict__ pos, int64_t b_max,
                                                   const int64_t* __restrict__ b_dev, int shard, int n_shards,
                                                   float* __restrict__ act0) {
    const ShardRows sr = shard_rows(b_max, b_dev, shard, n_shards);
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = t / g.L;
    const int l = (int)(t - r * g.L);
    if (sr.lo + r >= sr.hi) return;
    const int64_t i = sr.lo + r;
    const double pp[3] = {__ldg(pos + 3 * i), __ldg(pos + 3 * i + 1), __ldg(pos + 3 * i + 2)};
    double q[3];
    normalize(g, pp, q);
    encode_level_f32(g, params, q, l, act0 + r * (g.L * g.F) + l * g.F, nullptr, nullptr);
}

template <bool kWG>
__global__ void __launch_bounds__(kThreads, 4) k_train3(Net net, T3Layout tl, const float* __restrict__ params,
                                                       const float* __restrict__ act0g, int64_t b_max,
                                                       const int64_t* __restrict__ b_dev, int shard, int n_shards,
                                                       const float* __restrict__ tgt, const float* __restrict__ mask,
                                                       float* __restrict__ dact0g, float* __restrict__ part_w,
                                                       double* __restrict__ part_loss) {
    extern __shared__ __align__(16) float sm[];
    // tl arrives in the parameter bank (indexed per layer without a local-memory copy)
    const int tid = threadIdx.x;
    const ShardRows sr = shard_rows(b_max, b_dev, shard, n_shards);
    const int64_t b = b_dev ? *b_dev : b_max;
    const int64_t r0g = (int64_t)blockIdx.x * kRows;   // shard-local first row
    const int nr = (int)max((int64_t)0, min((int64_t)kRows, (sr.hi - sr.lo) - r0g));
    const int D0 = net.dims[0];
    const int K = net.dims[net.n_layers];

    // ---- W (padded rows), biases, act0 -> smem; all loads issued as float4 ----
    // (kWG: only the biases here; each layer's W is staged right before its use)
    auto stage_w = [&](int l) {
        const int N = net.dims[l + 1], Ki = net.dims[l], kq = Ki / 4;
        const float4* W = reinterpret_cast<const float4*>(params + net.woff[l]);
        float* dst = sm + tl.w[l];
#pragma unroll 4
        for (int e = tid; e < N * kq; e += kThreads) {
            float4 w = __ldg(W + e);
            if (tl.rbits && (tl.rwhat & 1)) w = make_float4(round_bits(w.x, tl.rbits), round_bits(w.y, tl.rbits),
                                          round_bits(w.z, tl.rbits), round_bits(w.w, tl.rbits));
            const int n = e / kq, k = (e - n * kq) * 4;
            *reinterpret_cast<float4*>(dst + n * tl.ws[l] + k) = w;
        }
    };
    for (int l = 0; l < net.n_layers; ++l) {
        if (!kWG) stage_w(l);
        for (int n = tid; n < net.dims[l + 1]; n += kThreads) sm[tl.bias[l] + n] = __ldg(params + net.boff[l] + n);
    }
    {
        const int q0 = D0 / 4;
        const float4* src = reinterpret_cast<const float4*>(act0g + r0g * D0);
        float4* dst = reinterpret_cast<float4*>(sm + tl.act[0]);
        for (int e = tid; e < kRows * q0; e += kThreads) {
            float4 a = (e / q0 < nr) ? __ldg(src + e) : make_float4(0.f, 0.f, 0.f, 0.f);
            if (tl.rbits && (tl.rwhat & 2)) a = make_float4(round_bits(a.x, tl.rbits), round_bits(a.y, tl.rbits),
                                          round_bits(a.z, tl.rbits), round_bits(a.w, tl.rbits));
            dst[e] = a;
        }
    }
    __syncthreads();

    // ---- forward: z = act W^T + b; thread tile 2 rows x 4 outputs (n strided by N/4) ----
    for (int l = 0; l < net.n_layers; ++l) {
        const int Ki = net.dims[l], N = net.dims[l + 1], ng = N / 4, S = tl.ws[l];
        const float* A = sm + tl.act[l];
        if (kWG) {
            if (l > 0) __syncthreads();   // (l = 0: the barrier after the act0 load follows)
            stage_w(l);
            __syncthreads();
        }
        const float* W = sm + tl.w[l];
        float* out = sm + tl.act[l + 1];
        const bool last = l == net.n_layers - 1;
        for (int t = tid; t < (kRows / kRPT) * ng; t += kThreads) {
            const int r0 = (t / ng) * kRPT, nn = t % ng;
            float acc[kRPT][4] = {};
            for (int k = 0; k < Ki; k += 4) {
                float4 av[kRPT];
#pragma unroll
                for (int i = 0; i < kRPT; ++i) av[i] = *reinterpret_cast<const float4*>(A + (r0 + i) * Ki + k);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 w = *reinterpret_cast<const float4*>(W + (nn + j * ng) * S + k);
#pragma unroll
                    for (int i = 0; i < kRPT; ++i) acc[i][j] = fmaf(av[i].x, w.x, acc[i][j]);
#pragma unroll
                    for (int i = 0; i < kRPT; ++i) acc[i][j] = fmaf(av[i].y, w.y, acc[i][j]);
#pragma unroll
                    for (int i = 0; i < kRPT; ++i) acc[i][j] = fmaf(av[i].z, w.z, acc[i][j]);
#pragma unroll
                    for (int i = 0; i < kRPT; ++i) acc[i][j] = fmaf(av[i].w, w.w, acc[i][j]);
                }
            }
#pragma unroll
            for (int i = 0; i < kRPT; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int n = nn + j * ng;
                    const float z = acc[i][j] + sm[tl.bias[l] + n];
                    const float o = (last && net.out_sigmoid) ? sigmoid_ref(z) : leaky(z, net.alpha);
                    out[(r0 + i) * N + n] = (tl.rbits && (tl.rwhat & 2) && !last) ? round_bits(o, tl.rbits) : o;
                }
        }
        __syncthreads();
    }

    // ---- loss + output delta (mlp.py:143-149, 160-168) ----
    float* dz = sm + tl.dz0;
    float* dzn = sm + tl.dz1;
    const float bk = (float)(b * K);
    double lsum = 0.0;
    for (int e = tid; e < kRows * K; e += kThreads) {
        const int r = e / K;
        float d = 0.0f;
        if (r < nr) {
            const int64_t li = r0g * K + e;
            const float sgm = sm[tl.act[net.n_layers] + e];
            const float outc = net.out_sigmoid ? fminf(fmaxf(sgm, 1e-6f), 0.999999f) : sgm;
            const float t = tgt[li];
            const float mk = mask ? mask[li] : 1.0f;
            float dd = __fsub_rn(outc, t);
            if (mask) dd = __fmul_rn(dd, mk);
            lsum += (double)__fmul_rn(dd, dd);
            float dout = __fdiv_rn(__fmul_rn(2.0f, __fsub_rn(sgm, t)), bk);
            if (mask) dout = __fmul_rn(dout, mk);
            d = net.out_sigmoid ? __fmul_rn(__fmul_rn(dout, sgm), __fsub_rn(1.0f, sgm))
                                : (sgm >= 0.0f ? dout : __fmul_rn(dout, net.alpha));
        }
        dz[e] = (tl.rbits && (tl.rwhat & 4)) ? round_bits(d, tl.rbits) : d;
    }
    {
        __shared__ double s_l[kThreads / 32];
        for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        if ((tid & 31) == 0) s_l[tid >> 5] = lsum;
        __syncthreads();
        if (tid == 0) {
            double t = 0.0;
            for (int w = 0; w < kThreads / 32; ++w) t += s_l[w];
            part_loss[blockIdx.x] = t / (double)K;
        }
    }
    __syncthreads();

    // ---- backward (mlp.py:170-183) ----
    float* part = part_w + (int64_t)blockIdx.x * net.mlp_count;
    for (int l = net.n_layers - 1; l >= 0; --l) {
        const int Ki = net.dims[l], N = net.dims[l + 1], S = tl.ws[l];
        const float* A = sm + tl.act[l];
        // grad W[n][k] = sum_r dz[r][n] A[r][k]   (4x4 tiles)
        float* gw = part + (net.woff[l] - net.grid_count);
        const int kg = Ki / 4;
        for (int t = tid; t < (N / 4) * kg; t += kThreads) {
            const int n0 = (t / kg) * 4, k0 = (t % kg) * 4;
            float acc[4][4] = {};
            for (int r = 0; r < kRows; ++r) {
                const float4 d4 = *reinterpret_cast<const float4*>(dz + r * N + n0);
                const float4 a4 = *reinterpret_cast<const float4*>(A + r * Ki + k0);
                const float dv[4] = {d4.x, d4.y, d4.z, d4.w}, av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(dv[i], av[j], acc[i][j]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
                *reinterpret_cast<float4*>(gw + (n0 + i) * Ki + k0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        }
        float* gb = part + (net.boff[l] - net.grid_count);
        for (int n = tid; n < N; n += kThreads) {
            float acc = 0.0f;
            for (int r = 0; r < kRows; ++r) acc += dz[r * N + n];
            gb[n] = acc;
        }
        // grad act[r][k] = sum_n dz[r][n] W[n][k], through leaky'(z_{l-1}) (2x4 tiles)
        if (kWG && l != net.n_layers - 1) {   // (the last layer's W is still staged from the forward pass)
            __syncthreads();   // the previous layer's dL/dact pass is done with the W buffer
            stage_w(l);
            __syncthreads();
        }
        const float* W = sm + tl.w[l];
        for (int t = tid; t < (kRows / kRPT) * kg; t += kThreads) {
            const int r0 = (t / kg) * kRPT, k0 = (t % kg) * 4;
            float acc[kRPT][4] = {};
            for (int n = 0; n < N; ++n) {
                const float4 w = *reinterpret_cast<const float4*>(W + n * S + k0);
#pragma unroll
                for (int i = 0; i < kRPT; ++i) {
                    const float d = dz[(r0 + i) * N + n];
                    acc[i][0] = fmaf(d, w.x, acc[i][0]);
                    acc[i][1] = fmaf(d, w.y, acc[i][1]);
                    acc[i][2] = fmaf(d, w.z, acc[i][2]);
                    acc[i][3] = fmaf(d, w.w, acc[i][3]);
                }
            }
            if (l > 0) {
                // 16-byte shared accesses (a thread's 4 columns are contiguous): scalar ones
                // at a 4-word stride across the warp were 4-way bank conflicts
#pragma unroll
                for (int i = 0; i < kRPT; ++i) {
                    const float4 a4 = *reinterpret_cast<const float4*>(A + (r0 + i) * Ki + k0);
                    const float av[4] = {a4.x, a4.y, a4.z, a4.w};
                    float o[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float v = acc[i][j];
                        if (!(av[j] >= 0.0f)) v = __fmul_rn(v, net.alpha);
                        o[j] = (tl.rbits && (tl.rwhat & 4)) ? round_bits(v, tl.rbits) : v;
                    }
                    *reinterpret_cast<float4*>(dzn + (r0 + i) * Ki + k0) = make_float4(o[0], o[1], o[2], o[3]);
                }
            } else {
#pragma unroll
                for (int i = 0; i < kRPT; ++i)
                    if (r0 + i < nr)
                        *reinterpret_cast<float4*>(dact0g + (r0g + r0 + i) * Ki + k0) =
                            make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
            }
        }
        __syncthreads();
        float* t = dz;
        dz = dzn;
        dzn = t;
    }
}

__global__ void __launch_bounds__(128) k_tr_scatter(GridDev g, const double* __restrict__ pos, int64_t b_max,
                                                    const int64_t* __restrict__ b_dev, int shard, int n_shards,
                                                    const float* __restrict__ dact0, GradSink gs) {
    const ShardRows sr = shard_rows(b_max, b_dev, shard, n_shards);
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = t / g.L;
    const int l = (int)(t - r * g.L);
    if (sr.lo + r >= sr.hi) return;
    const int64_t i = sr.lo + r;
    const double pp[3] = {__ldg(pos + 3 * i), __ldg(pos + 3 * i + 1), __ldg(pos + 3 * i + 2)};
    double q[3];
    normalize(g, pp, q);
    int c0[3];
    double f[3];
    cell(g.res[l], q, c0, f);
    float up[8];
    for (int k = 0; k < g.F; ++k) up[k] = __ldg(dact0 + r * (g.L * g.F) + l * g.F + k);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const uint32_t idx = corner_index(g, l, c0, (c >> 2) & 1, (c >> 1) & 1, c & 1);
        const double w = corner_weight(f, c);
        int64_t* gp = grid_grad(gs, (int64_t)l * g.T + idx);
        for (int k = 0; k < g.F; ++k) {
            const float contrib = (float)__dmul_rn(w, (double)up[k]);   // (w * g).astype(f32), hashgrid.py:146-151
            red_add_fx(gp + k, to_fx((double)contrib));
        }
    }
}

// ---------------------------------------------------------------------------
// Compact data-parallel gradient exchange.  Every rank builds the same global
// batch, so the set of table entries the batch touches is identical on all
// ranks: mark them in a bitmap (one bit per L*T entry), compact to a sorted
// entry list, and allreduce only those entries' fixed-point gradients (plus
// the MLP part) instead of the whole 8 B x param_count accumulator.  Untouched
// entries hold zero on every rank, so the result equals the dense allreduce.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_touch_mark(GridDev g, const double* __restrict__ pos, int64_t b_max,
                                                    const int64_t* __restrict__ b_dev, uint32_t* __restrict__ bits) {
    const int64_t b = b_dev ? *b_dev : b_max;
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t r = t / g.L;
    const int l = (int)(t - r * g.L);
    if (r >= b) return;
    const double pp[3] = {__ldg(pos + 3 * r), __ldg(pos + 3 * r + 1), __ldg(pos + 3 * r + 2)};
    double q[3];
    normalize(g, pp, q);
    int c0[3];
    double f[3];
    cell(g.res[l], q, c0, f);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int64_t e = (int64_t)l * g.T + corner_index(g, l, c0, (c >> 2) & 1, (c >> 1) & 1, c & 1);
        atomicOr(bits + (e >> 5), 1u << (e & 31));
    }
}

// per 1024-word chunk: number of set bits
__global__ void __launch_bounds__(256) k_touch_count(const uint32_t* __restrict__ bits, int64_t n_words,
                                                     int* __restrict__ chunk_count) {
    __shared__ int warp_tot[8];
    const int64_t w0 = (int64_t)blockIdx.x * 1024;
    int c = 0;
    for (int i = threadIdx.x; i < 1024; i += 256)
        if (w0 + i < n_words) c += __popc(bits[w0 + i]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0) warp_tot[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < 8; ++w) t += warp_tot[w];
        chunk_count[blockIdx.x] = t;
    }
}

// exclusive scan of the chunk counts (one block, sequential chunks of 1024)
__global__ void __launch_bounds__(1024) k_touch_scan(int* __restrict__ chunk_count, int n_chunks,
                                                     int64_t* __restrict__ total) {
    __shared__ int warp_sum[32];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < n_chunks; base += 1024) {
        const int i = base + threadIdx.x;
        const int v = i < n_chunks ? chunk_count[i] : 0;
        int incl = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        if (lane == 31) warp_sum[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int x = warp_sum[lane];
            int xi = x;
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += y;
            }
            warp_sum[lane] = xi - x;
        }
        __syncthreads();
        const int excl = carry + warp_sum[wid] + incl - v;
        if (i < n_chunks) chunk_count[i] = excl;
        __syncthreads();
        if (threadIdx.x == 1023) carry = excl + v;
        __syncthreads();
    }
    if (threadIdx.x == 0 && total) *total = carry;
}

// write the sorted entry list: chunk offset + prefix of popcounts inside the chunk
__global__ void __launch_bounds__(1024) k_touch_emit(const uint32_t* __restrict__ bits, int64_t n_words,
                                                     const int* __restrict__ chunk_off, int32_t* __restrict__ idx) {
    __shared__ int warp_sum[32];
    const int64_t wi = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    const uint32_t word = wi < n_words ? bits[wi] : 0u;
    const int v = __popc(word);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int x = warp_sum[lane];
        int xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        warp_sum[lane] = xi - x;
    }
    __syncthreads();
    int o = chunk_off[blockIdx.x] + warp_sum[wid] + incl - v;
    uint32_t w = word;
    while (w) {
        const int bit = __ffs(w) - 1;
        w &= w - 1;
        idx[o++] = (int32_t)(wi * 32 + bit);
    }
}

// per-word rank of the word's first marked entry (compact gradient mode)
__global__ void __launch_bounds__(1024) k_touch_offsets(const uint32_t* __restrict__ bits, int64_t n_words,
                                                        const int* __restrict__ chunk_off, int32_t* __restrict__ off) {
    __shared__ int warp_sum[32];
    const int64_t wi = (int64_t)blockIdx.x * 1024 + threadIdx.x;
    const int v = wi < n_words ? __popc(bits[wi]) : 0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        const int x = warp_sum[lane];
        int xi = x;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        warp_sum[lane] = xi - x;
    }
    __syncthreads();
    if (wi < n_words) off[wi] = chunk_off[blockIdx.x] + warp_sum[wid] + incl - v;
}

// buf = [grad of listed entries (F each, zero past the count) | MLP gradients]
__global__ void k_grad_pack(const int64_t* __restrict__ fx, const int32_t* __restrict__ idx,
                            const int64_t* __restrict__ count, int64_t max_entries, int F, int64_t grid_count,
                            int64_t mlp_count, int64_t* __restrict__ buf) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ng = max_entries * F;
    if (t < ng) {
        const int64_t i = t / F;
        buf[t] = i < *count ? fx[(int64_t)idx[i] * F + (t - i * F)] : 0;
    } else if (t < ng + mlp_count) {
        buf[t] = fx[grid_count + (t - ng)];
    }
}

__global__ void k_grad_unpack(int64_t* __restrict__ fx, const int32_t* __restrict__ idx,
                              const int64_t* __restrict__ count, int64_t max_entries, int F, int64_t grid_count,
                              int64_t mlp_count, const int64_t* __restrict__ buf) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t ng = max_entries * F;
    if (t < ng) {
        const int64_t i = t / F;
        if (i < *count) fx[(int64_t)idx[i] * F + (t - i * F)] = buf[t];
    } else if (t < ng + mlp_count) {
        fx[grid_count + (t - ng)] = buf[t];
    }
}

// fixed-order reduction of the per-block MLP partials and loss partials:
// block = 32 parameters x 8 warps; warp w sums partial blocks w, w+8, ...
// in order, then the 8 warp sums are combined in warp order (deterministic).
__global__ void __launch_bounds__(256) k_reduce_parts(const float* __restrict__ part_w,
                                                      const double* __restrict__ part_loss, int nblk,
                                                      int64_t mlp_count, int64_t grid_count,
                                                      GradSink gs, double* __restrict__ loss_out,
                                                      int64_t b_max, const int64_t* __restrict__ b_dev) {
    // Each 32-row block's partial is rounded to fixed point on its own and the
    // blocks are summed as integers: the MLP gradient then depends only on which
    // rows form each block, not on how blocks are split over data-parallel ranks
    // (shards aligned to 32 rows reproduce the full batch bit for bit).
    __shared__ long long s_acc[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    long long acc = 0;
    if (j < mlp_count) {
        // loads batched so eight are in flight per thread
        int b = w;
        for (; b + 56 < nblk; b += 64) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldg(part_w + (int64_t)(b + 8 * u) * mlp_count + j);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc += to_fx_mlp((double)v[u]);
        }
        for (; b < nblk; b += 8) acc += to_fx_mlp((double)__ldg(part_w + (int64_t)b * mlp_count + j));
    }
    s_acc[w][lane] = acc;
    __syncthreads();
    if (w == 0 && j < mlp_count) {
        long long t = 0;
        for (int i = 0; i < 8; ++i) t += s_acc[i][lane];
        *mlp_grad(gs, j) += t;
    }
    if (blockIdx.x == 0 && w == 1 && loss_out) {
        double t = 0.0;
        for (int b = lane; b < nblk; b += 32) t += part_loss[b];
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) {
            const int64_t b = b_dev ? *b_dev : b_max;
            loss_out[0] = t;                                  // sum over the shard's rows
            loss_out[1] = b > 0 ? t / (double)b : 0.0;         // its share of the global-batch mean
        }
    }
}

// ---------------------------------------------------------------------------
// Adam (mlp.py:203-218): exact FP32 op order, dense over every parameter
// ---------------------------------------------------------------------------
struct AdamK {
    float b1, c1, b2, c2, b1c, b2c, lr, eps;
    double inv_b1c, inv_b2c;   // RN(1 / (double)b1c), RN(1 / (double)b2c)
};

// One Adam element update with the reference's float32 rounding
// (mlp.py:209-217).  Quotients by the per-step constants use
// (float)(x * RN(1/c)) in binary64: a float/float quotient is never a float
// midpoint and lies >= 2^-49 (relative) from one, so the <= 2^-52 binary64
// error cannot change the float rounding; the variable quotient is an IEEE
// float division.
__device__ __forceinline__ float adam1(float p, float g, float& m, float& v, const AdamK& a) {
    m = __fadd_rn(__fmul_rn(m, a.b1), __fmul_rn(a.c1, g));
    v = __fadd_rn(__fmul_rn(v, a.b2), __fmul_rn(__fmul_rn(a.c2, g), g));
    const float mh = (float)__dmul_rn((double)m, a.inv_b1c);
    const float vh = (float)__dmul_rn((double)v, a.inv_b2c);
    const float num = __fmul_rn(a.lr, mh);
    const float den = __fadd_rn(__fsqrt_rn(vh), a.eps);
    return __fsub_rn(p, __fdiv_rn(num, den));   // float32 '/' (IEEE, correctly rounded)
}

// wpack offset (halfs) of W_i[n][k] in the tcgen05 swizzled K-major layout
__host__ __device__ inline int64_t wpack_index(const Net& net, int i, int n, int k) {
    int np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    umma_pads(net.dims, net.n_layers, np, kp);
    int64_t o = 0;
    for (int j = 0; j < i; ++j) o += umma_block_halfs(np[j], kp[j]);
    return o + umma_off(n, k, np[i], kp[i]) / 2;
}

// transposed packs (the backward dA = dZ . W operand of the tensor-core training
// step) follow the forward blocks: block l is W_l^T, [kp x np] K-major
__host__ __device__ inline bool wpack_has_t(const Net& net) {
    int np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    umma_pads(net.dims, net.n_layers, np, kp);
    for (int j = 0; j < net.n_layers; ++j)
        if (np[j] != 16 && np[j] != 32 && np[j] % 64 != 0) return false;
    return true;
}
__host__ __device__ inline int64_t wpack_t_index(const Net& net, int i, int n, int k) {
    int np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    umma_pads(net.dims, net.n_layers, np, kp);
    int64_t o = 0;
    for (int j = 0; j < net.n_layers; ++j) o += umma_block_halfs(np[j], kp[j]);
    for (int j = 0; j < i; ++j) o += umma_block_halfs(kp[j], np[j]);
    return o + umma_off(k, n, kp[i], np[i]) / 2;
}

__device__ __forceinline__ void put_pair(uint16_t* t2, int64_t i, int F, int64_t T, uint16_t h) {
    const int64_t e = i / F, f = i - e * F;
    t2[e * 2 * F + f] = h;                               // own slot, low half
    t2[pair_prev(e, T) * 2 * F + F + f] = h;             // previous slot's x-neighbour half
}

// Generic grid Adam: one parameter per thread.  The fixed-point accumulator
// is zero wherever no sample touched the entry, so it is read densely and
// cleared where nonzero (after a data-parallel allreduce it is already the
// global sum).
__global__ void __launch_bounds__(256) k_adam_flat(float* __restrict__ p, float* __restrict__ m,
                                                   float* __restrict__ v, GradSink gs,
                                                   uint16_t* __restrict__ table_h, int64_t n, int F, AdamK a,
                                                   int64_t T) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t e = i / F;
    long long q = 0;
    if (!gs.comp || grid_touched(gs, e)) {
        int64_t* gq = grid_grad(gs, e) + (i - e * F);
        q = *gq;
        if (q) *gq = 0;
    }
    float mm = m[i], vv = v[i];
    const float pn = adam1(p[i], from_fx(q), mm, vv, a);
    p[i] = pn;
    m[i] = mm;
    v[i] = vv;
    put_pair(table_h, i, F, T, __half_as_ushort(__float2half_rn(pn)));
}

// Streaming grid Adam (F == 2, whole tiles): a persistent kernel whose
// p / m / v / grad_fx tiles move by bulk copies (TMA) into a 4-stage shared
// memory ring and p / m / v go back by bulk stores, so three tiles per block
// are always in flight.  Reading the int64 accumulator densely (instead of
// gathering only touched entries) costs 8 B/parameter of sequential HBM
// traffic but removes every dependent random read from the stream.  The fp16
// x-pair slots (slot e = entry e | entry next(e)) are assembled in registers
// -- a thread's last neighbour comes from the next lane by shuffle -- so each
// thread writes 16 contiguous bytes; only a warp's last slot takes its high
// half from the next warp's lane 0.
#ifndef NVC_ADAM_THREADS
#define NVC_ADAM_THREADS 256
#endif
#ifndef NVC_ADAM_STAGES
#define NVC_ADAM_STAGES 3
#endif
constexpr int kAdamThreads = NVC_ADAM_THREADS, kAdamTile = 4 * kAdamThreads;   // 4 params per thread
constexpr int kAdamStages = NVC_ADAM_STAGES;
struct AdamStage {
    float p[kAdamTile], m[kAdamTile], v[kAdamTile];
    long long q[kAdamTile];
};

// kCompact: the grid gradients come from the compact slots (GradSink) of the
// batch's marked entries instead of a dense int64 tile stream.
template <bool kCompact>
__global__ void __launch_bounds__(kAdamThreads) k_adam_bulk(float* __restrict__ p, float* __restrict__ m,
                                                           float* __restrict__ v, GradSink gs,
                                                           uint16_t* __restrict__ table_h, int64_t ntiles, AdamK a,
                                                           int64_t T, int64_t tile0) {
    int64_t* __restrict__ fx = gs.dense;
    extern __shared__ __align__(128) uint8_t adam_smem[];
    AdamStage* st = reinterpret_cast<AdamStage*>(adam_smem);
    __shared__ uint64_t full[kAdamStages];
    const int tid = threadIdx.x, lane = tid & 31;
    const int n_local = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    auto tile_base = [&](int i) { return (tile0 + blockIdx.x + (int64_t)i * gridDim.x) * kAdamTile; };
    auto issue = [&](int i) {
        const int s = i % kAdamStages;
        const int64_t base = tile_base(i);
        tma::bar_expect_tx(&full[s], kCompact ? 3u * kAdamTile * 4u : (uint32_t)sizeof(AdamStage));
        tma::load(st[s].p, p + base, kAdamTile * 4, &full[s]);
        tma::load(st[s].m, m + base, kAdamTile * 4, &full[s]);
        tma::load(st[s].v, v + base, kAdamTile * 4, &full[s]);
        if (!kCompact) tma::load(st[s].q, fx + base, kAdamTile * 8, &full[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < kAdamStages; ++s) tma::bar_init(&full[s], 1);
        tma::bar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < min(kAdamStages, n_local); ++i) issue(i);
    for (int i = 0; i < n_local; ++i) {
        const int s = i % kAdamStages;
        const int64_t base = tile_base(i);
        const int64_t i0 = base + 4 * tid, e0 = i0 / 2;
        tma::bar_wait(&full[s], (uint32_t)(i / kAdamStages) & 1u);
        float4* P4 = reinterpret_cast<float4*>(st[s].p) + tid;
        float4* M4 = reinterpret_cast<float4*>(st[s].m) + tid;
        float4* V4 = reinterpret_cast<float4*>(st[s].v) + tid;
        longlong2 qa = make_longlong2(0, 0), qb = make_longlong2(0, 0);
        if constexpr (kCompact) {   // entries e0, e0+1 share a bitmap word (e0 even)
            const uint32_t w = __ldg(gs.bits + (e0 >> 5));
            const int b = (int)(e0 & 31);
            if ((w >> b) & 3u) {
                const int32_t r = __ldg(gs.off + (e0 >> 5)) + __popc(w & ((1u << b) - 1u));
                longlong2* g2 = reinterpret_cast<longlong2*>(gs.comp) + r;   // F == 2: one slot = 16 B
                if ((w >> b) & 1u) {
                    qa = *g2;
                    *g2 = make_longlong2(0, 0);
                    ++g2;
                }
                if ((w >> (b + 1)) & 1u) {
                    qb = *g2;
                    *g2 = make_longlong2(0, 0);
                }
            }
        } else {
            const longlong2* Q2 = reinterpret_cast<const longlong2*>(st[s].q) + 2 * tid;
            qa = Q2[0];
            qb = Q2[1];
            if (qa.x | qa.y) *reinterpret_cast<longlong2*>(fx + i0) = make_longlong2(0, 0);
            if (qb.x | qb.y) *reinterpret_cast<longlong2*>(fx + i0 + 2) = make_longlong2(0, 0);
        }
        const long long q[4] = {qa.x, qa.y, qb.x, qb.y};
        float4 P = *P4, M = *M4, V = *V4;
        float* Pp = &P.x;
        float* Mp = &M.x;
        float* Vp = &V.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) Pp[j] = adam1(Pp[j], from_fx(q[j]), Mp[j], Vp[j], a);
        *P4 = P;
        *M4 = M;
        *V4 = V;
        const uint32_t E0 = (uint32_t)__half_as_ushort(__float2half_rn(Pp[0])) |
                            ((uint32_t)__half_as_ushort(__float2half_rn(Pp[1])) << 16);
        const uint32_t E1 = (uint32_t)__half_as_ushort(__float2half_rn(Pp[2])) |
                            ((uint32_t)__half_as_ushort(__float2half_rn(Pp[3])) << 16);
        const uint32_t nxt = __shfl_down_sync(0xffffffffu, E0, 1);
        uint32_t* slot = reinterpret_cast<uint32_t*>(table_h + e0 * 4);   // 2 words per slot
        if (lane < 31) {
            *reinterpret_cast<uint4*>(slot) = make_uint4(E0, E1, E1, nxt);
        } else {
            *reinterpret_cast<uint2*>(slot) = make_uint2(E0, E1);
            slot[2] = E1;
        }
        if (lane == 0)   // previous slot's x-neighbour half (previous warp's last slot, or the level's last on wrap)
            reinterpret_cast<uint32_t*>(table_h + pair_prev(e0, T) * 4)[1] = E0;
        tma::fence_shared();
        __syncthreads();
        if (tid == 0) {
            tma::store(p + base, st[s].p, kAdamTile * 4);
            tma::store(m + base, st[s].m, kAdamTile * 4);
            tma::store(v + base, st[s].v, kAdamTile * 4);
            tma::commit();
            // refill the previous iteration's stage once its store has read smem
            if (i >= 1 && i - 1 + kAdamStages < n_local) {
                tma::wait_read<1>();
                issue(i - 1 + kAdamStages);
            }
        }
    }
    if (tid == 0) tma::wait_all();
}

// The dense-gradient grid Adam with two parameters (one x-pair entry) per
// thread and 512 threads: the same bulk-copy ring and tile as k_adam_bulk, twice
// the warps to hide the FP32 division / square-root latency of the update, and
// 8- / 16-byte shared-memory accesses that are bank-conflict free.
constexpr int kAdam2Threads = kAdamTile / 2;
__global__ void __launch_bounds__(kAdam2Threads) k_adam_dense2(float* __restrict__ p, float* __restrict__ m,
                                                               float* __restrict__ v, int64_t* __restrict__ fx,
                                                               uint16_t* __restrict__ table_h, int64_t ntiles,
                                                               AdamK a, int64_t T, int64_t tile0) {
    extern __shared__ __align__(128) uint8_t adam_smem[];
    AdamStage* st = reinterpret_cast<AdamStage*>(adam_smem);
    __shared__ uint64_t full[kAdamStages];
    const int tid = threadIdx.x, lane = tid & 31;
    const int n_local = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x + 1) : 0;
    auto tile_base = [&](int i) { return (tile0 + blockIdx.x + (int64_t)i * gridDim.x) * kAdamTile; };
    auto issue = [&](int i) {
        const int s = i % kAdamStages;
        const int64_t base = tile_base(i);
        tma::bar_expect_tx(&full[s], (uint32_t)sizeof(AdamStage));
        tma::load(st[s].p, p + base, kAdamTile * 4, &full[s]);
        tma::load(st[s].m, m + base, kAdamTile * 4, &full[s]);
        tma::load(st[s].v, v + base, kAdamTile * 4, &full[s]);
        tma::load(st[s].q, fx + base, kAdamTile * 8, &full[s]);
    };
    if (tid == 0) {
        for (int s = 0; s < kAdamStages; ++s) tma::bar_init(&full[s], 1);
        tma::bar_init_fence();
    }
    __syncthreads();
    if (tid == 0)
        for (int i = 0; i < min(kAdamStages, n_local); ++i) issue(i);
    for (int i = 0; i < n_local; ++i) {
        const int s = i % kAdamStages;
        const int64_t base = tile_base(i);
        const int64_t i0 = base + 2 * tid, e0 = i0 / 2;
        tma::bar_wait(&full[s], (uint32_t)(i / kAdamStages) & 1u);
        float2* P2 = reinterpret_cast<float2*>(st[s].p) + tid;
        float2* M2 = reinterpret_cast<float2*>(st[s].m) + tid;
        float2* V2 = reinterpret_cast<float2*>(st[s].v) + tid;
        const longlong2 q = reinterpret_cast<const longlong2*>(st[s].q)[tid];
        if (q.x | q.y) *reinterpret_cast<longlong2*>(fx + i0) = make_longlong2(0, 0);
        float2 P = *P2, M = *M2, V = *V2;
        P.x = adam1(P.x, from_fx(q.x), M.x, V.x, a);
        P.y = adam1(P.y, from_fx(q.y), M.y, V.y, a);
        *P2 = P;
        *M2 = M;
        *V2 = V;
        const uint32_t E0 = (uint32_t)__half_as_ushort(__float2half_rn(P.x)) |
                            ((uint32_t)__half_as_ushort(__float2half_rn(P.y)) << 16);
        const uint32_t nxt = __shfl_down_sync(0xffffffffu, E0, 1);
        uint32_t* slot = reinterpret_cast<uint32_t*>(table_h + e0 * 4);   // x-pair slot e0 = (entry e0 | entry e0 + 1)
        if (lane < 31)
            *reinterpret_cast<uint2*>(slot) = make_uint2(E0, nxt);
        else
            slot[0] = E0;
        if (lane == 0)   // previous slot's x-neighbour half (previous warp's last slot, or the level's last on wrap)
            reinterpret_cast<uint32_t*>(table_h + pair_prev(e0, T) * 4)[1] = E0;
        tma::fence_shared();
        __syncthreads();
        if (tid == 0) {
            tma::store(p + base, st[s].p, kAdamTile * 4);
            tma::store(m + base, st[s].m, kAdamTile * 4);
            tma::store(v + base, st[s].v, kAdamTile * 4);
            tma::commit();
            if (i >= 1 && i - 1 + kAdamStages < n_local) {
                tma::wait_read<1>();
                issue(i - 1 + kAdamStages);
            }
        }
    }
    if (tid == 0) tma::wait_all();
}

__global__ void k_adam_mlp(Net net, float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                           GradSink gs, uint16_t* __restrict__ wpack, AdamK a) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= net.mlp_count) return;
    const int64_t i = net.grid_count + j;
    int64_t* gq = mlp_grad(gs, j);
    const long long q = *gq;
    *gq = 0;
    float mm = m[i], vv = v[i];
    const float pn = adam1(p[i], from_fx_mlp(q), mm, vv, a);
    p[i] = pn;
    m[i] = mm;
    v[i] = vv;
    for (int l = 0; l < net.n_layers; ++l) {
        if (i >= net.woff[l] && i < net.boff[l]) {
            const int64_t e = i - net.woff[l];
            const int K = net.dims[l];
            const uint16_t hv = __half_as_ushort(__float2half_rn(pn));
            wpack[wpack_index(net, l, (int)(e / K), (int)(e % K))] = hv;
            if (wpack_has_t(net)) wpack[wpack_t_index(net, l, (int)(e / K), (int)(e % K))] = hv;
        }
    }
}

__global__ void k_shadow_grid(const float* __restrict__ p, uint16_t* __restrict__ h, int64_t n, int F, int64_t T) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) put_pair(h, i, F, T, __half_as_ushort(__float2half_rn(p[i])));
}

__global__ void k_shadow_wpack(Net net, const float* __restrict__ p, uint16_t* __restrict__ wpack, int64_t total) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= total) return;
    int np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    umma_pads(net.dims, net.n_layers, np, kp);
    // walk layers to find (layer, n, k) of padded slot t in row-major padded order
    int64_t o = t;
    for (int l = 0; l < net.n_layers; ++l) {
        const int64_t sz = (int64_t)np[l] * kp[l];
        if (o < sz) {
            const int n = (int)(o / kp[l]), k = (int)(o % kp[l]);
            float w = 0.0f;
            if (n < net.dims[l + 1] && k < net.dims[l]) w = p[net.woff[l] + (int64_t)n * net.dims[l] + k];
            wpack[wpack_index(net, l, n, k)] = __half_as_ushort(__float2half_rn(w));
            if (wpack_has_t(net)) wpack[wpack_t_index(net, l, n, k)] = __half_as_ushort(__float2half_rn(w));
            return;
        }
        o -= sz;
    }
}

}  // namespace

int64_t wpack_count_of(const nvc_model* m) {
    int np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    umma_pads(m->dims, m->n_layers, np, kp);
    int64_t c = 0;
    for (int i = 0; i < m->n_layers; ++i) c += umma_block_halfs(np[i], kp[i]);
    if (wpack_has_t(net_of(m)))
        for (int i = 0; i < m->n_layers; ++i) c += umma_block_halfs(kp[i], np[i]);
    return c;
}

int train_tc(const nvc_model* m, int64_t grid_count, const int64_t* woff, const int64_t* boff, int64_t mlp_count,
             const float* act0, int64_t b_max, const int64_t* b_dev, int shard, int n_shards, const float* tgt,
             const float* mask, float* dact0, float* part_w, double* part_loss, int nblk, cudaStream_t s);

}  // namespace nvc

using namespace nvc;

static int mlp_smem_bytes(const Net& net) { return tile_layout(net).total * 4 + 64; }

int nvc::nvc_infer_f32(const nvc_model* m, const double* pos, int64_t n, float* out, cudaStream_t s) {
    Net net = net_of(m);
    GridDev g = grid_of(m);
    const int smem = mlp_smem_bytes(net);
    NVC_REQUIRE(smem <= 200 * 1024, "nvc_infer: MLP too wide for the fp32 tile kernel");
    cudaFuncSetAttribute(k_mlp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mlp<false><<<grid1(n, kRows), kThreads, smem, s>>>(g, net, m->params, pos, n, nullptr, 0, 1, nullptr,
                                                          nullptr, out, GradSink{}, nullptr, nullptr);
    return check_launch("k_mlp<infer>");
}


namespace nvc {
namespace {
// grad_from_ctx (hashgrid.py:140-151): per level, np.add.at(grad[l], idx, w * g)
// in float32, i.e. every table entry is the sequential float sum of its
// contributions in (row, corner) order.  One CTA per level sorts the chunk's
// (entry, order) keys in shared memory (bitonic) and one thread per entry
// adds its run in order onto the entry's current value, so chunks applied in
// stream order reproduce the sequential sum bit for bit.
constexpr int kScatterChunk = 2048;            // rows per launch: 16384 keys, 128 KB
__global__ void __launch_bounds__(1024) k_grid_scatter(const int32_t* __restrict__ idx, const double* __restrict__ w,
                                                       const float* __restrict__ up, int64_t r0, int nr, int L, int F,
                                                       int64_t T, float* __restrict__ grad) {
    extern __shared__ unsigned long long keys[];
    const int l = blockIdx.x;
    const int n = nr * 8;
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = threadIdx.x; i < np2; i += blockDim.x) {
        if (i < n) {
            const int64_t r = r0 + i / 8;
            const uint32_t e = (uint32_t)idx[(r * L + l) * 8 + (i & 7)];
            keys[i] = ((unsigned long long)e << 32) | (unsigned)i;
        } else {
            keys[i] = ~0ull;
        }
    }
    __syncthreads();
    for (int k = 2; k <= np2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np2; i += blockDim.x) {
                const int x = i ^ j;
                if (x > i) {
                    const unsigned long long a = keys[i], b = keys[x];
                    if (((i & k) == 0) == (a > b)) {
                        keys[i] = b;
                        keys[x] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t e = (uint32_t)(keys[i] >> 32);
        if (i > 0 && (uint32_t)(keys[i - 1] >> 32) == e) continue;     // not the head of its run
        float* g = grad + ((int64_t)l * T + e) * F;
        for (int f = 0; f < F; ++f) {
            float acc = g[f];
            for (int q = i; q < n && (uint32_t)(keys[q] >> 32) == e; ++q) {
                const int o = (int)(keys[q] & 0xffffffffu);
                const int64_t r = r0 + o / 8;
                const double wc = w[(r * L + l) * 8 + (o & 7)];
                acc = __fadd_rn(acc, (float)(wc * (double)up[r * (int64_t)(L * F) + l * F + f]));
            }
            g[f] = acc;
        }
    }
}
}  // namespace
}  // namespace nvc

extern "C" {

const char* nvc_last_error(void) { return g_err; }
int32_t nvc_abi_version(void) { return NVC_ABI_VERSION; }
int64_t nvc_wpack_count(const nvc_model* m) { return m ? wpack_count_of(m) : 0; }

int64_t nvc_train_workspace_bytes(const nvc_model* m, int64_t b) {
    if (!m) return 0;
    Net net = net_of(m);
    const int64_t nblk = b / kRows + 2;
    return nblk * (net.mlp_count * 4 + 8) + 2 * (nblk * kRows * net.dims[0] * 4 + 256) + 512;
}

int nvc_refresh_shadow(const nvc_model* m, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(m->table_h && m->wpack, "nvc_refresh_shadow: shadow buffers not bound");
    Net net = net_of(m);
    cudaStream_t s = (cudaStream_t)stream;
    k_shadow_grid<<<grid1(net.grid_count, 256), 256, 0, s>>>(m->params, m->table_h, net.grid_count, m->features,
                                                             m->table_size);
    const int64_t wc = wpack_count_of(m);
    k_shadow_wpack<<<grid1(wc, 256), 256, 0, s>>>(net, m->params, m->wpack, wc);
    return check_launch("refresh_shadow");
}

int nvc_grid_scatter(int32_t levels, int32_t features, int64_t table_size, const int32_t* idx, const double* w,
                     const float* upstream, int64_t b, float* grad, void* stream) {
    NVC_REQUIRE(idx && w && upstream && grad, "nvc_grid_scatter: null argument");
    NVC_REQUIRE(levels > 0 && features > 0 && table_size > 0 && table_size <= (1ll << 32),
                "nvc_grid_scatter: bad grid shape");
    const int smem = kScatterChunk * 8 * 8;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_grid_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    for (int64_t r0 = 0; r0 < b; r0 += kScatterChunk) {
        const int nr = (int)std::min<int64_t>(kScatterChunk, b - r0);
        k_grid_scatter<<<levels, 1024, smem, (cudaStream_t)stream>>>(idx, w, upstream, r0, nr, levels, features,
                                                                     table_size, grad);
        const int rc = check_launch("k_grid_scatter");
        if (rc != NVC_OK) return rc;
    }
    return NVC_OK;
}

int nvc_encode(const nvc_model* m, const double* pos, int64_t n, float* feats, int32_t* idx_out, double* w_out,
               void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    if (n <= 0) return NVC_OK;
    NVC_REQUIRE(pos && feats, "nvc_encode: null argument");
    GridDev g = grid_of(m);
    k_encode<<<grid1(n * g.L, 128), 128, 0, (cudaStream_t)stream>>>(g, m->params, pos, n, feats, idx_out, w_out);
    return check_launch("k_encode");
}

int nvc_train_grads(const nvc_model* m, const double* pos, const float* tgt, const float* mask, int64_t b_max,
                    const int64_t* b_dev, int32_t shard, int32_t n_shards, void* ws, double* loss_out,
                    void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(pos && tgt && ws && (m->grad_fx || m->grad_c), "nvc_train_grads: null argument");
    NVC_REQUIRE(!m->grad_c || (m->touch_bits && m->touch_off), "nvc_train_grads: compact mode needs the touch index");
    NVC_REQUIRE(!m->grad_c || m->grad_c_entries >= std::min<int64_t>(b_max * m->levels * 8,
                                                                     (int64_t)m->levels * m->table_size),
                "nvc_train_grads: grad_c_entries below nvc_exchange_max_entries(b_max)");
    NVC_REQUIRE(n_shards >= 1 && shard >= 0 && shard < n_shards, "nvc_train_grads: bad shard");
    NVC_REQUIRE(m->out_sigmoid == 1 || m->out_sigmoid == 0, "bad output activation");
    if (b_max <= 0) return NVC_OK;
    Net net = net_of(m);
    GridDev g = grid_of(m);
    const int64_t rows_max = b_max / n_shards + 1;
    const int nblk = grid1(rows_max, kRows);
    float* part_w = (float*)ws;
    double* part_loss = (double*)((char*)ws + ((int64_t)nblk * net.mlp_count * 4 + 255) / 256 * 256);
    cudaStream_t s = (cudaStream_t)stream;
    bool split = g.F <= 8 && getenv("NVC_TRAIN_FUSED") == nullptr;
    for (int i = 0; i <= net.n_layers; ++i) split = split && (net.dims[i] % 4 == 0);
    const bool wg = t3_layout(net).total * 4 + 64 > 200 * 1024;   // too wide for every W in smem (C4): W staged per layer
    T3Layout tl3 = t3_layout(net, !wg);
    tl3.rbits = getenv("NVC_T3_BITS") ? atoi(getenv("NVC_T3_BITS")) : 0;
    if (getenv("NVC_T3_WHAT")) tl3.rwhat = atoi(getenv("NVC_T3_WHAT"));
    const int smem3 = tl3.total * 4 + 64;
    int nblk_red = nblk;   // partial sets k_reduce_parts sums (one per training block)
    bool reduced = false;  // launched on the side stream already
    if (split && smem3 <= 200 * 1024) {
        char* p2 = (char*)part_loss + ((int64_t)nblk * 8 + 255) / 256 * 256;
        float* act0 = (float*)p2;
        float* dact0 = (float*)(p2 + ((int64_t)nblk * kRows * net.dims[0] * 4 + 255) / 256 * 256);
        k_tr_encode<<<grid1(rows_max * g.L, 128), 128, 0, s>>>(g, m->params, pos, b_max, b_dev, shard, n_shards, act0);
        rc = check_launch("k_tr_encode");
        if (rc) return rc;
        const bool tc = getenv("NVC_TRAIN_TC") != nullptr &&
                        train_tc(m, net.grid_count, net.woff, net.boff, net.mlp_count, act0, b_max, b_dev, shard,
                                 n_shards, tgt, mask, dact0, part_w, part_loss, grid1(rows_max, 128), s) == 0;
        if (tc) {
            nblk_red = 2 * grid1(rows_max, 128);   // a hi and a lo partial set per 128-row tile
        } else if (wg) {
            cudaFuncSetAttribute(k_train3<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
            k_train3<true><<<nblk, kThreads, smem3, s>>>(net, tl3, m->params, act0, b_max, b_dev, shard, n_shards,
                                                         tgt, mask, dact0, part_w, part_loss);
        } else {
            cudaFuncSetAttribute(k_train3<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
            k_train3<false><<<nblk, kThreads, smem3, s>>>(net, tl3, m->params, act0, b_max, b_dev, shard, n_shards,
                                                          tgt, mask, dact0, part_w, part_loss);
        }
        rc = check_launch("k_train3");
        if (rc) return rc;
        if (SideStream* ss = side_stream()) {   // the MLP partial reduce beside the grid scatter
            cudaEventRecord(ss->fork, s);
            cudaStreamWaitEvent(ss->s, ss->fork, 0);
            k_reduce_parts<<<grid1(net.mlp_count, 32), 256, 0, ss->s>>>(part_w, part_loss, nblk_red, net.mlp_count,
                                                                        net.grid_count, sink_of(m), loss_out, b_max,
                                                                        b_dev);
            cudaEventRecord(ss->join, ss->s);
            reduced = true;
            k_tr_scatter<<<grid1(rows_max * g.L, 128), 128, 0, s>>>(g, pos, b_max, b_dev, shard, n_shards, dact0,
                                                                     sink_of(m));
            cudaStreamWaitEvent(s, ss->join, 0);
        } else {
            k_tr_scatter<<<grid1(rows_max * g.L, 128), 128, 0, s>>>(g, pos, b_max, b_dev, shard, n_shards, dact0,
                                                                     sink_of(m));
        }
    } else {
        const int smem = mlp_smem_bytes(net);
        NVC_REQUIRE(smem <= 200 * 1024, "nvc_train_grads: MLP too wide for the fp32 tile kernel");
        cudaFuncSetAttribute(k_mlp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_mlp<true><<<nblk, kThreads, smem, s>>>(g, net, m->params, pos, b_max, b_dev, shard, n_shards, tgt, mask,
                                                  nullptr, sink_of(m), part_w, part_loss);
    }
    rc = check_launch("nvc_train_grads");
    if (rc) return rc;
    if (!reduced)
        k_reduce_parts<<<grid1(net.mlp_count, 32), 256, 0, s>>>(part_w, part_loss, nblk_red, net.mlp_count,
                                                                 net.grid_count, sink_of(m), loss_out, b_max, b_dev);
    return check_launch("k_reduce_parts");
}

// ---- compact data-parallel gradient exchange ----
static int64_t touch_words(const nvc_model* m) { return ((int64_t)m->levels * m->table_size + 31) / 32; }

int64_t nvc_exchange_max_entries(const nvc_model* m, int64_t b) {
    if (!m) return 0;
    const int64_t e = (int64_t)m->levels * m->table_size;
    const int64_t bound = b * m->levels * 8;
    return bound < e ? bound : e;
}

int64_t nvc_exchange_workspace_bytes(const nvc_model* m) {
    if (!m) return 0;
    const int64_t words = touch_words(m);
    return (words * 4 + 255) / 256 * 256 + ((words + 1023) / 1024 * 4 + 255) / 256 * 256;
}

int64_t nvc_exchange_buffer_len(const nvc_model* m, int64_t max_entries) {
    if (!m) return 0;
    Net net = net_of(m);
    return max_entries * m->features + net.mlp_count;
}

int64_t nvc_touch_words(const nvc_model* m) { return m ? touch_words(m) : 0; }
int64_t nvc_touch_off_len(const nvc_model* m) { return m ? touch_words(m) + (touch_words(m) + 1023) / 1024 : 0; }

int nvc_train_index(const nvc_model* m, const double* pos, int64_t b_max, const int64_t* b_dev, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(pos && m->touch_bits && m->touch_off, "nvc_train_index: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    GridDev g = grid_of(m);
    const int64_t words = touch_words(m);
    const int n_chunks = (int)((words + 1023) / 1024);
    int* chunk = m->touch_off + words;
    cudaMemsetAsync(m->touch_bits, 0, words * 4, s);
    if (b_max > 0)
        k_touch_mark<<<grid1(b_max * g.L, 128), 128, 0, s>>>(g, pos, b_max, b_dev, m->touch_bits);
    k_touch_count<<<n_chunks, 256, 0, s>>>(m->touch_bits, words, chunk);
    k_touch_scan<<<1, 1024, 0, s>>>(chunk, n_chunks, nullptr);
    k_touch_offsets<<<n_chunks, 1024, 0, s>>>(m->touch_bits, words, chunk, m->touch_off);
    return check_launch("nvc_train_index");
}

int nvc_exchange_index(const nvc_model* m, const double* pos, int64_t b_max, const int64_t* b_dev, void* ws,
                       int32_t* idx, int64_t* count, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(pos && ws && idx && count, "nvc_exchange_index: null argument");
    cudaStream_t s = (cudaStream_t)stream;
    GridDev g = grid_of(m);
    const int64_t words = touch_words(m);
    const int n_chunks = (int)((words + 1023) / 1024);
    uint32_t* bits = (uint32_t*)ws;
    int* chunk = (int*)((char*)ws + (words * 4 + 255) / 256 * 256);
    cudaMemsetAsync(bits, 0, words * 4, s);
    if (b_max > 0)
        k_touch_mark<<<grid1(b_max * g.L, 128), 128, 0, s>>>(g, pos, b_max, b_dev, bits);
    k_touch_count<<<n_chunks, 256, 0, s>>>(bits, words, chunk);
    k_touch_scan<<<1, 1024, 0, s>>>(chunk, n_chunks, count);
    k_touch_emit<<<n_chunks, 1024, 0, s>>>(bits, words, chunk, idx);
    return check_launch("nvc_exchange_index");
}

int nvc_exchange_pack(const nvc_model* m, const int32_t* idx, const int64_t* count, int64_t max_entries,
                      int64_t* buf, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(idx && count && buf && m->grad_fx, "nvc_exchange_pack: null argument");
    Net net = net_of(m);
    const int64_t n = max_entries * m->features + net.mlp_count;
    k_grad_pack<<<grid1(n, 256), 256, 0, (cudaStream_t)stream>>>(m->grad_fx, idx, count, max_entries, m->features,
                                                                 net.grid_count, net.mlp_count, buf);
    return check_launch("k_grad_pack");
}

int nvc_exchange_unpack(const nvc_model* m, const int32_t* idx, const int64_t* count, int64_t max_entries,
                        const int64_t* buf, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(idx && count && buf && m->grad_fx, "nvc_exchange_unpack: null argument");
    Net net = net_of(m);
    const int64_t n = max_entries * m->features + net.mlp_count;
    k_grad_unpack<<<grid1(n, 256), 256, 0, (cudaStream_t)stream>>>(m->grad_fx, idx, count, max_entries, m->features,
                                                                   net.grid_count, net.mlp_count, buf);
    return check_launch("k_grad_unpack");
}

int nvc_adam_step(const nvc_model* m, int64_t t, double lr, void* stream) {
    return nvc_adam_step_shard(m, t, lr, 0, 1, stream);
}

int nvc_adam_shard_range(const nvc_model* m, int32_t shard, int32_t n_shards, int64_t* lo, int64_t* hi) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(lo && hi && n_shards >= 1 && shard >= 0 && shard < n_shards, "nvc_adam_shard_range: bad shard");
    const Net net = net_of(m);
    NVC_REQUIRE(m->features == 2 && m->table_size % 64 == 0 && net.grid_count % kAdamTile == 0,
                "nvc_adam_shard_range: the sharded optimizer needs F == 2 and whole Adam tiles");
    const int64_t ntiles = net.grid_count / kAdamTile;
    *lo = ntiles * shard / n_shards * kAdamTile;
    *hi = ntiles * (shard + 1) / n_shards * kAdamTile;
    return NVC_OK;
}

int nvc_adam_step_shard(const nvc_model* m, int64_t t, double lr, int32_t shard, int32_t n_shards, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(t >= 1, "nvc_adam_step: t must be >= 1");
    NVC_REQUIRE(n_shards >= 1 && shard >= 0 && shard < n_shards, "nvc_adam_step_shard: bad shard");
    NVC_REQUIRE(m->adam_m && m->adam_v && (m->grad_fx || m->grad_c) && m->table_h && m->wpack,
                "nvc_adam_step: state not bound");
    Net net = net_of(m);
    AdamK a;
    a.b1 = (float)0.9;
    a.c1 = (float)(1.0 - 0.9);
    a.b2 = (float)0.999;
    a.c2 = (float)(1.0 - 0.999);
    a.b1c = (float)(1.0 - pow(0.9, (double)t));
    a.b2c = (float)(1.0 - pow(0.999, (double)t));
    a.lr = (float)lr;
    a.eps = (float)1e-8;
    a.inv_b1c = 1.0 / (double)a.b1c;
    a.inv_b2c = 1.0 / (double)a.b2c;
    cudaStream_t s = (cudaStream_t)stream;
    // the MLP Adam (disjoint parameters) beside the grid Adam, on the side stream
    SideStream* ss = side_stream();
    if (ss) {
        cudaEventRecord(ss->fork, s);
        cudaStreamWaitEvent(ss->s, ss->fork, 0);
        k_adam_mlp<<<grid1(net.mlp_count, 256), 256, 0, ss->s>>>(net, m->params, m->adam_m, m->adam_v, sink_of(m),
                                                                 m->wpack, a);
        cudaEventRecord(ss->join, ss->s);
    }
    const bool bulk = m->features == 2 && m->table_size % 64 == 0 && net.grid_count % kAdamTile == 0;
    NVC_REQUIRE(n_shards == 1 || (bulk && !m->grad_c),
                "nvc_adam_step_shard: the sharded optimizer needs F == 2, whole Adam tiles and dense gradients");
    if (bulk && (n_shards > 1 || !getenv("NVC_ADAM_FLAT"))) {
        const int smem = kAdamStages * (int)sizeof(AdamStage);
        cudaFuncSetAttribute(k_adam_bulk<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_adam_bulk<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int sms = num_sms();
        const int64_t all_tiles = net.grid_count / kAdamTile;
        const int64_t tile0 = all_tiles * shard / n_shards, ntiles = all_tiles * (shard + 1) / n_shards - tile0;
        if (n_shards > 1) {   // the other shards' (allreduced) gradients are consumed by their owners
            if (tile0 > 0) cudaMemsetAsync(m->grad_fx, 0, (size_t)(tile0 * kAdamTile) * 8, s);
            const int64_t end = (tile0 + ntiles) * kAdamTile;
            if (end < net.grid_count)
                cudaMemsetAsync(m->grad_fx + end, 0, (size_t)(net.grid_count - end) * 8, s);
        }
        // CTAs per SM (default 2: 2 x 61 KB smem rings still stream at HBM rate and
        // leave each SM room for the previous frame's NLS blocks running beside it)
        const char* ge = getenv("NVC_ADAM_GRID");
        const int grid = (int)std::min<int64_t>(ntiles, (ge ? atoi(ge) : 2) * (int64_t)sms);
        if (ntiles > 0 && !m->grad_c && !getenv("NVC_ADAM_BULK4")) {   // default: 512 threads x 2 parameters
            cudaFuncSetAttribute(k_adam_dense2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_adam_dense2<<<grid, kAdam2Threads, smem, s>>>(m->params, m->adam_m, m->adam_v, m->grad_fx, m->table_h,
                                                            ntiles, a, m->table_size, tile0);
        } else if (ntiles > 0) {
            if (m->grad_c)
                k_adam_bulk<true><<<grid, kAdamThreads, smem, s>>>(m->params, m->adam_m, m->adam_v, sink_of(m),
                                                                   m->table_h, ntiles, a, m->table_size, tile0);
            else
                k_adam_bulk<false><<<grid, kAdamThreads, smem, s>>>(m->params, m->adam_m, m->adam_v, sink_of(m),
                                                                    m->table_h, ntiles, a, m->table_size, tile0);
        }
    } else {
        k_adam_flat<<<grid1(net.grid_count, 256), 256, 0, s>>>(m->params, m->adam_m, m->adam_v, sink_of(m),
                                                               m->table_h, net.grid_count, m->features, a,
                                                               m->table_size);
    }
    rc = check_launch("k_adam_grid");
    if (rc) return rc;
    if (ss) {
        cudaStreamWaitEvent(s, ss->join, 0);
    } else {
        k_adam_mlp<<<grid1(net.mlp_count, 256), 256, 0, s>>>(net, m->params, m->adam_m, m->adam_v, sink_of(m),
                                                             m->wpack, a);
    }
    return check_launch("k_adam_mlp");
}

}  // extern "C"
