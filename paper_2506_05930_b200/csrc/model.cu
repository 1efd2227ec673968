// model.cu -- FP32 encoder / MLP (parity path), training gradients with the
// fixed-point hash-grid scatter, fused dense Adam, and the fp16 shadow refresh
// (SURVEY table K: K1 parity mode, K3, K4).
//
// Reference routines (under /root/reference/pkg/src/viscache):
//   encode_batch hashgrid.py:117-131, grad_from_ctx :140-151,
//   forward mlp.py:110-140, l2_loss :143-149, backward_l2 :152-183,
//   adam_step :203-218, VisibilityCache.train_step cache.py:60-73.
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace nvc {

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

constexpr int kRows = 32;      // rows per block in the SIMT MLP kernels
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
                                                 float* __restrict__ out, int64_t* __restrict__ grad_fx,
                                                 uint16_t* __restrict__ touched, uint16_t epoch,
                                                 float* __restrict__ part_w, double* __restrict__ part_loss) {
    extern __shared__ float sm[];
    const TileLayout tl = tile_layout(net);
    const int64_t b = b_dev ? *b_dev : b_max;
    const int64_t lo = b * shard / n_shards, hi = b * (shard + 1) / n_shards;
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
        int64_t* gl = grad_fx + (int64_t)l * g.T * g.F;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t idx = corner_index(g, l, c0, (c >> 2) & 1, (c >> 1) & 1, c & 1);
            const double w = corner_weight(f, c);
            for (int k = 0; k < g.F; ++k) {
                const float contrib = (float)__dmul_rn(w, (double)up[k]);   // (w * g).astype(f32)
                red_add_fx(gl + (int64_t)idx * g.F + k, to_fx((double)contrib));
            }
            touched[(int64_t)l * g.T + idx] = epoch;
        }
    }
}

// ---------------------------------------------------------------------------
// Register-tiled SIMT training step (all widths multiples of 4, weights in
// smem as W and W^T).  Same maths and row partition as k_mlp<true>, ~10x less
// time: forward 2x4 tiles over Wt, grad-W 4x4 tiles over (dz, act), grad-act
// 2x4 tiles over W, all operands in shared memory.
// ---------------------------------------------------------------------------
struct T2Layout {
    int w[NVC_MAX_LAYERS], wt[NVC_MAX_LAYERS];   // float offsets of W_l [N][K] and W_l^T [K][N]
    int act[NVC_MAX_LAYERS + 1];                 // act_l [kRows][D_l]
    int dz0, dz1;                                // two [kRows][Dmax] buffers
    int total;
};

__host__ __device__ inline T2Layout t2_layout(const Net& net) {
    T2Layout t;
    int o = 0, dmax = 0;
    for (int l = 0; l < net.n_layers; ++l) {
        const int sz = net.dims[l] * net.dims[l + 1];
        t.w[l] = o;
        o += sz;
        t.wt[l] = o;
        o += sz;
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

__global__ void __launch_bounds__(kThreads) k_train2(GridDev g, Net net, const float* __restrict__ params,
                                                    const double* __restrict__ pos, int64_t b_max,
                                                    const int64_t* __restrict__ b_dev, int shard, int n_shards,
                                                    const float* __restrict__ tgt, const float* __restrict__ mask,
                                                    int64_t* __restrict__ grad_fx, uint16_t* __restrict__ touched,
                                                    uint16_t epoch, float* __restrict__ part_w,
                                                    double* __restrict__ part_loss) {
    extern __shared__ float sm[];
    const T2Layout tl = t2_layout(net);
    const int tid = threadIdx.x;
    const int64_t b = b_dev ? *b_dev : b_max;
    const int64_t lo = b * shard / n_shards, hi = b * (shard + 1) / n_shards;
    const int64_t row0 = lo + (int64_t)blockIdx.x * kRows;
    const int nr = (int)max((int64_t)0, min((int64_t)kRows, hi - row0));
    const int D0 = net.dims[0];
    const int K = net.dims[net.n_layers];

    // ---- weights -> smem (W and W^T), encode rows -> act0 ----
    for (int l = 0; l < net.n_layers; ++l) {
        const int N = net.dims[l + 1], Ki = net.dims[l];
        const float* W = params + net.woff[l];
        for (int e = tid; e < N * Ki; e += blockDim.x) {
            const float w = __ldg(W + e);
            const int n = e / Ki, k = e - n * Ki;
            sm[tl.w[l] + e] = w;
            sm[tl.wt[l] + k * N + n] = w;
        }
    }
    for (int e = tid; e < kRows * g.L; e += blockDim.x) {
        const int r = e / g.L, l = e - r * g.L;
        float* dst = sm + tl.act[0] + r * D0 + l * g.F;
        if (r < nr) {
            const int64_t i = row0 + r;
            const double pp[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
            double q[3];
            normalize(g, pp, q);
            encode_level_f32(g, params, q, l, dst, nullptr, nullptr);
        } else {
            for (int k = 0; k < g.F; ++k) dst[k] = 0.0f;
        }
    }
    __syncthreads();

    // ---- forward: z = act W^T + b, 2x4 register tiles ----
    for (int l = 0; l < net.n_layers; ++l) {
        const int Ki = net.dims[l], N = net.dims[l + 1];
        const float* A = sm + tl.act[l];
        const float* Wt = sm + tl.wt[l];
        float* out = sm + tl.act[l + 1];
        const bool last = l == net.n_layers - 1;
        const int ng = N / 4;
        for (int t = tid; t < (kRows / 2) * ng; t += blockDim.x) {
            const int r0 = (t / ng) * 2, n0 = (t % ng) * 4;
            float acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
            for (int k = 0; k < Ki; ++k) {
                const float4 w = *reinterpret_cast<const float4*>(Wt + k * N + n0);
                const float a0 = A[r0 * Ki + k], a1 = A[(r0 + 1) * Ki + k];
                acc[0][0] = fmaf(a0, w.x, acc[0][0]);
                acc[0][1] = fmaf(a0, w.y, acc[0][1]);
                acc[0][2] = fmaf(a0, w.z, acc[0][2]);
                acc[0][3] = fmaf(a0, w.w, acc[0][3]);
                acc[1][0] = fmaf(a1, w.x, acc[1][0]);
                acc[1][1] = fmaf(a1, w.y, acc[1][1]);
                acc[1][2] = fmaf(a1, w.z, acc[1][2]);
                acc[1][3] = fmaf(a1, w.w, acc[1][3]);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float z = acc[i][j] + __ldg(params + net.boff[l] + n0 + j);
                    out[(r0 + i) * N + n0 + j] = (last && net.out_sigmoid) ? sigmoid_ref(z) : leaky(z, net.alpha);
                }
        }
        __syncthreads();
    }

    // ---- loss + output delta (mlp.py:143-149, 160-168) ----
    float* dz = sm + tl.dz0;
    float* dzn = sm + tl.dz1;
    const float bk = (float)(b * K);
    double lsum = 0.0;
    for (int e = tid; e < kRows * K; e += blockDim.x) {
        const int r = e / K;
        float d = 0.0f;
        if (r < nr) {
            const int64_t li = (row0 - lo) * K + e;
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
        dz[e] = d;
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
        const int Ki = net.dims[l], N = net.dims[l + 1];
        const float* A = sm + tl.act[l];
        // grad W[n][k] = sum_r dz[r][n] A[r][k]   (4x4 tiles)
        float* gw = part + (net.woff[l] - net.grid_count);
        const int kg = Ki / 4;
        for (int t = tid; t < (N / 4) * kg; t += blockDim.x) {
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
        for (int n = tid; n < N; n += blockDim.x) {
            float acc = 0.0f;
            for (int r = 0; r < kRows; ++r) acc += dz[r * N + n];
            gb[n] = acc;
        }
        // grad act[r][k] = sum_n dz[r][n] W[n][k], through leaky'(z_{l-1}) (2x4 tiles)
        const float* W = sm + tl.w[l];
        for (int t = tid; t < (kRows / 2) * kg; t += blockDim.x) {
            const int r0 = (t / kg) * 2, k0 = (t % kg) * 4;
            float acc[2][4] = {{0, 0, 0, 0}, {0, 0, 0, 0}};
            for (int n = 0; n < N; ++n) {
                const float4 w = *reinterpret_cast<const float4*>(W + n * Ki + k0);
                const float d0 = dz[r0 * N + n], d1 = dz[(r0 + 1) * N + n];
                acc[0][0] = fmaf(d0, w.x, acc[0][0]);
                acc[0][1] = fmaf(d0, w.y, acc[0][1]);
                acc[0][2] = fmaf(d0, w.z, acc[0][2]);
                acc[0][3] = fmaf(d0, w.w, acc[0][3]);
                acc[1][0] = fmaf(d1, w.x, acc[1][0]);
                acc[1][1] = fmaf(d1, w.y, acc[1][1]);
                acc[1][2] = fmaf(d1, w.z, acc[1][2]);
                acc[1][3] = fmaf(d1, w.w, acc[1][3]);
            }
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    float v = acc[i][j];
                    if (l > 0 && !(A[(r0 + i) * Ki + k0 + j] >= 0.0f)) v = __fmul_rn(v, net.alpha);
                    dzn[(r0 + i) * Ki + k0 + j] = v;
                }
        }
        __syncthreads();
        float* t = dz;
        dz = dzn;
        dzn = t;
    }

    // ---- hash-grid scatter (hashgrid.py:140-151), fixed point ----
    for (int e = tid; e < nr * g.L; e += blockDim.x) {
        const int r = e / g.L, l = e - r * g.L;
        const int64_t i = row0 + r;
        const double pp[3] = {pos[3 * i], pos[3 * i + 1], pos[3 * i + 2]};
        double q[3];
        normalize(g, pp, q);
        int c0[3];
        double f[3];
        cell(g.res[l], q, c0, f);
        const float* up = dz + r * D0 + l * g.F;
        int64_t* gl = grad_fx + (int64_t)l * g.T * g.F;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const uint32_t idx = corner_index(g, l, c0, (c >> 2) & 1, (c >> 1) & 1, c & 1);
            const double w = corner_weight(f, c);
            for (int k = 0; k < g.F; ++k) {
                const float contrib = (float)__dmul_rn(w, (double)up[k]);
                red_add_fx(gl + (int64_t)idx * g.F + k, to_fx((double)contrib));
            }
            touched[(int64_t)l * g.T + idx] = epoch;
        }
    }
}

// fixed-order reduction of the per-block MLP partials and loss partials:
// block = 32 parameters x 8 warps; warp w sums partial blocks w, w+8, ...
// in order, then the 8 warp sums are combined in warp order (deterministic).
__global__ void __launch_bounds__(256) k_reduce_parts(const float* __restrict__ part_w,
                                                      const double* __restrict__ part_loss, int nblk,
                                                      int64_t mlp_count, int64_t grid_count,
                                                      int64_t* __restrict__ grad_fx, double* __restrict__ loss_out) {
    __shared__ double s_acc[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    double acc = 0.0;
    if (j < mlp_count)
        for (int b = w; b < nblk; b += 8) acc += (double)__ldg(part_w + (int64_t)b * mlp_count + j);
    s_acc[w][lane] = acc;
    __syncthreads();
    if (w == 0 && j < mlp_count) {
        double t = 0.0;
        for (int i = 0; i < 8; ++i) t += s_acc[i][lane];
        grad_fx[grid_count + j] += to_fx(t);
    }
    if (blockIdx.x == 0 && w == 1 && loss_out) {
        double t = 0.0;
        for (int b = lane; b < nblk; b += 32) t += part_loss[b];
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) *loss_out = t;
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
// error cannot change the float rounding; the variable quotient uses a
// binary64 division (double rounding is innocuous for p' >= 2p + 2).
__device__ __forceinline__ float adam1(float p, float g, float& m, float& v, const AdamK& a) {
    m = __fadd_rn(__fmul_rn(m, a.b1), __fmul_rn(a.c1, g));
    v = __fadd_rn(__fmul_rn(v, a.b2), __fmul_rn(__fmul_rn(a.c2, g), g));
    const float mh = (float)__dmul_rn((double)m, a.inv_b1c);
    const float vh = (float)__dmul_rn((double)v, a.inv_b2c);
    const float num = __fmul_rn(a.lr, mh);
    const float den = __fadd_rn(__fsqrt_rn(vh), a.eps);
    return __fsub_rn(p, (float)__ddiv_rn((double)num, (double)den));
}

// wpack offset (halfs) of W_i[n][k] in the tcgen05 swizzled K-major layout
__host__ __device__ inline int64_t wpack_index(const Net& net, int i, int n, int k) {
    int np[NVC_MAX_LAYERS], kp[NVC_MAX_LAYERS];
    umma_pads(net.dims, net.n_layers, np, kp);
    int64_t o = 0;
    for (int j = 0; j < i; ++j) o += umma_block_halfs(np[j], kp[j]);
    return o + umma_off(n, k, np[i], kp[i]) / 2;
}

// grid part: 8 params per thread, all loads issued before any math; the
// gradient of an entry is read (and zeroed) only when its epoch matches.
__device__ __forceinline__ float4 ld_stream(const float* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ void st_stream(float* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ void put_pair(uint16_t* t2, int64_t i, int F, int64_t T, uint16_t h) {
    const int64_t e = i / F, f = i - e * F;
    t2[e * 2 * F + f] = h;                               // own slot, low half
    t2[pair_prev(e, T) * 2 * F + F + f] = h;             // previous slot's x-neighbour half
}

__global__ void __launch_bounds__(256) k_adam_grid(float* __restrict__ p, float* __restrict__ m,
                                                   float* __restrict__ v, int64_t* __restrict__ fx,
                                                   const uint16_t* __restrict__ touched,
                                                   uint16_t* __restrict__ table_h, int64_t n, int F,
                                                   uint16_t epoch, int dense, AdamK a, int64_t T) {
    const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8;
    if (i0 >= n) return;
    if (i0 + 8 <= n) {
        float4 P[2], M[2], V[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            P[h] = ld_stream(p + i0 + 4 * h);
            M[h] = ld_stream(m + i0 + 4 * h);
            V[h] = ld_stream(v + i0 + 4 * h);
        }
        uint16_t tv[8];
        if (!dense) {
            if (F == 2) {
                const uint2 t4 = __ldg(reinterpret_cast<const uint2*>(touched + i0 / 2));
                tv[0] = tv[1] = (uint16_t)(t4.x & 0xffff);
                tv[2] = tv[3] = (uint16_t)(t4.x >> 16);
                tv[4] = tv[5] = (uint16_t)(t4.y & 0xffff);
                tv[6] = tv[7] = (uint16_t)(t4.y >> 16);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) tv[j] = __ldg(touched + (i0 + j) / F);
            }
        }
        float G[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            G[j] = 0.0f;
            if (dense || tv[j] == epoch) {
                const long long q = fx[i0 + j];
                if (q) {
                    G[j] = from_fx(q);
                    fx[i0 + j] = 0;
                }
            }
        }
        __align__(16) __half hv[8];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float* Pp = &P[h].x;
            float* Mp = &M[h].x;
            float* Vp = &V[h].x;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                Pp[j] = adam1(Pp[j], G[4 * h + j], Mp[j], Vp[j], a);
                hv[4 * h + j] = __float2half_rn(Pp[j]);
            }
            st_stream(p + i0 + 4 * h, P[h]);
            st_stream(m + i0 + 4 * h, M[h]);
            st_stream(v + i0 + 4 * h, V[h]);
        }
        if (F == 2) {   // 4 entries: own slots (4 x 4 B) + previous slots' neighbour halves
            const int64_t e0 = i0 / 2;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t w = (uint32_t)__half_as_ushort(hv[2 * j]) | ((uint32_t)__half_as_ushort(hv[2 * j + 1]) << 16);
                const int64_t e = e0 + j;
                *reinterpret_cast<uint32_t*>(table_h + e * 4) = w;
                *reinterpret_cast<uint32_t*>(table_h + pair_prev(e, T) * 4 + 2) = w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) put_pair(table_h, i0 + j, F, T, __half_as_ushort(hv[j]));
        }
    } else {
        for (int64_t i = i0; i < n; ++i) {
            const bool hot = dense || touched[i / F] == epoch;
            float g = 0.0f;
            if (hot && fx[i]) {
                g = from_fx(fx[i]);
                fx[i] = 0;
            }
            float mm = m[i], vv = v[i];
            p[i] = adam1(p[i], g, mm, vv, a);
            m[i] = mm;
            v[i] = vv;
            put_pair(table_h, i, F, T, __half_as_ushort(__float2half_rn(p[i])));
        }
    }
}

__global__ void k_adam_mlp(Net net, float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                           int64_t* __restrict__ fx, uint16_t* __restrict__ wpack, AdamK a) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= net.mlp_count) return;
    const int64_t i = net.grid_count + j;
    const long long q = fx[i];
    fx[i] = 0;
    float mm = m[i], vv = v[i];
    const float pn = adam1(p[i], from_fx(q), mm, vv, a);
    p[i] = pn;
    m[i] = mm;
    v[i] = vv;
    for (int l = 0; l < net.n_layers; ++l) {
        if (i >= net.woff[l] && i < net.boff[l]) {
            const int64_t e = i - net.woff[l];
            const int K = net.dims[l];
            wpack[wpack_index(net, l, (int)(e / K), (int)(e % K))] = __half_as_ushort(__float2half_rn(pn));
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
    return c;
}

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
                                                          nullptr, out, nullptr, nullptr, 0, nullptr, nullptr);
    return check_launch("k_mlp<infer>");
}


extern "C" {

const char* nvc_last_error(void) { return g_err; }
int32_t nvc_abi_version(void) { return NVC_ABI_VERSION; }
int64_t nvc_wpack_count(const nvc_model* m) { return m ? wpack_count_of(m) : 0; }

int64_t nvc_train_workspace_bytes(const nvc_model* m, int64_t b) {
    if (!m) return 0;
    Net net = net_of(m);
    const int64_t nblk = b / kRows + 2;
    return nblk * (net.mlp_count * 4 + 8) + 256;
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
                    const int64_t* b_dev, int32_t shard, int32_t n_shards, uint16_t epoch, void* ws,
                    double* loss_out, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(pos && tgt && ws && m->grad_fx && m->touched, "nvc_train_grads: null argument");
    NVC_REQUIRE(n_shards >= 1 && shard >= 0 && shard < n_shards, "nvc_train_grads: bad shard");
    NVC_REQUIRE(m->out_sigmoid == 1 || m->out_sigmoid == 0, "bad output activation");
    if (b_max <= 0) return NVC_OK;
    Net net = net_of(m);
    GridDev g = grid_of(m);
    const int smem = mlp_smem_bytes(net);
    NVC_REQUIRE(smem <= 200 * 1024, "nvc_train_grads: MLP too wide for the fp32 tile kernel");
    const int64_t rows_max = b_max / n_shards + 1;
    const int nblk = grid1(rows_max, kRows);
    float* part_w = (float*)ws;
    double* part_loss = (double*)((char*)ws + ((int64_t)nblk * net.mlp_count * 4 + 255) / 256 * 256);
    cudaStream_t s = (cudaStream_t)stream;
    bool tiled = true;
    for (int i = 0; i <= net.n_layers; ++i) tiled = tiled && (net.dims[i] % 4 == 0);
    const int smem2 = t2_layout(net).total * 4 + 64;
    if (tiled && smem2 <= 200 * 1024) {
        cudaFuncSetAttribute(k_train2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem2);
        k_train2<<<nblk, kThreads, smem2, s>>>(g, net, m->params, pos, b_max, b_dev, shard, n_shards, tgt, mask,
                                               m->grad_fx, m->touched, epoch, part_w, part_loss);
    } else {
        cudaFuncSetAttribute(k_mlp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        k_mlp<true><<<nblk, kThreads, smem, s>>>(g, net, m->params, pos, b_max, b_dev, shard, n_shards, tgt, mask,
                                                  nullptr, m->grad_fx, m->touched, epoch, part_w, part_loss);
    }
    rc = check_launch("k_mlp<train>");
    if (rc) return rc;
    k_reduce_parts<<<grid1(net.mlp_count, 32), 256, 0, s>>>(part_w, part_loss, nblk, net.mlp_count,
                                                             net.grid_count, m->grad_fx, loss_out);
    return check_launch("k_reduce_parts");
}

int nvc_adam_step(const nvc_model* m, int64_t t, double lr, uint16_t epoch, int32_t dense, void* stream) {
    int rc = validate(m);
    if (rc) return rc;
    NVC_REQUIRE(t >= 1, "nvc_adam_step: t must be >= 1");
    NVC_REQUIRE(m->adam_m && m->adam_v && m->grad_fx && m->touched && m->table_h && m->wpack,
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
    k_adam_grid<<<grid1((net.grid_count + 7) / 8, 256), 256, 0, s>>>(m->params, m->adam_m, m->adam_v, m->grad_fx,
                                                                     m->touched, m->table_h, net.grid_count,
                                                                     m->features, epoch, dense, a, m->table_size);
    rc = check_launch("k_adam_grid");
    if (rc) return rc;
    k_adam_mlp<<<grid1(net.mlp_count, 256), 256, 0, s>>>(net, m->params, m->adam_m, m->adam_v, m->grad_fx,
                                                         m->wpack, a);
    return check_launch("k_adam_mlp");
}

}  // extern "C"
