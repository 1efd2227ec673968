// query.cu -- the C entry points of the query path (infer / NLS / Neural DI
// through the three-stage pipeline in pipeline.cu) and the standalone
// WRS kernels used on given weights or visibilities (parity entry points).
//
// Reference routines (under /root/reference/pkg/src/viscache):
//   VisibilityCache.infer cache.py:54-58, clamp_visibility sampling.py:27-30,
//   wrs_select_batch :74-85, nls_weights_batch :184-191,
//   nls_sample_batch :194-205, neural_di_batch :215-218,
//   Scene.light_points scene.py:204-215.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"

namespace nvc {
namespace {

// streaming reservoir state of one pixel (wrs_select_batch, sequential FP64)
struct Reservoir {
    double s, wsel;
    int sel;
    uint64_t blk;       // cached Philox block index (n/4+1), 0 = none
    U4 u;
};

// one out-of-line copy of the 10-round Philox keeps the instruction footprint small
__device__ __noinline__ U4 philox_call(uint64_t counter, uint64_t key) { return philox_block(counter, key); }

__device__ __forceinline__ double draw_cached(Reservoir& r, uint64_t key, uint64_t n) {
    const uint64_t b = n / 4 + 1;
    if (b != r.blk) {
        r.u = philox_call(b, key);
        r.blk = b;
    }
    return u01(r.u.x[n & 3]);
}

__device__ __forceinline__ void reservoir_push(Reservoir& r, double w, int k, uint64_t key, uint64_t n) {
    r.s = __dadd_rn(r.s, w);
    if (w > 0.0) {   // u*s < 0 is impossible: zero-weight lights never need a uniform
        const double u = draw_cached(r, key, n);
        if (__dmul_rn(u, r.s) < w) {
            r.sel = k;
            r.wsel = w;
        }
    }
}

__device__ __forceinline__ void draw_pair(uint64_t key, uint64_t n, double& a, double& b) {
    const U4 blk = philox_call(n / 4 + 1, key);
    a = u01(blk.x[n & 3]);
    if ((n & 3) != 3) {
        b = u01(blk.x[(n & 3) + 1]);
    } else {
        const U4 nb = philox_call(n / 4 + 2, key);
        b = u01(nb.x[0]);
    }
}

// ---------------------------------------------------------------------------
// standalone WRS on given weights (parity entry points)
// ---------------------------------------------------------------------------
__global__ void k_wrs_select(const double* __restrict__ w, int64_t P, int K, uint64_t key, uint64_t offset,
                             int64_t* __restrict__ idx, double* __restrict__ wsel, double* __restrict__ wsum) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    Reservoir r;
    r.s = 0.0;
    r.wsel = 0.0;
    r.sel = -1;
    r.blk = 0;
    for (int k = 0; k < K; ++k) reservoir_push(r, w[p * K + k], k, key, offset + (uint64_t)p * K + k);
    idx[p] = r.sel;
    wsel[p] = r.sel >= 0 ? r.wsel : 0.0;
    wsum[p] = r.s;
}

template <typename T>
__global__ void k_nls_from_vis(nvc_scene sc, const float* __restrict__ vis, const T* __restrict__ lum, int64_t stride,
                               int64_t P, int K, int64_t p_first, int64_t p_total, uint64_t key, uint64_t offset,
                               double floor, int64_t* __restrict__ ids, double* __restrict__ pts,
                               double* __restrict__ big_w) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int64_t gp = p_first + p;
    Reservoir r;
    r.s = 0.0;
    r.wsel = 0.0;
    r.sel = -1;
    r.blk = 0;
    for (int k = 0; k < K; ++k) {
        double v = (double)vis[p * K + k];
        v = floor > 0.0 ? fmax(v, floor) : fmax(v, 0.0);
        reservoir_push(r, __dmul_rn(v, (double)lum[(int64_t)k * stride + p]), k, key,
                       offset + (uint64_t)gp * K + k);
    }
    double u0, u1, y[3];
    draw_pair(key, offset + (uint64_t)p_total * K + 2ull * gp, u0, u1);
    light_point(sc, r.sel, u0, u1, y);
    ids[p] = r.sel;
    big_w[p] = r.sel >= 0 ? __ddiv_rn(r.s, r.wsel > 0.0 ? r.wsel : 1.0) : 0.0;
    pts[3 * p] = y[0];
    pts[3 * p + 1] = y[1];
    pts[3 * p + 2] = y[2];
}

template <typename T>
__global__ void k_table_mask(const T* __restrict__ t, int64_t stride, int64_t P, int K, uint32_t* __restrict__ mask) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int w = blockIdx.y;
    if (p >= P) return;
    uint32_t m = 0;
    for (int j = 0; j < 32 && 32 * w + j < K; ++j)
        if (t[(int64_t)(32 * w + j) * stride + p] != (T)0) m |= 1u << j;
    mask[(int64_t)w * stride + p] = m;
}


inline int grid1(int64_t n, int bs) { return (int)((n + bs - 1) / bs); }

}  // namespace

int64_t pipeline_workspace_bytes(const nvc_model* m, int64_t P);
int pipeline_front(const nvc_model* m, const double* pos, int64_t P, void* ws, cudaStream_t s);
int pipeline_select(const nvc_model* m, const nvc_scene* sc, int64_t P, int mode, const void* lum, int lum_f64,
                    int64_t stride, const uint32_t* nz_mask, int64_t p_first, int64_t p_total, uint64_t key,
                    uint64_t offset, double floor, int64_t* ids, double* pts, double* big_w, const double* albedo,
                    double* rgb, float* vis_out, void* ws, cudaStream_t s);
int pipeline_query(const nvc_model* m, const nvc_scene* sc, const double* pos, int64_t P, int mode,
                   const void* lum, int lum_f64, int64_t stride, const uint32_t* nz_mask, int64_t p_first, int64_t p_total,
                   uint64_t key, uint64_t offset, double floor, int64_t* ids, double* pts, double* big_w,
                   const double* albedo, double* rgb, float* vis_out, void* ws, cudaStream_t s);

}  // namespace nvc

using namespace nvc;

extern "C" {

int64_t nvc_query_workspace_bytes(const nvc_model* m, int64_t p) {
    return (m && p > 0) ? pipeline_workspace_bytes(m, p) : 0;
}

int nvc_infer(const nvc_model* m, const double* pos, int64_t n, int32_t precision, float* out, void* workspace,
              void* stream) {
    if (n <= 0) return NVC_OK;
    NVC_REQUIRE(m && pos && out, "nvc_infer: null argument");
    if (precision == 0) return nvc_infer_f32(m, pos, n, out, (cudaStream_t)stream);
    NVC_REQUIRE(workspace, "nvc_infer: the fp16 path needs nvc_query_workspace_bytes() of workspace");
    return pipeline_query(m, nullptr, pos, n, 0, nullptr, 0, 0, nullptr, 0, n, 0, 0, 0.0, nullptr, nullptr, nullptr,
                          nullptr, nullptr, out, workspace, (cudaStream_t)stream);
}

int nvc_nls_sample(const nvc_model* m, const nvc_scene* sc, const double* pos, const void* lum, int32_t lum_f64,
                   const uint32_t* nz_mask, int64_t stride, int64_t p, int64_t p_first, int64_t p_total,
                   uint64_t key, uint64_t offset, double floor, int64_t* ids, double* pts, double* big_w,
                   void* workspace, void* stream) {
    NVC_REQUIRE(m && sc && pos && lum && ids && pts && big_w, "nvc_nls_sample: null argument");
    NVC_REQUIRE(sc->n_lights == m->dims[m->n_layers], "nvc_nls_sample: output_dim != scene lights");
    NVC_REQUIRE(stride >= p && p_total >= p_first + p, "nvc_nls_sample: bad stride / frame size");
    if (p <= 0) return NVC_OK;
    NVC_REQUIRE(workspace, "nvc_nls_sample: needs nvc_query_workspace_bytes() of workspace");
    return pipeline_query(m, sc, pos, p, 1, lum, lum_f64, stride, nz_mask, p_first, p_total, key, offset, floor, ids, pts,
                          big_w, nullptr, nullptr, nullptr, workspace, (cudaStream_t)stream);
}

int nvc_query_front(const nvc_model* m, const double* pos, int64_t p, void* workspace, void* stream) {
    NVC_REQUIRE(m && pos && workspace, "nvc_query_front: null argument");
    if (p <= 0) return NVC_OK;
    return pipeline_front(m, pos, p, workspace, (cudaStream_t)stream);
}

int nvc_nls_select(const nvc_model* m, const nvc_scene* sc, const void* lum, int32_t lum_f64, const uint32_t* nz_mask,
                   int64_t stride, int64_t p, int64_t p_first, int64_t p_total, uint64_t key, uint64_t offset,
                   double floor, int64_t* ids, double* pts, double* big_w, void* workspace, void* stream) {
    NVC_REQUIRE(m && sc && lum && ids && pts && big_w && workspace, "nvc_nls_select: null argument");
    NVC_REQUIRE(sc->n_lights == m->dims[m->n_layers], "nvc_nls_select: output_dim != scene lights");
    NVC_REQUIRE(stride >= p && p_total >= p_first + p, "nvc_nls_select: bad stride / frame size");
    if (p <= 0) return NVC_OK;
    return pipeline_select(m, sc, p, 1, lum, lum_f64, stride, nz_mask, p_first, p_total, key, offset, floor, ids, pts,
                           big_w, nullptr, nullptr, nullptr, workspace, (cudaStream_t)stream);
}

int nvc_neural_di(const nvc_model* m, const nvc_scene* sc, const double* pos, const double* albedo,
                  const void* factor, int32_t factor_f64, const uint32_t* nz_mask, int64_t stride, int64_t p,
                  double* rgb, void* workspace, void* stream) {
    NVC_REQUIRE(m && sc && pos && albedo && factor && rgb, "nvc_neural_di: null argument");
    NVC_REQUIRE(sc->n_lights == m->dims[m->n_layers], "nvc_neural_di: output_dim != scene lights");
    if (p <= 0) return NVC_OK;
    NVC_REQUIRE(workspace, "nvc_neural_di: needs nvc_query_workspace_bytes() of workspace");
    return pipeline_query(m, sc, pos, p, 2, factor, factor_f64, stride, nz_mask, 0, p, 0, 0, 0.0, nullptr, nullptr, nullptr,
                          albedo, rgb, nullptr, workspace, (cudaStream_t)stream);
}

int nvc_l2_persist(const void* ptr, int64_t bytes, void* stream) {
    // keep the fp16 hash table L2-resident while lum / G-buffer rows stream past it
    int dev = 0;
    cudaGetDevice(&dev);
    int max_persist = 0, max_window = 0;
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    if (max_persist <= 0 || max_window <= 0 || !ptr || bytes <= 0) return NVC_OK;
    const size_t want = (size_t)bytes < (size_t)max_persist ? (size_t)bytes : (size_t)max_persist;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
        cudaGetLastError();
        return NVC_OK;
    }
    cudaStreamAttrValue attr;
    memset(&attr, 0, sizeof attr);
    attr.accessPolicyWindow.base_ptr = const_cast<void*>(ptr);
    attr.accessPolicyWindow.num_bytes = (size_t)bytes < (size_t)max_window ? (size_t)bytes : (size_t)max_window;
    attr.accessPolicyWindow.hitRatio = (float)want / (float)attr.accessPolicyWindow.num_bytes;
    if (attr.accessPolicyWindow.hitRatio > 1.0f) attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (cudaStreamSetAttribute((cudaStream_t)stream, cudaStreamAttributeAccessPolicyWindow, &attr) != cudaSuccess)
        cudaGetLastError();
    return NVC_OK;
}

int nvc_table_mask(const void* table, int32_t f64, int64_t stride, int64_t p, int32_t k, uint32_t* mask,
                   void* stream) {
    NVC_REQUIRE(table && mask && k >= 1 && stride >= p, "nvc_table_mask: bad argument");
    if (p <= 0) return NVC_OK;
    dim3 g(grid1(p, 256), (k + 31) / 32);
    if (f64)
        k_table_mask<double><<<g, 256, 0, (cudaStream_t)stream>>>((const double*)table, stride, p, k, mask);
    else
        k_table_mask<float><<<g, 256, 0, (cudaStream_t)stream>>>((const float*)table, stride, p, k, mask);
    return check_launch("k_table_mask");
}

int nvc_wrs_select(const double* w, int64_t p, int32_t k, uint64_t key, uint64_t offset, int64_t* idx,
                   double* w_sel, double* w_sum, void* stream) {
    NVC_REQUIRE(w && idx && w_sel && w_sum && k >= 1, "nvc_wrs_select: bad argument");
    if (p <= 0) return NVC_OK;
    k_wrs_select<<<grid1(p, 128), 128, 0, (cudaStream_t)stream>>>(w, p, k, key, offset, idx, w_sel, w_sum);
    return check_launch("k_wrs_select");
}

int nvc_nls_from_vis(const nvc_scene* sc, const float* vis, const void* lum, int32_t lum_f64, int64_t stride,
                     int64_t p, int32_t k, int64_t p_first, int64_t p_total, uint64_t key, uint64_t offset,
                     double floor, int64_t* ids, double* pts, double* big_w, void* stream) {
    NVC_REQUIRE(sc && vis && lum && ids && pts && big_w && k >= 1, "nvc_nls_from_vis: bad argument");
    NVC_REQUIRE(stride >= p && p_total >= p_first + p, "nvc_nls_from_vis: bad stride / frame size");
    if (p <= 0) return NVC_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (lum_f64)
        k_nls_from_vis<double><<<grid1(p, 128), 128, 0, s>>>(*sc, vis, (const double*)lum, stride, p, k, p_first,
                                                             p_total, key, offset, floor, ids, pts, big_w);
    else
        k_nls_from_vis<float><<<grid1(p, 128), 128, 0, s>>>(*sc, vis, (const float*)lum, stride, p, k, p_first,
                                                            p_total, key, offset, floor, ids, pts, big_w);
    return check_launch("k_nls_from_vis");
}

}  // extern "C"
