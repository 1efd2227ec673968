/* nvc.h -- C ABI of the B200-native neural visibility cache (libnvc.so).
 *
 * The reference (`viscache` 0.1.0, /root/reference/pkg/src/viscache) is a pure
 * Python package; its "plugin" interface for this path is the duck-typed
 * cache object (`mode`, `output_dim`, `infer`, `train_step`) plus the sampling
 * functions that consume it.  Each entry point below replaces one reference
 * routine; the citation names the routine it stands in for.  A Python
 * (ctypes) host layer, `paper_2506_05930_b200`, mirrors the reference API on
 * top of these calls.
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer unless named `host_*`.
 *  - Every call is asynchronous on the given CUDA stream (NULL = legacy).
 *  - Return 0 on success, a negative nvc_status on error; nvc_last_error()
 *    returns a thread-local message describing the last failure.
 *  - The caller owns all memory (model state included); nvc_model only
 *    carries pointers and shapes.  No torch types cross this boundary.
 *  - Doubles are IEEE binary64, integers little-endian, arrays row-major.
 */
#ifndef NVC_H_
#define NVC_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NVC_MAX_LEVELS 32
#define NVC_MAX_LAYERS 8
#define NVC_ABI_VERSION 11

typedef enum {
    NVC_OK = 0,
    NVC_ERR_ARG = -1,          /* invalid argument (bad shape, null pointer, unsupported config) */
    NVC_ERR_CUDA = -2,         /* a CUDA runtime call or kernel launch failed */
    NVC_ERR_UNSUPPORTED = -3   /* valid config the requested kernel does not handle */
} nvc_status;

/* Fixed-point scale of the hash-grid / MLP gradient accumulators (int64):
 * value = fx * 2^-48.  Integer accumulation makes the scatter deterministic
 * and makes the data-parallel allreduce order-independent. */
#define NVC_GRAD_FX_BITS 48

/* Hash grid + MLP: the reference VisibilityCache state (cache.py:25-45,
 * hashgrid.py:32-65, mlp.py:24-60).  Parameter order in `params` is the
 * reference `_param_dict` / snapshot order: grid (L,T,F), w0 (out,in), b0, w1, ... */
typedef struct {
    int32_t levels;                       /* L */
    int32_t features;                     /* F */
    int64_t table_size;                   /* T (power of two) */
    int32_t resolution[NVC_MAX_LEVELS];   /* floor(base * scale^l), computed by the host */
    int32_t dense[NVC_MAX_LEVELS];        /* (res+1)^3 <= T */
    double aabb_min[3];
    double span[3];                       /* max(aabb_max - aabb_min, 1e-12) */
    int32_t n_layers;                     /* number of weight matrices */
    int32_t dims[NVC_MAX_LAYERS + 1];     /* input (= L*F), hidden..., output (= K) */
    float alpha;                          /* leaky-ReLU slope (0.01) */
    int32_t out_sigmoid;                  /* 1: sigmoid + clip output, 0: leaky output */
    /* device state, caller-allocated */
    float *params;                        /* f32 master parameters, param_count */
    float *adam_m, *adam_v;               /* f32 Adam moments, param_count */
    int64_t *grad_fx;                     /* fixed-point gradient accumulator, param_count (dense mode) */
    /* Compact gradient mode (grad_c != NULL; grad_fx is then unused).
     * nvc_train_index marks the batch's table entries in touch_bits (L*T bits)
     * and writes touch_off (per 32-entry word: rank of its first marked entry;
     * nvc_touch_off_len(m) int32 including scratch).  The scatter and Adam
     * address entry e's gradient as grad_c[rank(e)*F + f] and the MLP
     * gradients as grad_c[grad_c_entries*F + j]: a few MB that stay in L2,
     * and exactly the data-parallel allreduce buffer
     * (nvc_exchange_buffer_len(m, grad_c_entries) int64). */
    uint32_t *touch_bits;
    int32_t *touch_off;
    int64_t *grad_c;
    int64_t grad_c_entries;
    uint16_t *table_h;                    /* fp16 query table, x-pair layout: slot e = (f[e], f[next(e)]), 2*L*T*F */
    uint16_t *wpack;                      /* fp16 weights in the tcgen05 K-major core-matrix layout */
    int64_t param_count;
    int64_t wpack_count;                  /* halfs in wpack (nvc_wpack_count) */
} nvc_model;

/* Scene tables (scene.py:158-215, geometry.py:97-158).  BVH arrays are in the
 * reference's build order; tri_* arrays are in original triangle order. */
typedef struct {
    const double *node_min, *node_max;    /* (n_nodes, 3) */
    const int32_t *node_left, *node_right, *node_start, *node_count;
    const double *bv0, *bv1, *bv2;        /* (n_tris, 3), BVH leaf order */
    const int64_t *perm;                  /* BVH index -> original triangle index */
    const double *tv0, *tv1, *tv2;        /* (n_tris, 3), original order */
    const int32_t *tri_material, *tri_light;
    const double *mat_albedo;             /* (n_materials, 3) */
    const uint8_t *lt_kind;               /* 0 rect, 1 point */
    const double *lt_verts;               /* (K, 4, 3) */
    const double *lt_normal;              /* (K, 3) */
    const double *lt_radiance;            /* (K, 3) */
    const double *lt_lumaw;               /* (K, 3) LUMA * radiance, precomputed by the host */
    const double *lt_area;                /* (K) scene.py:189 (shade_batch's area term) */
    /* Shadow-ray acceleration data, precomputed by the host (scene.py
     * shadow_accel).  In BVH triangle order: tri_plane (n_tris, 4) f32 unit
     * normal and offset of each triangle's plane (all zeros: never culled --
     * zero area or a sliver); tri_box (n_tris, 8) f32 AABB for the
     * crossing-box filter; tri_leaf (n_tris) the BVH leaf holding the
     * triangle.  node_parent (n_nodes): parent node, -1 at the root.  With
     * anyhit_bf set, any-hit queries cull triangles with f32 tests whose
     * margin (plane_margin * (plane_r + |p0|inf + |p1|inf)) bounds their error
     * 32x, test the rest with the exact FP64 ray_tri, and accept a hit only if
     * every BVH ancestor of its leaf passes the FP64 slab test -- the same
     * answer as the reference's pruned BVH traversal (geometry.cu). */
    const float *tri_plane;
    const float *tri_box;                 /* (n_tris, 8) f32: min xyz, flag, max xyz, 0; flag 1 = no box test */
    const int32_t *tri_leaf;
    const int32_t *node_parent;
    float plane_margin, plane_r;
    int32_t anyhit_bf;
    int32_t pad0;
    int64_t n_nodes, n_tris;
    int32_t n_lights, n_materials;
    double shadow_eps;                    /* geometry.py:221-223 */
    double aabb_min[3], aabb_max[3];
} nvc_scene;

/* Pinhole camera with the basis precomputed by the host (scene.py:109-139). */
typedef struct {
    double pos[3], fwd[3], right[3], up[3];
    double tan_half, aspect;
    int32_t width, height;
} nvc_camera;

/* ---- library ---------------------------------------------------------- */
const char *nvc_last_error(void);
int32_t nvc_abi_version(void);
/* halfs of packed fp16 weights the tcgen05 path needs for this topology */
int64_t nvc_wpack_count(const nvc_model *m);
/* bytes of scratch nvc_train_grads needs for b rows */
int64_t nvc_train_workspace_bytes(const nvc_model *m, int64_t b);

/* Pin [ptr, ptr+bytes) (the fp16 hash table) in the persisting L2 carve-out
 * for kernels launched on `stream` (best effort; no-op if unsupported). */
int nvc_l2_persist(const void *ptr, int64_t bytes, void *stream);
/* Profiling aid: while enabled, the fp16 query (nvc_nls_sample /
 * nvc_neural_di / nvc_infer precision 1) records library-owned events on its
 * stream around its three kernels; nvc_profile_stage_ms waits for the last
 * query and returns the encoder, MLP and selection kernel times (ms). */
int nvc_profile_stages(int32_t enable);
int nvc_profile_stage_ms(float *ms3);

/* ---- state ------------------------------------------------------------ */
/* Rebuild table_h and wpack from params (after loading / setting params). */
int nvc_refresh_shadow(const nvc_model *m, void *stream);

/* ---- encoder: hashgrid.py:94-131 (encode_batch, _level_lookup, spatial_hash) */
/* feats (n, L*F) f32 from the f32 master table (exact reference op order);
 * idx_out (n, L, 8) int32 and w_out (n, L, 8) f64 are optional (may be NULL). */
int nvc_encode(const nvc_model *m, const double *pos, int64_t n, float *feats,
               int32_t *idx_out, double *w_out, void *stream);

/* grad_from_ctx (hashgrid.py:140-151) on nvc_encode's context: idx (b, L, 8)
 * int32 and w (b, L, 8) f64, upstream (b, L*F) f32; adds into grad (L, T, F)
 * f32 (zero it first for the reference's fresh table) every entry's
 * contributions float(w * g) in (row, corner) order -- bit-identical to
 * np.add.at. */
int nvc_grid_scatter(int32_t levels, int32_t features, int64_t table_size, const int32_t *idx,
                     const double *w, const float *upstream, int64_t b, float *grad, void *stream);

/* ---- inference: cache.py:54-58 (VisibilityCache.infer) ---------------- */
/* precision 0: f32 SIMT (parity: f32 table + f32 weights; workspace unused);
 * precision 1: fp16 table + tcgen05/TMEM MLP (fp32 accumulate). */
int nvc_infer(const nvc_model *m, const double *pos, int64_t n, int32_t precision,
              float *out, void *workspace, void *stream);
/* Scratch for the fp16 query pipeline (encode tiles -> tcgen05 MLP ->
 * selection) over p pixels; required by nvc_infer (precision 1),
 * nvc_nls_sample and nvc_neural_di. */
int64_t nvc_query_workspace_bytes(const nvc_model *m, int64_t p);

/* ---- training: cache.py:60-73 (train_step) split at the allreduce point --- */
/* Accumulates the gradient of the loss into grad_fx (int64 fixed point,
 * 2^-48; order-independent, so shards and atomics stay deterministic).  The batch has b global rows (b = *b_dev when b_dev
 * is non-NULL, else b_max); this call handles the shard rows
 * [b*shard/n_shards, b*(shard+1)/n_shards): pos is indexed by global row,
 * targets/mask (may be NULL) by shard-local row.  d_out is scaled by the
 * global b*K (mlp.py:162) so data-parallel shards sum to the full-batch
 * gradient.  loss_sum_out (device double[2]) receives [0] = sum_rows(sum_k d^2)/K
 * over the shard's rows and [1] = that sum / b (summing [1] over shards gives
 * the reference's batch loss, l2_loss mlp.py:143-149). */
int nvc_train_grads(const nvc_model *m, const double *pos, const float *targets,
                    const float *mask, int64_t b_max, const int64_t *b_dev,
                    int32_t shard, int32_t n_shards,
                    void *workspace, double *loss_sum_out, void *stream);
/* ---- data-parallel gradient exchange ------------------
 * Every rank builds the same global batch, so the table entries it touches
 * are the same on every rank.  nvc_exchange_index lists them (sorted, from the
 * positions of all b global rows); nvc_exchange_pack copies their fixed-point
 * gradients (zero-padded to max_entries) and the MLP gradients into one int64
 * buffer of nvc_exchange_buffer_len elements; the caller allreduces (sum) that
 * buffer instead of the whole grad_fx; nvc_exchange_unpack writes it back.
 * Entries nobody touched are zero on every rank, so this equals the dense
 * allreduce bit for bit. */
int64_t nvc_exchange_max_entries(const nvc_model *m, int64_t b);
/* Compact gradient mode: sizes of touch_bits (uint32 words) and touch_off
 * (int32), and the per-batch index build (before nvc_train_grads; b rows of
 * the GLOBAL batch, identical on every data-parallel rank). */
int64_t nvc_touch_words(const nvc_model *m);
int64_t nvc_touch_off_len(const nvc_model *m);
int nvc_train_index(const nvc_model *m, const double *pos, int64_t b_max, const int64_t *b_dev,
                    void *stream);
int64_t nvc_exchange_workspace_bytes(const nvc_model *m);
int64_t nvc_exchange_buffer_len(const nvc_model *m, int64_t max_entries);
int nvc_exchange_index(const nvc_model *m, const double *pos, int64_t b_max, const int64_t *b_dev,
                       void *workspace, int32_t *idx, int64_t *count, void *stream);
int nvc_exchange_pack(const nvc_model *m, const int32_t *idx, const int64_t *count, int64_t max_entries,
                      int64_t *buf, void *stream);
int nvc_exchange_unpack(const nvc_model *m, const int32_t *idx, const int64_t *count, int64_t max_entries,
                        const int64_t *buf, void *stream);

/* One bias-corrected Adam step over every parameter (mlp.py:203-218, dense
 * like the reference), consuming and zeroing grad_fx; refreshes table_h and
 * wpack.  t is the post-increment Adam step (>= 1), lr from lr_at (mlp.py:76).
 * grad_fx may hold a data-parallel allreduced sum. */
int nvc_adam_step(const nvc_model *m, int64_t t, double lr, void *stream);
/* Sharded optimizer for data parallelism: the same update on
 * the hash-table parameters [lo, hi) of shard `shard` of n_shards only (whole
 * Adam tiles; nvc_adam_shard_range gives the range), the MLP on every shard;
 * the other shards' gradients are cleared.  The caller then all-gathers the
 * table parameters and calls nvc_refresh_shadow.  Dense gradients, F == 2.
 * nvc_adam_step == shard 0 of 1. */
int nvc_adam_step_shard(const nvc_model *m, int64_t t, double lr, int32_t shard, int32_t n_shards,
                        void *stream);
int nvc_adam_shard_range(const nvc_model *m, int32_t shard, int32_t n_shards, int64_t *lo, int64_t *hi);

/* ---- light selection: sampling.py:74-85, 184-218 ---------------------- */
/* wrs_select_batch: weights (p, k) f64; draw for (row r, light j) is
 * offset + r*k + j of Philox stream `key` (rng.py:54-56). */
int nvc_wrs_select(const double *w, int64_t p, int32_t k, uint64_t key, uint64_t offset,
                   int64_t *idx, double *w_sel, double *w_sum, void *stream);
/* nls_sample_batch given visibility (p, k) f32 and luminance weights in
 * light-major layout lum[j*p_stride + r] (f32 if lum_f64 == 0 else f64).
 * Rows are pixels p_first.. of a p_total-pixel frame (screen-tile shards
 * reproduce the whole-frame draws).  floor <= 0 selects the biased mode. */
int nvc_nls_from_vis(const nvc_scene *sc, const float *vis, const void *lum, int32_t lum_f64,
                     int64_t p_stride, int64_t p, int32_t k, int64_t p_first, int64_t p_total,
                     uint64_t key, uint64_t offset, double floor,
                     int64_t *ids, double *pts, double *big_w, void *stream);
/* The hot path: encode -> tcgen05 MLP -> clamp * lum -> WRS -> light point
 * (three kernels: encoder tiles, persistent MLP, per-pixel reservoir) over
 * p pixels.  pos (p, 3) f64; lum light-major (k, p_stride); nz_mask
 * ceil(k/32) words per pixel, word w of pixel r at w*p_stride + r, bit j set
 * iff lum[32w+j][r] != 0 (nvc_table_mask; may be NULL); workspace from
 * nvc_query_workspace_bytes. */
int nvc_nls_sample(const nvc_model *m, const nvc_scene *sc, const double *pos,
                   const void *lum, int32_t lum_f64, const uint32_t *nz_mask, int64_t p_stride,
                   int64_t p, int64_t p_first, int64_t p_total, uint64_t key, uint64_t offset,
                   double floor, int64_t *ids, double *pts, double *big_w, void *workspace,
                   void *stream);
/* Fused Neural DI (sampling.py:215-218): rgb (p,3) f64 = sum_k v_k f_k L_k * albedo/pi,
 * factor in light-major layout (f32 or f64). */
/* nvc_nls_sample split in two (same results): the encoder + MLP write the fp16
 * visibilities of p pixels into the workspace, and the selection reads them.
 * The selection may run on another stream (e.g. overlapping the next frame's
 * train step) as long as no other nvc_query_front reuses the workspace before
 * it has finished. */
int nvc_query_front(const nvc_model *m, const double *pos, int64_t p, void *workspace, void *stream);
int nvc_nls_select(const nvc_model *m, const nvc_scene *sc, const void *lum, int32_t lum_f64,
                   const uint32_t *nz_mask, int64_t p_stride, int64_t p, int64_t p_first,
                   int64_t p_total, uint64_t key, uint64_t offset, double floor, int64_t *ids,
                   double *pts, double *big_w, void *workspace, void *stream);
int nvc_neural_di(const nvc_model *m, const nvc_scene *sc, const double *pos,
                  const double *albedo, const void *factor, int32_t factor_f64,
                  const uint32_t *nz_mask, int64_t p_stride, int64_t p, double *rgb, void *workspace,
                  void *stream);
/* Nonzero mask of a light-major table (K <= 32 uses one word per pixel):
 * bit j of mask[w*p_stride + r] is set iff table[(32w+j)*p_stride + r] != 0.
 * Passed as nz_mask above, it lets the fused kernels skip zero-weight lights
 * (exact: they add 0 to the reservoir sum and are never selected). */
int nvc_table_mask(const void *table, int32_t f64, int64_t p_stride, int64_t p, int32_t k,
                   uint32_t *mask, void *stream);

/* ---- RIS / screen-space ReSTIR baselines: sampling.py:369-637 ---------- */
/* A reservoir grid (ReservoirGrid, sampling.py:369-402), struct of arrays on
 * the device: y (p) i64, point (p,3) f64, w_y/w_sum/M/W (p) f64, valid (p) u8. */
typedef struct nvc_rgrid {
    int64_t *y;
    double *point, *w_y, *w_sum, *M, *W;
    uint8_t *valid;
} nvc_rgrid;
/* ris_initial_batch (:405-432): m_cand candidates per pixel from
 * integers(0, K) (Lemire, rejections and the kept 32-bit half exact; kept_in
 * -1: none), phat from the light-major luminance table, streaming WRS, light
 * points.  state_dev (2 int64, device): the stream's next 64-bit output and
 * kept half after the call.  ws: nvc_ris_workspace_bytes. */
int64_t nvc_ris_workspace_bytes(int64_t p, int32_t m_cand, int32_t k);
int nvc_ris_initial(const nvc_scene *sc, const void *lum, int32_t lum_f64, int64_t stride, int64_t p,
                    int32_t m_cand, uint64_t key, uint64_t offset, int64_t kept_in, const nvc_rgrid *out,
                    void *ws, int64_t *state_dev, void *stream);
/* restir_temporal_batch (:487-526): clamp_mode 0 "m", 1 "contribution";
 * phat from the f64 light-major factor table and the pixel albedos. */
int nvc_restir_temporal(const nvc_scene *sc, const double *factor, int64_t stride, const double *alb,
                        int64_t p, const nvc_rgrid *cur, const nvc_rgrid *prev, uint64_t key, uint64_t offset,
                        double clamp, int32_t clamp_mode, const nvc_rgrid *out, void *stream);
/* restir_spatial_batch (:541-595) over a width x height frame (out must not alias grid). */
int nvc_restir_spatial(const nvc_scene *sc, const double *factor, int64_t stride, const double *alb,
                       const double *nrm, const uint8_t *hit, const double *depth, int32_t width,
                       int32_t height, const nvc_rgrid *grid, uint64_t key, uint64_t offset, int32_t radius,
                       int32_t neighbors, const nvc_rgrid *out, void *stream);
/* PixelCtx.phat_ids (:141-155), one id per pixel (id < 0 -> 0). */
int nvc_phat_ids(const nvc_scene *sc, const double *factor, int64_t stride, const double *alb,
                 const int64_t *ids, int64_t p, double *out, void *stream);

/* ---- geometry + training data: geometry.py, render.py, training.py ----- */
/* make_gbuffer / trace_rays (render.py:49-117) for pixels [p_first, p_first+p):
 * pos/nrm/alb (p,3) f64, hit (p) u8, light_id (p) i32, depth (p) f64 (+inf on a
 * miss) and emissive (p,3) f64 (the radiance of an emitter hit on its front
 * face); hit, light_id, depth and emissive may be NULL. */
int nvc_gbuffer(const nvc_scene *sc, const nvc_camera *cam, uint64_t jitter_key,
                int64_t p_first, int64_t p, double *pos, double *nrm, double *alb,
                uint8_t *hit, int32_t *light_id, double *depth, double *emissive, void *stream);
/* light_factors_all (kernels.py:299-316) -> light-major f32/f64 factor and,
 * optionally, lum = factor * (albedo . LUMA*L)/pi (sampling.py:134-139). */
int nvc_light_factors(const nvc_scene *sc, const double *pos, const double *nrm,
                      const double *alb, int64_t p, int64_t p_stride, int32_t out_f64,
                      void *factor_out, void *lum_out, void *stream);
/* visibility_batch (geometry.py:233-247): vis (n) f32 in {0,1}. */
int nvc_visibility(const nvc_scene *sc, const double *x, const double *y, int64_t n,
                   float *vis, void *stream);
/* Cluster-mode shadow-ray targets (training.py:121-128) for a batch already in
 * pos / n_rows (nvc_gen_train_batch with tgt = NULL): per cluster j (ascending)
 * a uniform member -- numpy Generator.integers, exact including its rejection
 * loop and the bit generator's kept 32-bit half -- then the member's light point
 * from the same stream; tgt (rows of this shard, m) f32.  Clusters as device
 * int32 arrays c_off (m+1) and c_mem (c_off[m]) (clusters.ClusterSet.packed).
 * The stream starts at 64-bit output `offset` with the bit generator's kept
 * 32-bit half `kept_in` (-1: none) -- a used numpy Generator continues exactly;
 * ws: nvc_cluster_workspace_bytes(b_max, m); at nvc_cluster_state_offset the
 * call leaves int64 [m+2]: per cluster the first output of its random() draws,
 * then the stream's next 64-bit output and its kept 32-bit half (-1: none). */
int64_t nvc_cluster_workspace_bytes(int64_t b_max, int32_t m);
int64_t nvc_cluster_state_offset(int64_t b_max, int32_t m);
int nvc_cluster_targets(const nvc_scene *sc, uint64_t key, uint64_t offset, int64_t kept_in,
                        const double *pos, const int64_t *n_rows, int64_t b_max, int32_t shard,
                        int32_t n_shards, int32_t m, const int32_t *c_off, const int32_t *c_mem,
                        float *tgt, void *ws, void *stream);
/* clustered_sample_batch (sampling.py:302-352): WRS over the m clamped cluster
 * visibilities vis (p, vis_stride) f32, then per cluster (ascending) a WRS over
 * its member lights with weights phat / p_src on the continuing stream (draws
 * for a cluster's pixels in pixel order), then light points -- ids (p) i64,
 * pts (p,3) f64, big_w (p) f64.  Whole frames (pixel 0 .. p-1), p <= 2^31.
 * factor: NULL (factors computed per pixel and member) or the per-camera
 * light-major f64 table (K, p) of nvc_light_factors (identical values).
 * ws: nvc_clustered_workspace_bytes(p, m); at nvc_clustered_state_offset an
 * int64 holds the first light-point draw (the call consumes it + 2p - offset). */
int64_t nvc_clustered_workspace_bytes(int64_t p, int32_t m);
int64_t nvc_clustered_state_offset(int64_t p, int32_t m);
int nvc_clustered_select(const nvc_scene *sc, const float *vis, int64_t vis_stride, const double *pos,
                         const double *nrm, const double *alb, const double *factor, int64_t p, int32_t m,
                         const int32_t *c_off, const int32_t *c_mem, uint64_t key, uint64_t offset, double floor,
                         int64_t *ids, double *pts, double *big_w, void *ws, void *stream);
/* The clustered selection with the factors read from a cluster-ordered
 * pixel-major table: nvc_cluster_factor_table writes out (p, k) f64 with
 * out[q*k + i] = factor[c_mem[i]*p + q] (factor: the light-major (K, p) table
 * of nvc_light_factors, k = c_off[m] members), so a pixel's candidate members
 * are one contiguous run; nvc_clustered_select_ct then takes that table
 * (ct_stride = k) in place of the light-major one.  Identical results to
 * nvc_clustered_select with the light-major table. */
int nvc_cluster_factor_table(const double *factor, int64_t p, int32_t k, const int32_t *c_mem, double *out,
                             void *stream);
int nvc_clustered_select_ct(const nvc_scene *sc, const float *vis, int64_t vis_stride, const double *pos,
                            const double *nrm, const double *alb, const double *factor_ct, int64_t ct_stride,
                            int64_t p, int32_t m, const int32_t *c_off, const int32_t *c_mem, uint64_t key,
                            uint64_t offset, double floor, int64_t *ids, double *pts, double *big_w, void *ws,
                            void *stream);
/* shade_batch (render.py:220-246): one-shadow-ray estimate per row,
 * rgb (n,3) f64 = albedo/pi * L_e[id] * G * V * (area) * W; rows with id < 0,
 * id >= K or W <= 0 (and rows with G <= 0) are 0.  Bit-identical to the
 * reference.  pos/nrm/alb/pts (n,3) f64, ids (n) i64, big_w (n) f64. */
int nvc_shade(const nvc_scene *sc, const double *pos, const double *nrm, const double *alb,
              const int64_t *ids, const double *pts, const double *big_w, int64_t n, double *rgb,
              void *stream);
/* trace_rays (render.py:49-75) for camera rays through screen points
 * sxy (n, 2) f64 (camera_rays_batch, scene.py:129-139): the hit attributes
 * gen_screen_hits (training.py:67-94) keeps. */
int nvc_primary_hits(const nvc_scene *sc, const nvc_camera *cam, const double *sxy, int64_t n,
                     double *pos, double *nrm, double *alb, uint8_t *hit, int32_t *light_id,
                     void *stream);
/* intersect_scene_batch (geometry.py:191-207): t, original tri index (-1 miss). */
int nvc_closest_hit(const nvc_scene *sc, const double *orig, const double *dir,
                    const double *t_min, const double *t_max, int64_t n,
                    double *t_out, int64_t *tri_out, void *stream);
/* One training batch (training.py:44-129, 176-195): world samples, screen
 * samples (<= 9 rounds, order-preserving compaction) and targets.  Every
 * shard generates all b = n_world + screen-hits global positions (cheap,
 * keeps the in-order compaction global) and the targets of its rows
 * [b*shard/n_shards, b*(shard+1)/n_shards) only (tgt may be NULL: no targets).  pos capacity:
 * n_world+n_screen rows; tgt capacity: same rows x K (shard-local rows);
 * n_rows (device int64) receives b. */
int64_t nvc_batch_workspace_bytes(int32_t n_world, int32_t n_screen);
/* compute_visibility_targets (training.py:103-120, light mode) for given
 * positions (b,3): tgt (b,K) f32, light j / row i use draws
 * offset + j*2b + 2i, +1 (offset: the stream's position when called). */
int nvc_targets(const nvc_scene *sc, uint64_t key, uint64_t offset, const double *pos, int64_t b,
                float *tgt, void *stream);
int nvc_gen_train_batch(const nvc_scene *sc, const nvc_camera *cam, uint64_t key_world,
                        uint64_t key_screen, uint64_t key_targets, uint64_t off_world,
                        uint64_t off_screen, int32_t n_world, int32_t n_screen, int32_t shard,
                        int32_t n_shards, double *pos, float *tgt, int64_t *n_rows,
                        void *workspace, void *stream);
/* (off_world / off_screen: the world / screen streams' positions -- 0 for the
 * fresh per-frame streams; the screen stream's position after the call is the
 * int64 at byte 16 of the workspace) */

#ifdef __cplusplus
}
#endif
#endif /* NVC_H_ */
