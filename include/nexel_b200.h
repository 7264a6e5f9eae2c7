/*
 * nexel_b200.h — C-ABI of the B200 (sm_100a) Nexel render path.
 *
 * This is the drop-in boundary for the reference's render hot path
 * (reference: /root/reference/proj/core, namespace nexel):
 *
 *   reference C++ entry point                         C-ABI replacement
 *   ------------------------------------------------  -------------------------------------
 *   collection_pass(Scene, Camera, RenderResult&)      nx_collection_pass
 *       include/nexel/renderer.hpp:22, src/renderer.cpp:115-171
 *   texturing_pass(Scene, Camera, FrameBuffers&)       nx_texturing_pass
 *       include/nexel/renderer.hpp:26, src/renderer.cpp:207-237
 *   render(Scene, Camera) -> RenderResult              nx_render (+ nx_frame_download)
 *       include/nexel/renderer.hpp:28, src/renderer.cpp:239-244
 *   Scene / RenderSettings / TextureField (scene.hpp:10-32,
 *       texture_field.hpp:16-25, hash_grid.hpp:39-66, mlp.hpp:11-33)
 *                                                      nx_scene_create (device-resident copy)
 *   FrameBuffers / RenderResult (framebuffers.hpp:61-86,
 *       renderer.hpp:11-16)                            nx_frame_* (device-resident buffers)
 *   nexel::Error{code,msg} (error.hpp:10-22)           int status codes + nx_ctx_last_error
 *       "bad-settings"  renderer.cpp:13-21  -> NX_BAD_SETTINGS
 *       "bad-camera"    camera.cpp:8-31     -> NX_BAD_CAMERA
 *       "bad-primitive" primitive.cpp:47-63 -> NX_BAD_PRIMITIVE
 *
 * Conventions: every function returns NX_OK (0) or an NX_* code; on failure the
 * message is available from nx_ctx_last_error(). Exceptions never cross this
 * boundary. Host arrays use the reference's in-memory layouts (doubles, row-major
 * [out][in] MLP weights, [level][row][feature] hash table, 60 doubles per Nexel in
 * field order). `stream` arguments are cudaStream_t passed as void* (NULL = the
 * context's own stream). A context is bound to one device and one host thread.
 */
#ifndef NEXEL_B200_H
#define NEXEL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NX_OK 0
#define NX_BAD_SETTINGS 1    /* "bad-settings"  (renderer.cpp:13-21) */
#define NX_BAD_CAMERA 2      /* "bad-camera"    (camera.cpp:8-31)    */
#define NX_BAD_PRIMITIVE 3   /* "bad-primitive" (primitive.cpp:47-63) */
#define NX_MISSING_FILE 4    /* "missing-file"  (checkpoint.cpp:57)   */
#define NX_BAD_CHECKPOINT 5  /* "bad-checkpoint" (checkpoint.cpp:59-269) */
#define NX_INVALID_ARGUMENT 10
#define NX_UNSUPPORTED 11
#define NX_OUT_OF_MEMORY 12
#define NX_CUDA_ERROR 13
#define NX_NO_DEVICE 14

#define NX_MAX_TOP_K 8          /* kMaxTopK, scene.hpp:23 */
#define NX_PARAMS_PER_NEXEL 60  /* kParamsPerPrimitive, primitive.hpp:14 */
#define NX_SH_VALUES 48         /* kShValues, primitive.hpp:12 */

typedef struct nx_ctx nx_ctx;
typedef struct nx_scene nx_scene;
typedef struct nx_frame nx_frame;

/* RenderSettings (scene.hpp:10-21). Booleans are 0/1. */
typedef struct nx_settings {
    int32_t top_k;              /* 0..8; 0 disables the texture pass */
    int32_t tile;               /* >= 1; the CUDA path supports tile <= 32 */
    double background[3];
    double near_eps;            /* default 1e-3 */
    double alpha_max;           /* default 0.999 */
    double min_transmittance;   /* default 1e-4 */
    int32_t no_gamma;
    int32_t no_prim_sh;
    int32_t no_downweight;
    int32_t precision;          /* NX_PRECISION_DEFAULT: fp64 decisions / depths / weights, fp32 colour,
                                   bf16x3 tensor-core decoder; NX_PRECISION_F64: fp64 colour as well
                                   (SH, hash grid, decoder, base, texture, final — the reference's
                                   FrameBuffers precision; fp64 copies of SH / table / MLP kept on the
                                   device; render-only: no optimizer / density control) */
} nx_settings;
enum { NX_PRECISION_DEFAULT = 0, NX_PRECISION_F64 = 1 };

/* HashGridConfig (hash_grid.hpp:39-56) + TextureMlp shapes (mlp.hpp:11-33). */
typedef struct nx_field_desc {
    int32_t levels;       /* 16 */
    int32_t log2_table;   /* 20 */
    int32_t features;     /* 2 */
    int32_t n_hidden;     /* 64; n_in = levels*features, n_out = 48 */
    double base_scale;    /* 1/extent */
    double growth;        /* 32768^(1/(levels-1)) */
} nx_field_desc;

/* Camera (camera.hpp:17-43): pinhole, OpenCV axes, X_cam = R X_world + t. */
typedef struct nx_camera {
    int32_t width, height;
    double fx, fy, cx, cy;
    double R[9];   /* row-major */
    double t[3];
} nx_camera;

/* Device-resident frame buffers (FrameBuffers, framebuffers.hpp:61-86).
 * Slot layout is pixel-major, slot-minor like the reference: slot = pix*K + j.
 * Types: decisions and contributor data stay fp64 (depths, weights); colour
 * buffers are fp32 (tolerance-checked). */
typedef struct nx_frame_view {
    int32_t width, height, top_k, tiles_x, tiles_y;
    float* base;          /* H*W*3 */
    int32_t* ids;         /* H*W*K, -1 sentinel */
    double* depths;       /* H*W*K */
    double* weights;      /* H*W*K */
    float* texture;       /* H*W*K*3 */
    float* final_img;     /* H*W*3 */
    float* residual;      /* H*W */
} nx_frame_view;

/* Host destination for nx_frame_download; any pointer may be NULL (skipped). */
typedef struct nx_host_frame {
    float* base;
    int32_t* ids;
    double* depths;
    double* weights;
    float* texture;
    float* final_img;
    float* residual;
    double* base_f64;  /* fp64 base (Eq. 6) kept for render_backward; download: copied if the
                          frame keeps it (nx_frame_set_backward); upload: makes the frame keep it */
    double* residual_f64;  /* fp64 terminal transmittance, kept with the fp64 base (same rules) —
                              FrameBuffers::residual at the reference's precision */
    double* texture_f64;   /* download only: fp64 texture / final of an NX_PRECISION_F64 render */
    double* final_f64;
    float* weights_f32;    /* download only, pinned memory, exclusive with `weights`: the slot weights
                              as fp32. Display frames composite in fp32 (certified march), so their
                              weights are fp32 values and this halves their bytes losslessly (the few
                              pixels the exact redo re-renders are rounded to fp32). */
} nx_host_frame;

/* Per-frame binning / work statistics (read back with nx_frame_stats). */
typedef struct nx_frame_stats {
    int64_t n_nexels;
    int64_t n_entries;        /* primitives with a binning entry (renderer.cpp:100) */
    int64_t n_dropped_support;/* ru<=0 or rv<=0 (renderer.cpp:54-56) */
    int64_t n_behind;         /* fully behind the pinhole (renderer.cpp:77) */
    int64_t n_offscreen;      /* rect off screen (renderer.cpp:88) */
    int64_t n_rect;           /* rect-binned */
    int64_t n_straddlers;     /* all-tile fallback (renderer.cpp:93-98) */
    int64_t n_straddlers_kept;/* straddlers whose refined work rect is non-empty */
    int64_t tile_keys;        /* reference tile-key count P (sum of tile-list lengths) */
    int64_t work_keys;        /* keys materialised and walked by the composite kernel */
    int64_t n_queries;        /* texture queries Q (non-empty slots) */
    /* near-threshold decisions (margin below >= 100x what device vs reference math can
     * differ by): zero means every decision of the frame is the reference's beyond doubt */
    int64_t near_alpha;        /* hits with alpha within 1e-12 (relative) of 1/255 (kernel.hpp:11) */
    int64_t near_transmittance;/* T within 1e-11 of min_transmittance at a composite step */
    int64_t near_topk;         /* top-K comparisons between weights within 1e-11 */
    int64_t near_depth;        /* sorted neighbours with depths within 1e-13 (renderer.cpp:102-105) */
    int64_t near_rect;         /* rect floor / ceil arguments within 1e-9 px of an integer */
    int64_t near_support;      /* 2 ln(255 o) within 1e-13 of 0 (support radius sign) */
    int64_t redo_tiles;        /* pixels the certified composite handed to the exact redo */
} nx_frame_stats;

/* ---- context ---------------------------------------------------------- */
const char* nx_version(void);
const char* nx_status_name(int status);            /* "bad-settings", ... */
int nx_device_count(int* count);
int nx_ctx_create(int device, nx_ctx** out);
void nx_ctx_destroy(nx_ctx* ctx);
const char* nx_ctx_last_error(const nx_ctx* ctx, int* status);
void* nx_ctx_stream(nx_ctx* ctx);                  /* the context's own (first) stream */
int nx_ctx_synchronize(nx_ctx* ctx);                /* both context streams */
/* Makes the first stream wait for all work queued on the second one (texture
 * passes and downloads issued with stream == NULL run there, overlapping the next
 * frame's collection pass). */
int nx_ctx_join(nx_ctx* ctx);

/* Stage timing (CUDA events recorded between the stages of each frame). */
#define NX_STAGE_PREPROCESS 0
#define NX_STAGE_DEPTH_SORT 1
#define NX_STAGE_EMIT 2
#define NX_STAGE_TILE_SORT 3
#define NX_STAGE_COMPOSITE 4
#define NX_STAGE_TEXTURE 5      /* the whole texture pass */
#define NX_STAGE_TEXTURE_MLP 6  /* its tensor-core decoder (0 on the fused / SIMT paths) */
#define NX_NUM_STAGES 7
int nx_ctx_set_profiling(nx_ctx* ctx, int enable);
/* Mean per-stage device time (ms per frame) over the profiled frames since the last
 * call, then resets; synchronises. Stage events bracket each stage on the stream. */
int nx_ctx_stage_times(nx_ctx* ctx, float* ms, int n, int* frames);
const char* nx_stage_name(int stage);
/* Number of kernels this library has launched (all contexts, host-side count). */
uint64_t nx_launch_count(void);

/* ---- scene (Scene, scene.hpp:25-32) ----------------------------------- */
/* nexels: n*60 doubles in Nexel field order (primitive.hpp:21-28): mu[3],
 * quat[4] (w,x,y,z), log_scale[2], opacity_raw, gamma_raw[2], sh[48].
 * table: levels * 2^log2_table * features doubles; w1 [hidden][levels*features],
 * w2 [hidden][hidden], w3 [48][hidden]. Validation of the primitives follows
 * activate() (primitive.cpp:47-63); a failure is recorded and reported by the
 * render calls (after settings/camera validation, as in collection_pass). */
int nx_scene_create(nx_ctx* ctx, const nx_settings* settings, int64_t n_nexels,
                    const double* nexels, const nx_field_desc* field, const double* table,
                    const double* w1, const double* w2, const double* w3, nx_scene** out);
int nx_scene_set_settings(nx_ctx* ctx, nx_scene* scene, const nx_settings* settings);
int nx_scene_get_settings(const nx_scene* scene, nx_settings* out);
void nx_scene_destroy(nx_scene* scene);

/* ---- NEXL checkpoints (checkpoint.hpp:19-28, checkpoint.cpp:173-271) --- */
/* Header facts of a checkpoint (CheckpointExtra + the scene's shape). */
typedef struct nx_nexl_info {
    uint64_t iteration;
    int64_t n_nexels;
    int32_t n_cameras;
    int32_t has_optimizer;   /* optimizer section present (skipped by the loader) */
    double extent;
    nx_settings settings;
    nx_field_desc field;
} nx_nexl_info;
/* load_checkpoint straight into a device scene: the fp32 SoA sections are read into
 * pinned staging and converted / uploaded on the device (positions & shape params to
 * the fp64 geometry layout, SH, table and MLP weights as stored). Validation and error
 * codes as the reference: missing-file, bad-checkpoint (magic, version, implausible
 * shapes, truncation), then bad-primitive at render time like nx_scene_create. */
int nx_scene_load_nexl(nx_ctx* ctx, const char* path, nx_scene** out, nx_nexl_info* info);
/* The training cameras stored in the checkpoint (CheckpointExtra::cameras); `names`
 * (nullable) receives up to 63 chars + NUL per camera. *n = number stored. */
int nx_nexl_cameras(const char* path, nx_camera* cams, char (*names)[64], int capacity, int* n);

/* ---- frames (FrameBuffers) -------------------------------------------- */
int nx_frame_create(nx_ctx* ctx, int width, int height, int top_k, nx_frame** out);
void nx_frame_destroy(nx_frame* frame);
int nx_frame_view_get(const nx_frame* frame, nx_frame_view* out);
/* Async device->host copy on `stream`; pinned destinations overlap with compute. */
int nx_frame_download(nx_ctx* ctx, const nx_frame* frame, const nx_host_frame* dst, void* stream);
/* Host->device: (re)shapes the frame and copies the given buffers (NULL = skip), e.g.
 * to run texturing_pass on FrameBuffers that a caller holds on the host. */
int nx_frame_upload(nx_ctx* ctx, nx_frame* frame, int width, int height, int top_k, const nx_host_frame* src,
                    void* stream);
int nx_frame_stats_get(nx_ctx* ctx, const nx_frame* frame, nx_frame_stats* out); /* synchronises */

/* ---- the render path --------------------------------------------------- */
/* collection_pass: binning, global (depth,id) order, front-to-back compositing with
 * early termination and top-K (renderer.cpp:115-171). The frame is (re)shaped to
 * the camera size and settings.top_k like FrameBuffers::allocate. */
int nx_collection_pass(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cam,
                       nx_frame* frame, void* stream);
/* texturing_pass: field queries at the buffered crossings + Eq. 7 composite
 * (renderer.cpp:207-237). Consumes the frame's ids/depths/weights/base. */
int nx_texturing_pass(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cam,
                      nx_frame* frame, void* stream);
/* render = collection_pass + texturing_pass (renderer.cpp:239-244). */
int nx_render(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cam, nx_frame* frame,
              void* stream);
/* A batch of views: cams[i] rendered into frames[i % n_frames],
 * pipelined as back-to-back nx_render calls; n_frames frames are in flight. */
int nx_render_views(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cams, int n_views,
                    nx_frame* const* frames, int n_frames, void* stream);

/* ---- render_backward (renderer.hpp:30-53, renderer.cpp:251-401) ------- */
/* UpstreamGrads (renderer.hpp:40-44): fp64 arrays in the FrameBuffers layouts; any
 * pointer may be NULL (treated as zero). */
typedef struct nx_upstream {
    const double* d_final;    /* H*W*3 */
    const double* d_weights;  /* H*W*K */
    const double* d_texture;  /* H*W*K*3 */
} nx_upstream;

/* SceneGrads (renderer.hpp:31-36) = PrimitiveGrad per nexel (primitive.hpp:53-62,
 * 60 doubles in Nexel field order: mu, quat, log_scale, opacity_raw, gamma_raw, sh)
 * + FieldGrads (texture_field.hpp:41-47: table [level][row][feature], w1, w2, w3).
 * All fp64; render_backward ACCUMULATES into them (+=) like the reference. */
typedef struct nx_grads {
    double* prims;   /* N*60 */
    double* table;   /* levels * 2^log2_table * features */
    double* w1;      /* hidden * levels*features */
    double* w2;      /* hidden * hidden */
    double* w3;      /* 48 * hidden */
} nx_grads;

/* Makes collection passes into `frame` keep the fp64 base the reverse pass needs
 * (3 doubles per pixel). Must be enabled before the forward that render_backward
 * differentiates. */
int nx_frame_set_backward(nx_ctx* ctx, nx_frame* frame, int enable);
/* render_backward: re-bins the scene for `cam` (as renderer.cpp:257 does), runs the
 * field branch (field_backward_batch, texture_field.cpp:77-146) at the buffered
 * crossings and the reverse compositing march, and accumulates into `grads`.
 * `frame` must be the unmodified forward output for scene/cam (with the backward
 * state kept). err_pixel (H*W, nullable) accumulates sum w * err_pixel into
 * blended_error (N, nullable) per primitive. Device pointers; asynchronous on
 * `stream`. Top-K membership is constant, as in the reference. */
int nx_render_backward(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cam, nx_frame* frame,
                       const nx_upstream* up, const nx_grads* grads, const double* err_pixel,
                       double* blended_error, void* stream);
/* Same with HOST arrays (copied in, accumulated, copied back; synchronous): the
 * binding for the reference-typed nexel::render_backward shim. */
int nx_render_backward_host(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cam, nx_frame* frame,
                            const nx_upstream* up, const nx_grads* grads, const double* err_pixel,
                            double* blended_error);

/* ---- losses_backward (losses.hpp:52-56, losses.cpp:107-238) ------------ */
/* LossWeights (losses.hpp:12-18). */
typedef struct nx_loss_weights {
    double dssim;    /* 0.2: blend inside the image term */
    double alpha;    /* 0.005 */
    double texture;  /* 0.5 */
    double opacity;  /* 0.01 */
    double grid;     /* 0.01 */
} nx_loss_weights;
/* LossTerms (losses.hpp:20-26). */
typedef struct nx_loss_terms {
    double l1, dssim, image, texture, alpha, opacity, grid, total;
} nx_loss_terms;
void nx_loss_weights_default(nx_loss_weights* out);
/* losses_backward: the image term (1-dssim) L1 + dssim (1-SSIM)/2 on final_img (11x11
 * Gaussian SSIM, ssim.cpp:99-151), the texture supervision and coverage terms on the
 * buffered slots, and the opacity / grid regularisers. Writes (overwrites) the upstream
 * gradients d_final (H*W*3), d_weights (H*W*K), d_texture (H*W*K*3) for
 * nx_render_backward and ACCUMULATES the direct parameter terms into grads->prims
 * (opacity_raw) and grads->table. gt: H*W*3 fp64. Device pointers; `terms` is a device
 * nx_loss_terms written asynchronously on `stream`. */
int nx_losses_backward(nx_ctx* ctx, const nx_scene* scene, const nx_frame* frame, const double* gt,
                       const nx_loss_weights* w, double* d_final, double* d_weights, double* d_texture,
                       const nx_grads* grads, nx_loss_terms* terms, void* stream);
/* Per-pixel error of the frame's final image against gt, err[p] = sum_c |final - gt| / 3
 * (trainer.cpp:288-295): the err_pixel render_backward spreads onto the primitives.
 * gt: H*W*3 fp64, err: H*W fp64, device pointers, on `stream`. */
int nx_pixel_error(nx_ctx* ctx, const nx_frame* frame, const double* gt, double* err, void* stream);
/* Same with HOST arrays and host `terms` (synchronous). */
int nx_losses_backward_host(nx_ctx* ctx, const nx_scene* scene, const nx_frame* frame, const double* gt,
                            const nx_loss_weights* w, double* d_final, double* d_weights, double* d_texture,
                            const nx_grads* grads, nx_loss_terms* terms);

/* ---- Adam on the device scene (adam.cpp:9-22, trainer.cpp:238-323) -------- */
/* AdamConfig (adam.hpp:8-13). */
typedef struct nx_adam_config {
    double lr, beta1, beta2, eps;
} nx_adam_config;
/* Parameter groups in the trainer's order (trainer.cpp:238-250, one AdamState each). */
#define NX_GROUP_POSITION 0
#define NX_GROUP_QUAT 1
#define NX_GROUP_SCALE 2
#define NX_GROUP_OPACITY 3
#define NX_GROUP_GAMMA 4
#define NX_GROUP_SH_DC 5
#define NX_GROUP_SH_REST 6
#define NX_GROUP_GRID 7
#define NX_GROUP_W1 8
#define NX_GROUP_W2 9
#define NX_GROUP_W3 10
#define NX_NUM_GROUPS 11
typedef struct nx_optimizer nx_optimizer;
/* fp64 first / second moments for every parameter of the scene, zeroed (step 0), and
 * fp64 master copies of the parameters the device scene stores in fp32 (SH, hash table,
 * MLP weights), initialised from the scene's fp32 values: Adam updates the masters in
 * fp64, like the reference's fp64 parameters, and refreshes the scene's fp32 copies. */
int nx_optimizer_create(nx_ctx* ctx, const nx_scene* scene, nx_optimizer** out);
/* Parameter count of a group (AdamState size once stepped). */
int nx_optimizer_size(const nx_optimizer* opt, int group, int64_t* count);
/* nx_losses_backward with the grid regulariser (losses.cpp:212-228) evaluated on the
 * optimizer's fp64 master of the hash table — the values being trained — instead of
 * the scene's fp32 render copy (what the trainer drop-in calls). opt may be NULL. */
int nx_losses_backward_opt(nx_ctx* ctx, const nx_scene* scene, const nx_frame* frame, const double* gt,
                           const nx_loss_weights* w, double* d_final, double* d_weights, double* d_texture,
                           const nx_grads* grads, nx_loss_terms* terms, const nx_optimizer* opt, void* stream);
/* Sets the fp64 master values of a group from HOST memory (count = its size, in the
 * group's row layout: per-nexel rows of the group's width, or the flat field block),
 * e.g. the exact fp64 initialisation the fp32 scene upload rounded. Geometry groups
 * (0..4) are fp64 in the scene already and are written there. Synchronous. */
int nx_optimizer_set_params(nx_ctx* ctx, nx_optimizer* opt, nx_scene* scene, int group, const double* host,
                            int64_t count);
/* Reads a group back to HOST memory (any NULL skipped): the fp64 parameter values
 * (masters / scene geometry) and the moments, in the group's row layout. Synchronous. */
int nx_optimizer_download(nx_ctx* ctx, const nx_optimizer* opt, const nx_scene* scene, int group, double* params,
                          double* m, double* v);
void nx_optimizer_destroy(nx_optimizer* opt);
/* One adam_step per group (cfg[NX_NUM_GROUPS]) on the device scene's parameters in
 * place, from device SceneGrads: per group step += 1, m/v EMAs, bias-corrected update.
 * Parameters the device stores in fp32 (SH, hash table, MLP weights) are updated on the
 * optimizer's fp64 masters, whose rounding refreshes the scene. lr == 0 steps the moments like adam_step; a group with lr < 0 is
 * skipped (its step does not advance). */
int nx_optimizer_step(nx_ctx* ctx, nx_optimizer* opt, nx_scene* scene, const nx_grads* grads,
                      const nx_adam_config* cfg, void* stream);
/* Per-group step counters (AdamState::step). */
int nx_optimizer_steps(const nx_optimizer* opt, int64_t* steps /* NX_NUM_GROUPS */);
/* Reads the device scene back in the reference's layouts (fp64 host arrays; any NULL
 * is skipped): 60 doubles per nexel, table, w1, w2, w3. */
int nx_scene_download(nx_ctx* ctx, const nx_scene* scene, double* nexels, double* table, double* w1, double* w2,
                      double* w3);

/* ---- density control (density.cpp:102-177, trainer.cpp:324-332) -------- */
/* prune: removes the nexels with sigmoid(opacity_raw) < min_opacity, keeping the
 * survivors' order; the optimizer's per-nexel rows follow (adam_remap_rows,
 * adam.cpp:24-42; opt may be NULL). new_to_old (device, capacity N, nullable) receives
 * the source row of each survivor; *n_out the new count. Synchronous. */
int nx_scene_prune(nx_ctx* ctx, nx_scene* scene, nx_optimizer* opt, double min_opacity, int32_t* new_to_old,
                   int64_t* n_out);
/* densify_split: splits min(ceil(split_fraction N), budget - N) distinct nexels sampled
 * without replacement with probability proportional to errors[i] (keys u_i^(1/e_i),
 * largest first, ties to the lower index), each parent replaced by two children along
 * its longest axis (the first reuses the parent's row, the second is appended). The
 * uniforms are the caller's draws, one per nexel in order — what the reference's
 * uniform_real_distribution<double>(0,1)(rng) yields — so the selection reproduces the
 * reference's. errors / uniforms: device, N doubles. new_to_old: device, capacity
 * N + splits (nullable). Synchronous. */
int nx_scene_densify_split(nx_ctx* ctx, nx_scene* scene, nx_optimizer* opt, const double* errors,
                           const double* uniforms, int64_t budget, double split_fraction, int32_t* new_to_old,
                           int64_t* n_out, int64_t* split_count);

/* ---- parity / debug (not on the timed path) ---------------------------- */
/* Tile lists for `cam`: reference_lists=1 materialises the reference's lists
 * (Binning::tile_lists, renderer.cpp:102-110, straddlers in every tile) on
 * settings.tile tiles; reference_lists=0 returns the work lists the composite
 * kernel walks (8x8-pixel tiles; *tiles_x, *tiles_y report the list geometry).
 * offsets: n_tiles+1 host ints; ids: `capacity` host ints; *total = keys. */
int nx_debug_tile_lists(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cam,
                        int reference_lists, int64_t* offsets, int32_t* ids,
                        int64_t capacity, int64_t* total, int32_t* tiles_x, int32_t* tiles_y);
/* Per-pixel contributor sequences (ids of every hit composited, in order, up to
 * termination) for image rows [y0, y1): hits[(row*W+x)*max_hits + i], counts[...]. */
int nx_debug_pixel_hits(nx_ctx* ctx, const nx_scene* scene, const nx_camera* cam, int y0,
                        int y1, int max_hits, int32_t* hits, int32_t* counts);

/* fp64 exp / log of the compositing kernels (table-driven, nx_fastmath.cuh) or CUDA's
 * library routines, on n host arguments (allocates, synchronises; parity tests only). */
enum { NX_FM_LOG = 0, NX_FM_EXP = 1, NX_FM_CUDA_LOG = 2, NX_FM_CUDA_EXP = 3,
       NX_FM_CERT = 4 /* quintuples (u, v, gx, gy, o) -> (alpha32, eps, oma32, eps_oma, alpha64) */ };
int nx_debug_fastmath(int fn, const double* x, double* y, int64_t n);
/* The binning primitives on n host elements (allocate, synchronise; parity tests only):
 * the stable LSD radix sort of (key, value) pairs over key bits [begin_bit, end_bit)
 * (key_bytes 4 or 8; keys / vals sorted in place), launched on a capacity cap >= n with
 * the count n on the device as the frame's sorts run; and the exclusive scan (total may
 * be NULL). */
int nx_debug_radix_sort(int key_bytes, void* keys, uint32_t* vals, int64_t n, int64_t cap, int begin_bit,
                        int end_bit);
int nx_debug_scan(const int32_t* in, int32_t* out, int64_t n, int64_t cap, int32_t* total);

/* ---- synthetic inputs -------------------- */
/* stump_like(N, c, seed, R_ground): fills nexels (n*60), settings and field desc;
 * table/w1/w2/w3 may be NULL to query sizes only (field desc is always filled). */
int nx_synth_stump_like(int64_t n, double coverage, uint64_t seed, double ground_radius,
                        int32_t log2_table, double grid_init, uint64_t field_seed,
                        double* nexels, nx_settings* settings, nx_field_desc* field,
                        double* table, double* w1, double* w2, double* w3);
int nx_synth_ring_camera(int index, int n_views, int width, int height, nx_camera* out);
void nx_settings_default(nx_settings* out);

#ifdef __cplusplus
}
#endif
#endif /* NEXEL_B200_H */
