/*
 * ngprt_cuda.h — C ABI of the B200-native NGP-RT per-ray renderer.
 *
 * This is the drop-in boundary for the reference's render path. The reference
 * (/root/reference/proj/include/ngprt, header-only C++20, CPU) exposes the path
 * as C++ value types, not as an FFI; each entry point below names the reference
 * interface it replaces:
 *
 *   ngprt_scene_desc / ngprt_scene_create  <- ngprt::BakedScene           baking.hpp:55-64
 *                                             (+ load_baked sections       baking.hpp:229-254,351-485)
 *   ngprt_camera                           <- PosedDataset + Frame::c2w   scene.hpp:191-201
 *   ngprt_render_opts                      <- march() arguments           occupancy.hpp:302-305
 *                                             + render CLI flags
 *   ngprt_render / ngprt_render_host       <- render_ray (specified, never implemented)
 *                                             SPEC.md:309-317, composed from generate_rays
 *                                             scene.hpp:211-228, march occupancy.hpp:302-326,
 *                                             decode_point_baked baking.hpp:84-91,
 *                                             composite volume.hpp:51-75, shade volume.hpp:118-137
 *   ngprt_ray_stats                        <- MarchCounters               occupancy.hpp:197-210
 *   ngprt_build_pyramid                    <- build_pyramid               occupancy.hpp:114-119
 *   ngprt_build_distance_grid              <- build_distance_grid         occupancy.hpp:136-194
 *   ngprt_last_error                       <- the exception text the reference throws
 *
 * Conventions: plain pointers and sizes only; no C++ or torch types; no
 * exceptions cross this boundary. Every call returns an ngprt_status and
 * leaves a thread-local message for ngprt_last_error(). Host inputs are copied
 * at scene creation; the scene is immutable afterwards and may be rendered
 * concurrently on different streams.
 */
#ifndef NGPRT_CUDA_H
#define NGPRT_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NGPRT_ABI_VERSION 2
#define NGPRT_MAX_FINE_LEVELS 4 /* kMaxFineLevels, fusion.hpp:33 */
#define NGPRT_PYRAMID_LEVELS 5  /* kPyramidLevels, occupancy.hpp:104 */

typedef enum {
    NGPRT_OK = 0,
    NGPRT_EINVAL = 1,       /* std::invalid_argument / std::domain_error / out_of_range */
    NGPRT_ECUDA = 2,        /* CUDA runtime failure (message carries cudaGetErrorString) */
    NGPRT_ENOMEM = 3,       /* device allocation failed */
    NGPRT_EUNSUPPORTED = 4, /* valid in the reference, not implemented here (message says what) */
    NGPRT_ENODEV = 5,       /* no CUDA device / not an sm_100 device */
    NGPRT_ENCCL = 6         /* NCCL failure in the multi-device calls (message carries ncclGetErrorString) */
} ngprt_status;

/* FusionTag, fusion.hpp:44-51 (same numeric values as the .ngrt header byte). */
typedef enum {
    NGPRT_FUSION_SUM = 0,
    NGPRT_FUSION_SHARED_ATT_INV = 1,
    NGPRT_FUSION_SEPARATE_ATT_INV = 2,
    NGPRT_FUSION_SHARED_ATT_V = 3,
    NGPRT_FUSION_SEPARATE_ATT_V = 4,
    NGPRT_FUSION_MLP = 5 /* ablation (PAPER Table 3): fine features through an {8L,64,8} MLP */
} ngprt_fusion_tag;

/* How feature rows are stored in HBM. AUTO picks fp16 when every coarse row
 * and fine-table value survives an f32->f16->f32 round trip (lossless, so the
 * render stays bit-exact), else f32. F16 forced on values that are not
 * fp16-exact is an opt-in LOSSY mode (round to nearest): on the f32 config-3
 * scene it renders 1.38x faster than F32 with RGB max-abs 4.4e-4 (<= 1e-3,
 * PSNR 93 dB), and ~0.1 % of rays change their counters (early stop moves);
 * tests/test_gpu_parity.py::test_forced_fp16_storage_is_within_tolerance. */
typedef enum { NGPRT_STORAGE_AUTO = 0, NGPRT_STORAGE_F32 = 1, NGPRT_STORAGE_F16 = 2 } ngprt_storage;

/* Deferred MLP (shade, volume.hpp:118-137) implementation.
 * EXACT  : f32 CUDA-core forward in the reference's operation order -> bit-exact RGB.
 * TENSOR : tcgen05.mma (fp16 split-precision operands, f32 TMEM accumulators) -> RGB
 *          within 1e-3 of the reference (north_star tolerance). Default. */
typedef enum { NGPRT_MLP_TENSOR = 0, NGPRT_MLP_EXACT = 1 } ngprt_mlp_mode;

/* POD view of a BakedScene (baking.hpp:55-64). All pointers are HOST pointers,
 * copied by ngprt_scene_create. */
typedef struct ngprt_scene_desc {
    uint32_t L;                                  /* EncodingConfig::fine_levels (1..4)       */
    uint32_t L_C;                                /* EncodingConfig::corner_grid_res          */
    uint32_t fine_res[NGPRT_MAX_FINE_LEVELS];    /* HashLevel::resolution (1024 << l)         */
    uint64_t fine_table_len[NGPRT_MAX_FINE_LEVELS]; /* HashLevel::table_len                  */
    uint8_t fine_hashed[NGPRT_MAX_FINE_LEVELS];  /* HashLevel::addressing (0 direct, 1 hash) */
    uint8_t fusion_tag;                          /* ngprt_fusion_tag                          */
    uint8_t storage;                             /* ngprt_storage                             */
    uint8_t reserved[2];
    uint64_t n_coarse;                           /* SparseCoarseGrid::count()                 */
    const uint64_t* coarse_keys;                 /* key_of(corner), any order, unique         */
    const float* coarse_rows;                    /* n_coarse x (8+2L) f32                     */
    const float* fine_tables[NGPRT_MAX_FINE_LEVELS]; /* table_len x 8 f32, row-major          */
    const float* psi_w[3];                       /* TinyMlp 23->64->64->3, row-major out x in */
    const float* psi_b[3];
    const float* att_globals;                    /* FusionMode::global_pre, 2L (Inv modes)    */
    uint32_t occ_base_res;                       /* pyramid.levels[0].res                     */
    uint32_t dist_res;                           /* DistanceGrid::resolution; 0 = no grid     */
    const uint64_t* pyramid_words[NGPRT_PYRAMID_LEVELS]; /* [0] required; [1..4] NULL => built on device */
    const uint8_t* dist_values;                  /* dist_res^3, NULL => built on device from the
                                                    pyramid level whose res == dist_res       */
    const float* fusion_mlp_w[2];                /* FusionMode::mlp {8L, 64, 8} (MLP mode only): */
    const float* fusion_mlp_b[2];                /* W0 64 x 8L, b0 64, W1 8 x 64, b1 8       */
} ngprt_scene_desc;

/* Pinhole camera: PosedDataset intrinsics + one Frame (scene.hpp:191-201).
 * c2w is row-major 4x4 camera-to-world (x right, y down, z forward). */
typedef struct ngprt_camera {
    double c2w[16];
    double fx, fy, cx, cy;
    uint32_t width, height;
} ngprt_camera;

typedef struct ngprt_render_opts {
    float step;            /* march step gamma*s0; <= 0 => kBaseStep = 2*sqrt(3)/512 (config.hpp:11) */
    uint8_t use_dist_grid; /* pass &distance (1) or nullptr (0) to march()                 */
    uint8_t max_step_rule; /* occupancy.hpp:272                                             */
    uint8_t early_stop;    /* T < 2e-3 termination (volume.hpp:36,70)                       */
    int8_t keep_level;     /* 0 = off; 1..L = level_masked_fine(keep_level) (fusion.hpp:198-209) */
    uint8_t mlp_mode;      /* ngprt_mlp_mode                                                */
    uint8_t profile;       /* record CUDA events around each kernel (ngprt_render_timing)  */
    uint8_t reserved[2];
    uint32_t x0, y0, w, h; /* pixel window; w == 0 || h == 0 => full frame. Output is w x h. */
    /* Interleaved-tile sharding of the window over `shard_world` renderers
     * (SURVEY.md §8(e)): the window is cut into shard_tile x shard_tile pixel
     * tiles, row-major, and tile T belongs to rank T % shard_world. With
     * shard_world >= 1 one call renders only this rank's tiles (one K0/K1/K2
     * launch) into a COMPACT output: per camera ngprt_shard_pixels(w, h,
     * shard_world, shard_tile) pixels, local tile j (global tile rank + j *
     * shard_world) at j * shard_tile^2, row-major inside the tile; pixels past
     * the window edge (and a rank's missing last tile) are black. Every rank's
     * buffer has the same size, so an all-gather / gather needs no padding step;
     * ngprt_shard_assemble rebuilds the frames. shard_world 0 = unsharded (row-major window); 1 = every tile, in tile-major order. */
    uint32_t shard_world, shard_rank;
    uint32_t shard_tile;   /* multiple of 8 (K1's 4x8 ray tiles); 0 => 32 */
    uint32_t reserved2;
} ngprt_render_opts;

/* MarchCounters (occupancy.hpp:197-210), per ray. */
typedef struct ngprt_ray_stats {
    uint32_t marching;
    uint32_t occupied;
    uint32_t occ_acc;
    uint32_t dist_acc;
} ngprt_ray_stats;

typedef struct ngprt_scene ngprt_scene; /* opaque; owns device memory */

typedef struct ngprt_scene_info {
    int device;
    uint8_t storage;          /* resolved ngprt_storage (F32 or F16) */
    uint8_t reserved[3];
    uint32_t coarse_row_stride; /* elements per stored coarse row */
    uint64_t device_bytes;    /* total device memory owned by the scene */
    uint64_t coarse_bytes, fine_bytes, pyramid_bytes, dist_bytes;
    const void* dev_pyramid[NGPRT_PYRAMID_LEVELS]; /* device pointers (u64 words) */
    const void* dev_dist;                          /* device pointer (u8), NULL if none */
} ngprt_scene_info;

int ngprt_abi_version(void);
const char* ngprt_last_error(void);

/* Scene lifetime (replaces constructing / load_baked-ing a BakedScene). */
ngprt_status ngprt_scene_create(const ngprt_scene_desc* desc, int device, ngprt_scene** out);
void ngprt_scene_destroy(ngprt_scene* scene);
ngprt_status ngprt_scene_info_get(const ngprt_scene* scene, ngprt_scene_info* info);

/* Render n_cams frames. rgb_dev: n_cams x h x w x 3 f32 (Image::rgb layout per
 * frame, image.hpp:12-22); stats_dev: n_cams x h x w (nullable). Device
 * pointers, asynchronous on `stream` (cudaStream_t, NULL = legacy default).
 * A frame (window) of 2^31 pixels or more is NGPRT_EINVAL. */
ngprt_status ngprt_render(const ngprt_scene* scene, const ngprt_camera* cams, int n_cams,
                          const ngprt_render_opts* opts, float* rgb_dev,
                          ngprt_ray_stats* stats_dev, void* stream);

/* Same with HOST buffers: copies cameras in and rgb/stats out, synchronous.
 * This is the call that replaces a host-side render(BakedScene, PosedDataset, frame). */
ngprt_status ngprt_render_host(const ngprt_scene* scene, const ngprt_camera* cams, int n_cams,
                               const ngprt_render_opts* opts, float* rgb_host,
                               ngprt_ray_stats* stats_host);

/* Pipelined host-buffer rendering for a stream of frames (serving). Same
 * arguments as ngprt_render_host, but returns once the frame is enqueued: it is
 * rendered into a device buffer and copied to rgb_host / stats_host by the copy
 * engine while the NEXT enqueued frame renders, so the device->host transfer
 * overlaps the march. At most two frames are in flight per scene (enqueueing a
 * third waits for the oldest). Host buffers must stay valid, and should be
 * pinned for the copy to be asynchronous, until ngprt_render_host_wait returns. */
ngprt_status ngprt_render_host_async(const ngprt_scene* scene, const ngprt_camera* cams,
                                     int n_cams, const ngprt_render_opts* opts, float* rgb_host,
                                     ngprt_ray_stats* stats_host);
/* Blocks until every frame enqueued with ngprt_render_host_async is in host memory. */
ngprt_status ngprt_render_host_wait(const ngprt_scene* scene);

/* Interleaved-tile sharding (ngprt_render_opts.shard_*): pixels per camera in
 * every rank's compact output, ceil(n_tiles / world) * tile^2 with n_tiles =
 * ceil(w / tile) * ceil(h / tile) (tile 0 => 32, world 0 => 1). */
uint64_t ngprt_shard_pixels(uint32_t w, uint32_t h, uint32_t world, uint32_t tile);
/* De-interleave gathered shard outputs into frames (device pointers, async):
 * shards = world consecutive rank buffers, each n_cams x ngprt_shard_pixels(w,
 * h, world, tile) x `channels` floats (rank-major, as an all-gather / gather to
 * one device lays them out); frames = n_cams x h x w x channels. channels = 3
 * for RGB, 4 for ngprt_ray_stats viewed as u32 words. */
ngprt_status ngprt_shard_assemble(const float* shards_dev, uint32_t world, uint32_t n_cams,
                                  uint32_t w, uint32_t h, uint32_t tile, uint32_t channels,
                                  float* frames_dev, void* stream);

/* ---------------------------------------------------------------------------
 * Multi-device rendering in ONE process: a scene replica per
 * device, one NCCL communicator per device (ncclCommInitAll), one stream per
 * device. Rays are independent and the scenes read-only, so the only exchange
 * is the gather of finished pixels to devices[0] (grouped ncclSend/ncclRecv on
 * the render streams). NCCL is loaded at run time (libnccl.so.2); a missing
 * library or an NCCL error is NGPRT_ENCCL. When `devices` repeats a device
 * (several replicas on one GPU: a functional configuration, not a fast one)
 * the gather uses device-to-device copies instead of NCCL.
 * ------------------------------------------------------------------------- */
typedef struct ngprt_multi ngprt_multi;
ngprt_status ngprt_multi_create(const ngprt_scene_desc* desc, const int* devices, int n_dev,
                                ngprt_multi** out);
void ngprt_multi_destroy(ngprt_multi* m);
/* 1 when the gather runs over NCCL, 0 when over peer copies (repeated devices). */
int ngprt_multi_uses_nccl(const ngprt_multi* m);
/* The replica on devices[i] (owned by m), e.g. for ngprt_scene_info_get. */
const ngprt_scene* ngprt_multi_scene(const ngprt_multi* m, int i);
/* One frame per camera, each cut into interleaved tile x tile tiles shared by
 * all devices (one K0/K1/K2 launch per device per call), gathered to
 * devices[0] and de-interleaved there into rgb_dev0 (n_cams x h x w x 3, a
 * devices[0] pointer; stats_dev0 likewise n_cams x h x w, nullable). Enqueued
 * on stream0 (devices[0]); the other devices run on internal streams ordered
 * after stream0's prior work. opts->shard_* are ignored (set by the call). */
ngprt_status ngprt_multi_render_tiles(ngprt_multi* m, const ngprt_camera* cams, int n_cams,
                                      const ngprt_render_opts* opts, uint32_t tile,
                                      float* rgb_dev0, ngprt_ray_stats* stats_dev0, void* stream0);
/* Camera sharding: camera c rendered whole by device c % n_dev, gathered to
 * devices[0] into rgb_dev0 (n_cams x h x w x 3; stats_dev0 nullable). */
ngprt_status ngprt_multi_render_cameras(ngprt_multi* m, const ngprt_camera* cams, int n_cams,
                                        const ngprt_render_opts* opts, float* rgb_dev0,
                                        ngprt_ray_stats* stats_dev0, void* stream0);

/* Per-kernel device time of the most recent ngprt_render on this scene with
 * opts.profile set: CUDA events recorded on the render stream around the march
 * kernel (K1) and the deferred-MLP kernel (K2), summed over launches; n_launches
 * counts every kernel of the render (K0, K1, K2 per batch of up to 64 cameras).
 * Call after synchronising that stream. Single-stream benchmarking aid. */
ngprt_status ngprt_render_timing(const ngprt_scene* scene, float* ms_march, float* ms_shade,
                                 int* n_launches);
/* The same with the ray-generation kernel (K0) timed separately. */
ngprt_status ngprt_render_timing3(const ngprt_scene* scene, float* ms_raygen, float* ms_march,
                                  float* ms_shade, int* n_launches);

/* Occupancy structures on device (device pointers, async on stream).
 * levels_dev[k-1] receives level k (res base>>k), k = 1..4, u64 words x-fastest. */
ngprt_status ngprt_build_pyramid(const uint64_t* base_words_dev, uint32_t base_res,
                                 uint64_t* const levels_dev[NGPRT_PYRAMID_LEVELS - 1],
                                 void* stream);
/* out_dev: res^3 u8, G = min(255, max(0, D_cheb - 1)). scratch-free (in-place u8 passes). */
ngprt_status ngprt_build_distance_grid(const uint64_t* occ_words_dev, uint32_t res,
                                       uint8_t* out_dev, void* stream);

/* Test hooks (device pointers): the device port of glibc expf, and the fine-level
 * row index (HashLevel::hash_index, hash_grid.hpp:83-94) for corner triples. */
ngprt_status ngprt_test_expf(const float* x_dev, float* y_dev, uint64_t n, void* stream);
ngprt_status ngprt_test_expf_range(uint32_t first_bits, uint64_t n, uint32_t* y_bits_dev,
                                   void* stream);
/* The K1 marcher (same device code path) over n_rays given rays (8 f32 each:
 * origin, dir, t_near, t_far; device pointers) with emit(t) always continuing:
 * records each ray's empty-skip segments (t, t + s) and occupied sample t's, as
 * the reference's march(..., skip_segments) does (occupancy.hpp:302-326), for the
 * skip-safety check against dda_oracle. seg: n_rays x max_seg x 2,
 * samples: n_rays x max_seg, n_seg / n_samples: full counts (may exceed max_seg),
 * counters: n_rays x 4 (MarchCounters). */
ngprt_status ngprt_test_march_segments(const ngprt_scene* scene, const float* rays8_dev,
                                       int n_rays, float step, int use_grid, int max_step_rule,
                                       int max_seg, float* seg_dev, int* n_seg_dev,
                                       float* samples_dev, int* n_samples_dev,
                                       uint32_t* counters_dev, void* stream);
ngprt_status ngprt_test_hash_index(const int32_t* corners_dev, uint64_t n, uint32_t res,
                                   uint64_t table_len, uint8_t hashed, uint64_t* out_dev,
                                   void* stream);

/* ---------------------------------------------------------------------------
 * The reference's baked-scene file (".ngrt", baking.hpp:229-485): magic "NGRT",
 * version 1, header {L_C, L, fine_res[L], table_lens[6+L], fusion tag}, then
 * CRC-32-checked sections 1 coarse map, 2 fine tables, 3 view MLP, 4 pyramid
 * (512..32), 5 distance grid (256^3), 6 attention logits, 7 fusion MLP.
 * ngprt_baked_load parses and validates on the host (errors carry the
 * reference's messages and byte offsets); ngprt_scene_load uploads in one call.
 * ------------------------------------------------------------------------- */
typedef struct ngprt_baked ngprt_baked;
ngprt_status ngprt_baked_load(const char* path, ngprt_baked** out);
const ngprt_scene_desc* ngprt_baked_desc(const ngprt_baked* b);
void ngprt_baked_free(ngprt_baked* b);
ngprt_status ngprt_scene_load(const char* path, int device, ngprt_scene** out);

/* Writes an ngprt_baked in the reference's format (save_baked, baking.hpp:266-349).
 * Pyramid must be 512-based with a 256^3 distance grid, as the format fixes. */
ngprt_status ngprt_baked_save(const ngprt_baked* b, const char* path);

/* ---------------------------------------------------------------------------
 * Bake (baking.hpp:107-202): a trained NgpRtModel (model.hpp:27-107) plus its
 * training occupancy -> the render-time BakedScene, on the GPU:
 *   density cull of the training voxels with the live decode (decode_point,
 *   model.hpp:195-239), dilation, upsampling to the 512 render grid, pyramid
 *   and distance grid (K3/K4), corner retention on the L_C grid, and corner
 *   evaluation (evaluate_corner, model.hpp:71-87: six coarse hash levels through
 *   the aux MLP 24 -> 64 -> 8+2L), all in the reference's f32 operation order.
 * ------------------------------------------------------------------------- */
typedef struct ngprt_model_desc {
    uint32_t L, L_C;
    uint32_t coarse_res[6];                      /* EncodingConfig::coarse_resolutions     */
    uint64_t coarse_table_len;                   /* max table length of a coarse level      */
    const float* coarse_tables[6];               /* min((res+1)^3, len) x 4 each            */
    const float* aux_w[2];                       /* TinyMlp 24 -> 64 -> 8+2L (out x in)      */
    const float* aux_b[2];
    uint32_t fine_res[NGPRT_MAX_FINE_LEVELS];
    uint64_t fine_table_len[NGPRT_MAX_FINE_LEVELS];
    uint8_t fine_hashed[NGPRT_MAX_FINE_LEVELS];
    const float* fine_tables[NGPRT_MAX_FINE_LEVELS];
    const float* psi_w[3];
    const float* psi_b[3];
    uint8_t fusion_tag;
    uint8_t reserved[7];
    const float* att_globals;
    const float* fusion_mlp_w[2];
    const float* fusion_mlp_b[2];
} ngprt_model_desc;

typedef struct ngprt_bake_opts {   /* BakeOptions, baking.hpp:93-97 */
    double cull_step;              /* <= 0 => kBaseStep                */
    double cull_alpha_thresh;      /* 0.005                            */
    uint32_t dilate_voxels;        /* 1                                */
    uint32_t reserved;
} ngprt_bake_opts;

ngprt_status ngprt_bake(const ngprt_model_desc* model, const uint64_t* train_words,
                        uint32_t train_res, const ngprt_bake_opts* opts, int device,
                        ngprt_baked** out);

/* ---------------------------------------------------------------------------
 * Synthetic scenes (host-only input generation). Restates the reference's own
 * generators so the GPU and the CPU oracle consume the same scene object:
 * make_scene/scene_occupancy (scene.hpp:168-183,329-385), Rng (common.hpp:46-75),
 * TinyMlp::init (nn.hpp:154-173), sphere_views (scene.hpp:254-265).
 * ------------------------------------------------------------------------- */
typedef struct ngprt_synth_params {
    char occupancy[32];     /* "bench" | "toy" | "slab" (make_scene presets) | "blob" |
                               "mip360" | "boxes" */
    uint64_t scene_seed;    /* make_scene seed (41) */
    uint32_t n_boxes;       /* "boxes" preset only */
    uint32_t occ_base_res;  /* pyramid base resolution (512 / 256) */
    uint32_t dist_level;    /* distance grid built from pyramid.levels[dist_level] (1); 5 = none */
    uint32_t L;             /* fine levels */
    uint32_t L_C;           /* corner grid resolution */
    uint32_t fusion_tag;
    uint64_t fine_table_len;
    uint64_t table_seed;    /* fine tables, Rng(7) */
    uint64_t coarse_seed;   /* coarse rows, Rng(13) */
    uint64_t psi_seed;      /* psi init, Rng(11) */
    double sigma_lo, sigma_hi;  /* coarse sigma_pre ~ U[lo,hi] */
    double feat_scale;          /* fine-table and coarse colour channels ~ U[-s,s] */
    double att_scale;           /* attention logits ~ U[-a,a] */
    double psi_bias_scale;      /* 0 => zero biases (TinyMlp::init); else U[-b,b] */
    uint8_t fp16_exact;         /* round every value to an fp16-representable f32 */
    uint8_t reserved[7];
} ngprt_synth_params;

typedef struct ngprt_synth ngprt_synth;

void ngprt_synth_default_params(ngprt_synth_params* p);
ngprt_status ngprt_synth_create(const ngprt_synth_params* p, ngprt_synth** out);
const char* ngprt_synth_last_error(void);
/* The desc points into memory owned by the synth object (valid until destroy). */
const ngprt_scene_desc* ngprt_synth_desc(const ngprt_synth* s);
void ngprt_synth_destroy(ngprt_synth* s);
/* A seeded synthetic NgpRtModel (the bake input): coarse hash levels {16..512}
 * ~ U[-feat_scale, feat_scale], aux/psi/fusion MLPs via TinyMlp::init
 * (nn.hpp:154-173), fine tables as for scenes, plus a training occupancy grid
 * scene_occupancy(make_scene(occupancy), occ_base_res) (training resolution). */
typedef struct ngprt_synth_model ngprt_synth_model;
ngprt_status ngprt_synth_model_create(const ngprt_synth_params* p, ngprt_synth_model** out);
const ngprt_model_desc* ngprt_synth_model_desc(const ngprt_synth_model* m);
const uint64_t* ngprt_synth_model_train_words(const ngprt_synth_model* m, uint32_t* train_res);
void ngprt_synth_model_destroy(ngprt_synth_model* m);

/* sphere_views(n, radius) with fx = fy = 1.1 W, cx = W/2, cy = H/2 (scene.hpp:388-395). */
ngprt_status ngprt_synth_cameras(int n, double radius, uint32_t width, uint32_t height,
                                 ngprt_camera* out);
/* Host-side helpers exposed for the tests: CRC-32 (common.hpp:78-92) and the
 * splitmix64 uniform stream (common.hpp:46-60). */
uint32_t ngprt_crc32(const void* data, uint64_t len, uint32_t seed);
void ngprt_rng_uniform(uint64_t seed, double lo, double hi, uint64_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* NGPRT_CUDA_H */
