/*
 * sf_gpu.h — C-ABI boundary of the B200-native sparse-TSDF hot path.
 *
 * Drop-in for the reference library "sparsefusion" (/root/reference/proj). Every entry
 * point below replaces one reference C++ interface (cited as file:line, relative to
 * /root/reference/proj). Plain C types only: opaque handles, plain pointers and sizes,
 * int status codes plus a thread-local message (sf_last_error). No CUDA, torch or Eigen
 * types appear in the signatures; `stream` is a cudaStream_t passed as void* (NULL =
 * the legacy default stream).
 *
 * Conventions
 *   - Poses are `double pose[12]`: rotation row-major R[r*3+c] in pose[0..8], translation
 *     in pose[9..11]; camera -> world, x_w = R x_c + t (include/sparsefusion/pose.hpp:9-16).
 *   - Depth frames are row-major float, 0 = invalid, optional per-pixel sigma plane
 *     (include/sparsefusion/camera.hpp:45-63). Normal maps are float xyz per pixel, zero =
 *     invalid (camera.hpp:67-78).
 *   - Frame/output pointers may be host or device memory, flagged per call. Host pointers
 *     are staged through the volume's device buffers on `stream`.
 *   - Calls that return statistics synchronise `stream`; the *_async variants do not.
 *   - A volume handle is not thread-safe (mirrors grid.hpp:93-95: single writer).
 *   - Numerics follow the reference bit-for-bit (FP64, no contraction, same operation
 *     order). The only non-bitwise stage is the ICP reduction order
 *     (compensated sums merged in a tree; pose parity 1e-6).
 */
#ifndef SF_GPU_H
#define SF_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (reference exception types) ------------------------ */
typedef enum {
    SF_OK = 0,
    SF_INVALID_ARGUMENT = 1, /* std::invalid_argument  (grid.cpp:14-17, fusion.cpp:12-16, ...) */
    SF_OUT_OF_RANGE = 2,     /* std::out_of_range      (grid.cpp:83,122,133)                   */
    SF_LOGIC_ERROR = 3,      /* std::logic_error       (grid.cpp:139)                          */
    SF_POOL_EXHAUSTED = 4,   /* PoolExhausted          (grid.hpp:24-26, grid.cpp:90-92)        */
    SF_TRACKING_LOST = 5,    /* TrackingLost           (registration.hpp:18-20, .cpp:202-204)  */
    SF_CUDA_ERROR = 6,
    SF_IO_ERROR = 7,         /* std::runtime_error from snapshot I/O (grid.cpp:333-408)        */
    SF_UNSUPPORTED = 8       /* option not implemented on the device path (fails loudly)      */
} sf_status;

/* Message of the last failing call on this thread ("" if none). */
const char* sf_last_error(void);
/* Library/ABI version, e.g. "sf_gpu 0.1 sm_100a". */
const char* sf_version(void);

/* ---- plain data (mirrors of the reference structs) ---------------------------------- */

/* GridConfig (grid.hpp:28-40). truncation <= 0 -> 4 * voxel_size. */
typedef struct {
    int32_t blocks_per_axis;       /* N */
    int32_t voxels_per_block_axis; /* M */
    double box_origin[3];
    double box_side;
    double truncation;
} sf_grid_config;

/* AuxQuantization (grid.hpp:53-63). mode 0 = Weight, 1 = Variance. */
typedef struct {
    int32_t mode;
    double w_max;
    double p_min;
    double p_max;
} sf_aux_quant;

/* Intrinsics (camera.hpp:9-24). */
typedef struct {
    int32_t width;
    int32_t height;
    double fx, fy, cx, cy;
    double near_plane, far_plane;
} sf_intrinsics;

/* DepthFrame (camera.hpp:45-63). sigma may be NULL (no recorded sigma plane). */
typedef struct {
    sf_intrinsics intrinsics;
    const float* depth; /* width*height */
    const float* sigma; /* width*height or NULL */
    int32_t on_device;  /* 1: device pointers; 0: host pointers */
} sf_frame;

/* FusionParams (fusion.hpp:18-31). mode 0 Simple, 1 Weighted, 2 Kalman. */
typedef struct {
    int32_t mode;
    double w_fixed;
    double w_max;
    double process_variance; /* < 0 -> (0.1 * delta / 127)^2 (fusion.cpp:19-23) */
    double sigma0;
    double delta; /* ignored: taken from the grid (fusion.cpp:278) */
    int32_t refinement_steps;
    int32_t edge_downweight;
    double min_variance;
} sf_fusion_params;

/* FusionStats (fusion.hpp:93-98). */
typedef struct {
    uint64_t voxels_updated;
    uint64_t blocks_allocated_now;
    uint64_t blocks_total;
    uint64_t memory_bytes;
} sf_fusion_stats;

/* RaycastStats (render.hpp:41-49). */
typedef struct {
    uint64_t sample_steps;
    uint64_t hit_pixels;
    uint64_t rays_with_bounds;
} sf_raycast_stats;

/* MatchParams (registration.hpp:22-34) incl. its NormalOptions (camera.hpp:77-80). */
typedef struct {
    double max_distance;
    double max_normal_angle;
    int32_t max_iterations;
    double convergence_epsilon;
    double eigen_threshold;
    double shrink_floor;
    double normal_sigma0;
    double normal_spatial_scale;
    /* Not in the reference struct: the order of the normal-equation sums.
     * 0 (default): tree-reduced compensated sums in unshrunk form (one launch per iteration);
     *    the pose equals the reference's to ~1e-15 per call.
     * 1: the reference's order (registration.cpp:52-123): matches compacted in row-major order,
     *    shrunk per match, 28 sequential Kahan sums, cyclic Jacobi, spectral gated solve and
     *    the SVD apply_motion — bit-identical poses, so a tracked sequence stays bit-identical
     *    to the reference frame after frame (slower: the Kahan chains are sequential). */
    int32_t reduction;
} sf_match_params;

/* IcpResult + GatedSolution (registration.hpp:68-83). */
typedef struct {
    double delta[12];
    int32_t iterations;
    uint64_t matches;
    /* GatedSolution of the last iteration */
    double motion_r[3];
    double motion_t[3];
    double eigenvalues[6];   /* ascending */
    double eigenvectors[36]; /* column-major: eigenvectors[col*6 + row] */
    int32_t gated_mask[6];
    double residual_rms;
    double shrunk_motion_norm;
    uint64_t pair_count;
} sf_icp_result;

/* Volume summary (grid.hpp:103-108, 132-133). */
typedef struct {
    sf_grid_config config;
    sf_aux_quant aux;
    double delta;
    double voxel_size;
    uint64_t pool_capacity;
    uint64_t allocated_count;
    uint64_t memory_bytes;
} sf_volume_info;

/* ---- volume lifecycle: SparseTsdfGrid (grid.hpp:96-193) ------------------------------ */
typedef struct sf_volume* sf_volume_t;

/* SparseTsdfGrid::SparseTsdfGrid(config, pool_capacity = 0, aux) (grid.hpp:100-101,
 * grid.cpp:53-72). pool_capacity 0 -> max(1, N^3/8). aux may be NULL (defaults). */
int sf_volume_create(const sf_grid_config* config, uint64_t pool_capacity, const sf_aux_quant* aux,
                     int32_t device, sf_volume_t* out);
int sf_volume_destroy(sf_volume_t vol);
int sf_volume_get_info(sf_volume_t vol, sf_volume_info* out);

/* ---- DFRM depth frames (frame_io.hpp:15-16, frame_io.cpp:28-79) ------------------------
 * write: the reference's byte layout; frame buffers may be host or device (frame->on_device).
 * read: depth == NULL only fills *intrinsics (size query); out-of-range depths become 0. */
int sf_dfrm_write(const char* path, const sf_frame* frame);
int sf_dfrm_read(const char* path, sf_intrinsics* intrinsics, float* depth, float* sigma, int32_t* has_sigma,
                 int32_t out_on_device);

/* ---- trajectory CSV (frame_io.hpp:18-28, frame_io.cpp:81-126) -------------------------
 * Rows "frame_index,r00,...,r22,t0,t1,t2" printed with 17 significant digits (byte-identical
 * to write_trajectory). read: 12 or 13 values per row ('#' lines and empty lines skipped; no
 * frame index -> 0); a rotation that is not orthonormal within 1e-6 is replaced by its nearest
 * rotation, as parse_trajectory_row does. frame_index / poses12 NULL: *count = rows (size
 * query); otherwise *count is the capacity in and the row count out. */
int sf_trajectory_write(const char* path, const int32_t* frame_index, const double* poses12, uint64_t count);
int sf_trajectory_read(const char* path, int32_t* frame_index, double* poses12, uint64_t* count);

/* ---- marching cubes (marching_cubes.hpp:37-44, marching_cubes.cpp:74-196) -----------
 * The reference's mesh exactly: same vertices (float, welded per batch by cube-edge id in
 * first-reference order), normals and triangles. region_pose / region_intrinsics: optional
 * FrustumRegion (both or neither); batch_memory_budget: MarchingCubesOptions (0 = 64 MiB).
 * The mesh lives on the device until sf_mesh_read (triangles as 3 x uint32). */
typedef struct sf_mesh* sf_mesh_t;
int sf_marching_cubes(sf_volume_t vol, const double region_pose[12], const sf_intrinsics* region_intrinsics,
                      uint64_t batch_memory_budget, sf_mesh_t* out, void* stream);
int sf_mesh_counts(sf_mesh_t mesh, uint64_t* vertices, uint64_t* triangles);
int sf_mesh_read(sf_mesh_t mesh, float* vertices_xyz, float* normals_xyz, uint32_t* triangles,
                 int32_t out_on_device, void* stream);
int sf_mesh_destroy(sf_mesh_t mesh);

/* ---- spatial sharding across GPUs --------------------
 * No reference counterpart: the reference volume is one process. A sharded volume
 * allocates only the blocks its rank owns: owner(block) = hash of its (2^brick_shift)^3-block
 * brick % world (sf_shard_owner). Call on an empty volume. Integrating the same frame on
 * every rank's volume yields, over the union of ranks, exactly the single volume's blocks
 * and payloads. */
int sf_volume_set_shard(sf_volume_t vol, int32_t rank, int32_t world, int32_t brick_shift);
int32_t sf_shard_owner(int32_t bx, int32_t by, int32_t bz, int32_t brick_shift, int32_t world);
/* Composite of per-rank raycasts (device pointers, asynchronous on `stream`):
 * key[i] = float_bits(depth) << 32 | (normal missing) << 31 | rank for hit pixels, INT64_MAX
 * otherwise; after an all-reduce MIN of `key` over ranks, sf_composite_select zeroes the
 * depth / normals of pixels this rank did not win, so an all-reduce SUM of their bit
 * patterns (int32) assembles the nearest-depth composite on every rank. */
/* Halo exchange after an integrate on a sharded volume (device pointers; synchronises):
 * pack writes (table index, M^3 payload codes) records of the blocks the last sf_integrate
 * processed that touch (26-neighbourhood) a brick of another rank; *count = records (error
 * SF_OUT_OF_RANGE if > cap). apply mirrors, read-only, the records that touch a brick of this
 * rank (allocating them on first sight; *applied = mirrored). With every rank's records applied
 * on every rank, each trilinear sample the reference raycast takes is evaluable on the rank
 * owning its base voxel, so the composite is exact. */
int sf_shard_pack_halo(sf_volume_t vol, int32_t* keys, uint16_t* payloads, uint64_t cap, uint32_t* count,
                       void* stream);
int sf_shard_apply_halo(sf_volume_t vol, const int32_t* keys, const uint16_t* payloads, uint64_t n,
                        uint32_t* applied, void* stream);
int sf_composite_key(const float* depth, const float* normals_xyz, uint64_t n, int32_t rank, int64_t* key,
                     void* stream);
int sf_composite_select(const int64_t* key, uint64_t n, int32_t rank, float* depth, float* normals_xyz,
                        void* stream);

/* SparseTsdfGrid::allocate_block / free_block / block_slot (grid.cpp:82-119). */
int sf_volume_allocate_block(sf_volume_t vol, const int32_t bc[3], int32_t* slot_out);
int sf_volume_free_block(sf_volume_t vol, const int32_t bc[3]);
int sf_volume_block_slot(sf_volume_t vol, const int32_t bc[3], int32_t* slot_out);

/* SparseTsdfGrid::read_voxel / write_voxel (grid.cpp:121-154). read: *is_chi = 1 for chi
 * (nullopt); write: tsdf_is_chi = 1 writes chi. */
int sf_volume_read_voxel(sf_volume_t vol, const int32_t vc[3], int32_t* is_chi, double* tsdf, double* aux);
int sf_volume_write_voxel(sf_volume_t vol, const int32_t vc[3], int32_t tsdf_is_chi, double tsdf, double aux);

/* Block-buffer layout export (grid.hpp:98,178-181 and 65-68,159-162,189-191):
 *   table:   int32[N^3], z-major / x fastest, -1 = EMPTY
 *   payload: uint16 per voxel = {int8 tsdf_code (low byte), uint8 aux_code (high byte)},
 *            M^3 per slot, x fastest. */
int sf_volume_read_table(sf_volume_t vol, int32_t* host_table);
int sf_volume_read_payload(sf_volume_t vol, uint64_t first_slot, uint64_t slot_count, uint16_t* host_payload);
int sf_volume_write_payload(sf_volume_t vol, uint64_t first_slot, uint64_t slot_count, const uint16_t* host_payload);
/* Bulk import of a host grid's complete state into a freshly created (empty) volume: the
 * N^3 offset table, payload slots [0, slot_count) and the free-list stack bottom to top
 * (grid.hpp:189-191); allocated + free must equal the pool capacity. Used by the C++ drop-in
 * layer, whose host SparseTsdfGrid stays the source of truth. */
int sf_volume_import_state(sf_volume_t vol, const int32_t* table, const uint16_t* payload, uint64_t slot_count,
                           const int32_t* free_list, uint64_t free_count);
/* Free-list stack, bottom to top (grid.hpp:191); *count_out receives its length. */
int sf_volume_read_free_list(sf_volume_t vol, int32_t* host_out, uint64_t* count_out);

/* STSG v1 snapshot (grid.cpp:333-408). */
int sf_volume_save_snapshot(sf_volume_t vol, const char* path);
int sf_volume_load_snapshot(const char* path, uint64_t pool_capacity, int32_t device, sf_volume_t* out);

/* Float payload mode (block-sparse FloatShadowGrid semantics, grid.hpp:77-88): a
 * device-resident float2 {tsdf, aux} per pool voxel, chi = +inf / aux 0, updated by
 * sf_integrate alongside the quantized codes and used as the prior (fusion.cpp:313-318).
 * Unlike the reference shadow it is block-sparse, so any N is allowed. */
int sf_volume_enable_float_payload(sf_volume_t vol);

/* Payload layouts:
 *   SF_PAYLOAD_CODES (default)        P1: the reference's 2-byte {int8 tsdf, uint8 aux} codes.
 *   SF_PAYLOAD_CODES_FLOAT_SHADOW     P1 + the float shadow above (sf_volume_enable_float_payload).
 *   SF_PAYLOAD_FLOAT2                 P2: float2 {tsdf, aux} per voxel ONLY, block-sparse, with
 *                                     FloatShadowGrid semantics (chi = +inf / aux 0, the prior is
 *                                     the float value, fusion.cpp:313-318, 357-361). Decisions
 *                                     (pixel, band, chi cut) are the reference's; values are within
 *                                     the north-star 1e-5. Set on an empty volume. The quantized
 *                                     codes are not maintained: raycast, marching cubes, voxel and
 *                                     payload-code access and snapshots return SF_UNSUPPORTED. */
typedef enum {
    SF_PAYLOAD_CODES = 0,
    SF_PAYLOAD_CODES_FLOAT_SHADOW = 1,
    SF_PAYLOAD_FLOAT2 = 2
} sf_payload_layout;
int sf_volume_set_payload_layout(sf_volume_t vol, int32_t layout);
int sf_volume_get_payload_layout(sf_volume_t vol, int32_t* layout);
int sf_volume_read_float_payload(sf_volume_t vol, uint64_t first_slot, uint64_t slot_count, float* host_tsdf_aux);
int sf_volume_write_float_payload(sf_volume_t vol, uint64_t first_slot, uint64_t slot_count, const float* host_tsdf_aux);

/* ---- hot path ------------------------------------------------------------------------ */

/* fuse_frame(grid, frame, pose, params) (fusion.hpp:102-103, fusion.cpp:274-376):
 * surface-sampled block keys -> sort/unique -> ordered slot allocation -> frustum/probe
 * visibility -> per-voxel measurement + filter. On pool exhaustion the allocate-list
 * prefix before the first unallocatable block is integrated and SF_POOL_EXHAUSTED is
 * returned (fusion.cpp:369, grid.cpp:90-92). stats may be NULL (then nothing syncs). */
int sf_integrate(sf_volume_t vol, const sf_frame* frame, const double pose[12],
                 const sf_fusion_params* params, sf_fusion_stats* stats, void* stream);

/* select_update_blocks (fusion.hpp:71-72, fusion.cpp:187-235), for parity tests: block
 * coordinates (x,y,z triples) of the allocate list (ascending (z,y,x)) and of the update
 * list (ascending table order). Counts are in/out: capacity in, size out. */
int sf_select_update_blocks(sf_volume_t vol, const sf_frame* frame, const double pose[12],
                            int32_t* allocate_xyz, uint64_t* allocate_count,
                            int32_t* update_xyz, uint64_t* update_count, void* stream);

/* compute_ray_bounds (render.hpp:38-39, render.cpp:65-153). Outputs width*height floats. */
int sf_ray_bounds(sf_volume_t vol, const double pose[12], const sf_intrinsics* intr,
                  float* t_start, float* t_end, int32_t out_on_device, void* stream);

/* raycast(grid, pose, intrinsics) (render.hpp:61-63, render.cpp:155-250). depth: width*height
 * floats (0 = miss); normals_xyz: 3*width*height floats, camera frame. stats may be NULL. */
int sf_raycast(sf_volume_t vol, const double pose[12], const sf_intrinsics* intr,
               float* depth, float* normals_xyz, int32_t out_on_device,
               sf_raycast_stats* stats, void* stream);
/* raycast(grid, pose, intrinsics, bounds) with caller-supplied bounds (render.hpp:61-63):
 * the sharded path marches every rank's volume from the all-reduced (global) bounds.
 * `on_device` applies to the bounds and the outputs alike. */
int sf_raycast_with_bounds(sf_volume_t vol, const double pose[12], const sf_intrinsics* intr,
                           const float* t_start, const float* t_end, float* depth, float* normals_xyz,
                           int32_t on_device, sf_raycast_stats* stats, void* stream);

/* compute_normals(frame, opts) (camera.hpp:90, camera.cpp:44-76). */
int sf_compute_normals(const sf_frame* frame, double sigma0, double spatial_scale,
                       float* normals_xyz, int32_t out_on_device, void* stream);

/* icp(source, [source_normals,] target, target_normals, initial, params)
 * (registration.hpp:120-124, registration.cpp:195-220). source_normals may be NULL:
 * then compute_normals(source, params.normal_options) is used (registration.cpp:218).
 * Normal-map pointers live where the frames live (frame->on_device). */
int sf_icp(const sf_frame* source, const float* source_normals, const sf_frame* target,
           const float* target_normals, const double initial[12], const sf_match_params* params,
           sf_icp_result* result, void* stream);

/* ---- fused frame loop: run() per-frame body (pipeline.cpp:233-301) ------------------ */
/* A tracker owns the device-resident state of one reconstruction: the current pose, the
 * raycast model maps and the per-frame work buffers. Each step is raycast(current pose)
 * -> icp(captured vs rendered) -> compose -> fuse_frame, or fuse_frame at the supplied
 * pose (first frame / ground-truth tracking). Steps are fully asynchronous (no host
 * synchronisation); results are fetched with sf_tracker_fetch. */
typedef struct sf_tracker* sf_tracker_t;

typedef struct {
    sf_fusion_params fusion;
    sf_match_params match;
    sf_intrinsics camera;
    int32_t use_graphs; /* capture the per-frame launch sequence in a CUDA graph */
    /* 0 (default): reference-exact pose chain. The reference forms
     * initial_delta = compose(invert(current), current) and current = compose(current, delta)
     * (pipeline.cpp:262-282), which multiplies the rotation's departure from orthonormality by
     * ~3 per tracked frame (R R^T R); after ~30 frames tracking collapses in the reference and
     * here alike. 1: project the estimated rotation back onto SO(3) (nearest_rotation) after
     * every registration — a numerical fix that departs from reference bits. */
    int32_t orthonormalize;
} sf_tracker_config;

typedef struct {
    int32_t frame;
    int32_t registered;
    int32_t status; /* sf_status of this frame (SF_OK, SF_POOL_EXHAUSTED, SF_TRACKING_LOST) */
    double pose[12];
    int32_t iterations;
    uint64_t matches;
    double residual_rms;
    double lambda_over_n[6];
    int32_t gated_mask[6];
    sf_fusion_stats fusion;
    sf_raycast_stats raycast;
    uint64_t blocks_processed; /* allocate-list prefix + update list integrated this frame */
    uint64_t voxels_visited;   /* blocks_processed * M^3 */
    uint64_t kernel_launches;  /* device kernels this frame ran (graph: top level + 2 per ICP iteration) */
    uint64_t exact_voxels;     /* voxels the integrate kernel settled on its FP64 fallback (uncertain FP32 decision) */
    uint64_t integrate_ns;     /* integrate kernel span on the device clock: first CTA start to last CTA end (%globaltimer) */
    uint64_t icp_ns;           /* ICP span on the device clock: first step start to the end of the last iteration's solve */
    int32_t icp_steps;         /* ICP step launches this frame (device-side loop: one per iteration) */
    int32_t pad_;
    uint64_t ray_dda_cells;      /* reference DDA cells of the rays reaching the occupied box (roofline count) */
    uint64_t ray_refine_samples; /* stage-2 secant + gradient samples of the raycast */
} sf_frame_metrics;

int sf_tracker_create(sf_volume_t vol, const sf_tracker_config* config, const double initial_pose[12],
                      sf_tracker_t* out);
int sf_tracker_destroy(sf_tracker_t tr);
/* mode 0: track (raycast + ICP, except for the tracker's first frame which is fused at the
 * current pose); mode 1: ground truth (fuse at gt_pose, no raycast/ICP); mode 2: track with
 * an external initial delta passed in gt_pose (tracking.mode = icp_with_hook: ICP starts
 * from compose(current, external), pipeline.cpp:262-267, registration.cpp:222-224).
 * Host frames (captured->on_device == 0) are copied asynchronously: the depth / sigma host
 * buffers must stay valid and UNMODIFIED until this step has completed — i.e. until
 * sf_tracker_fetch, sf_tracker_fetch_frame(k) of this step, or a synchronisation of `stream`.
 * A capture loop that refills one pinned buffer must alternate two (or fetch first).
 * The frame that raises TrackingLost / PoolExhausted reports what run()'s catch block pushes
 * (pipeline.cpp:289-299); every later step is a no-op carrying the same status. */
int sf_tracker_step(sf_tracker_t tr, const sf_frame* captured, int32_t mode, const double gt_pose[12],
                    void* stream);
/* Re-seed the tracker's current pose (relocalisation; asynchronous on `stream`). */
int sf_tracker_set_pose(sf_tracker_t tr, const double pose[12], void* stream);
/* Synchronises `stream` and copies the metrics of the last step. */
int sf_tracker_fetch(sf_tracker_t tr, sf_frame_metrics* out, void* stream);
/* Streaming: metrics of frame `frame` (one of the last two steps) without waiting for later
 * steps. With host frames, step k's host->device copy overlaps step k-1's compute, so a
 * caller that issues step k+1 before fetching step k pipelines input transfer and compute. */
int sf_tracker_fetch_frame(sf_tracker_t tr, int32_t frame, sf_frame_metrics* out);
/* Device-timed stages of the last step, in ms (CUDA events recorded inside the step /
 * graph): [0] raycast (bounds + march), [1] ICP (source normals + all iterations),
 * [2] fuse prologue (frame prep, keys, sort/unique, allocation, visibility),
 * [3] the per-voxel integrate kernel, [4] whole step. Call after sf_tracker_fetch. A stage
 * whose events are not recorded (sf_tracker_set_stage_timing) reads -1. */
int sf_tracker_stage_times(sf_tracker_t tr, float ms[5]);
/* Stage-timing events inside the step: 2 = all stages (default), 1 = the integrate kernel's
 * pair only, 0 = none. Each event is a node of the frame graph and costs a few microseconds
 * of the step, so throughput runs switch them off. Rebuilds the cached graphs. */
int sf_tracker_set_stage_timing(sf_tracker_t tr, int32_t level);
/* Device pointer to the tracker's pose (12 doubles). */
int sf_tracker_device_pose(sf_tracker_t tr, const double** device_pose);
/* Number of this library's kernels the last sf_tracker_step launched at issue time. With
 * graphs the ICP iterations run as a device-side loop whose kernels are counted only after
 * the fact: sf_frame_metrics.kernel_launches (after fetch) is the complete per-frame count. */
int sf_tracker_last_launch_count(sf_tracker_t tr, uint64_t* count);
/* Bytes one step moves across PCIe when the frame is a host frame (depth [+ sigma]) and
 * bytes sf_tracker_fetch reads back. */
int sf_tracker_io_bytes(sf_tracker_t tr, int32_t has_sigma, uint64_t* h2d, uint64_t* d2h);

/* ---- sharded fused frame --------------------------------
 * run()'s per-frame body over a block pool partitioned across ranks, one CUDA graph per frame
 * with the exchanges inside: ray bounds per rank -> MIN/MAX all-reduce (global bounds), each
 * rank marches only the rays its own blocks meet, nearest-depth composite, ICP on the
 * composite (icp_mode 0: replicated on every rank; 1: partial normal-equation sums over pixel
 * slices combined by an all-reduce), pose update, per-rank fuse, halo exchange through
 * fixed-capacity buffers. Ranks are in-process (create_local: `count` volumes of this GPU,
 * volume i sharded as rank i of count; the exchanges are kernels) or one per process
 * (create_nccl: NCCL on the stream, captured into the graph; rank 0 makes the id with
 * sf_nccl_unique_id and the caller broadcasts it). No reference counterpart. */
typedef struct sf_shard_tracker* sf_shard_tracker_t;
typedef struct {
    sf_tracker_config base;
    int32_t icp_mode;       /* 0: replicas, 1: partial sums + all-reduce */
    int32_t pad_;
    uint64_t halo_capacity; /* halo records per rank per frame (0 -> 16384); overflow is reported */
} sf_shard_tracker_config;
typedef struct {
    int32_t frame, registered, status, iterations;
    double pose[12];
    uint64_t matches;
    uint64_t voxels_updated;  /* summed over ranks */
    uint64_t blocks_total;    /* owned blocks summed over ranks (mirrored halo blocks excluded) */
    uint64_t hit_pixels;      /* composite raycast */
    uint64_t halo_records;    /* records packed this frame, all ranks */
    uint64_t halo_overflow;   /* records beyond halo_capacity (not exchanged: raise the capacity) */
    uint64_t kernel_launches; /* this process's kernels this frame */
    int32_t icp_steps, pad_;
} sf_shard_frame_metrics;
int sf_nccl_unique_id(uint8_t out[128]);
int sf_shard_tracker_create_local(sf_volume_t* volumes, int32_t count, const sf_shard_tracker_config* config,
                                  const double initial_pose[12], sf_shard_tracker_t* out);
int sf_shard_tracker_create_nccl(sf_volume_t volume, const uint8_t nccl_id[128], int32_t rank, int32_t world,
                                 const sf_shard_tracker_config* config, const double initial_pose[12],
                                 sf_shard_tracker_t* out);
int sf_shard_tracker_destroy(sf_shard_tracker_t tr);
/* modes as sf_tracker_step (0 track, 1 ground truth, 2 track with an external delta) */
int sf_shard_tracker_step(sf_shard_tracker_t tr, const sf_frame* captured, int32_t mode, const double gt_pose[12],
                          void* stream);
int sf_shard_tracker_set_pose(sf_shard_tracker_t tr, const double pose[12], void* stream);
int sf_shard_tracker_fetch(sf_shard_tracker_t tr, sf_shard_frame_metrics* out, void* stream);

/* ---- synthetic input (scene.hpp:69-79, scene.cpp:101-177) --------------------------- */
/* Analytic scene of spheres (cx,cy,cz,r), planes (nx,ny,nz,offset; normalised as
 * AnalyticScene::add_plane does) and axis-aligned boxes (cx,cy,cz,hx,hy,hz). Depth is
 * sphere traced on the device in FP64 (bit-identical to render_synthetic_depth for
 * sigma0 == 0); with noise, the Gaussian sequence is drawn on the host with
 * std::mt19937_64 / std::normal_distribution in the reference's pixel order. */
typedef struct {
    const double* spheres; int32_t sphere_count;
    const double* planes;  int32_t plane_count;
    const double* boxes;   int32_t box_count;
} sf_scene;

int sf_render_synthetic_depth(const sf_scene* scene, const double pose[12], const sf_intrinsics* intr,
                              double noise_sigma0, uint64_t noise_seed, int32_t max_steps,
                              double tolerance_scale, double domain_size,
                              float* depth_host, float* sigma_host /* NULL if sigma0 == 0 */);

#ifdef __cplusplus
}
#endif

#endif /* SF_GPU_H */
