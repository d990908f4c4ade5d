// sf_internal.h — host-side internals shared by the translation units of libsf_gpu.so.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "../../include/sf_gpu.h"
#include "sf_common.cuh"

namespace sf {

// ---- error plumbing: C++ exceptions inside, sf_status at the C boundary -------------
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void set_last_error(const std::string& msg);
[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file, int line);

#define SF_CUDA(call)                                                       \
    do {                                                                    \
        cudaError_t sf_e_ = (call);                                         \
        if (sf_e_ != cudaSuccess) ::sf::throw_cuda(sf_e_, #call, __FILE__, __LINE__); \
    } while (0)
#define SF_LAUNCH_CHECK() SF_CUDA(cudaGetLastError())

// Programmatic dependent launch (SF_PDL=0 disables): the launch of a kernel is prepared
// while its stream predecessor runs; the kernel calls pdl_wait() (a no-op for a normal
// launch) before anything else, which returns once the predecessor has completed and its
// writes are visible. No kernel triggers early (griddepcontrol.launch_dependents): CTAs of
// a waiting dependent would take SM slots from the predecessor's tail (measured slower).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    SF_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}

// Timing event usable both eagerly and under stream capture (as an event-record node).
inline void record_event(cudaEvent_t ev, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    SF_CUDA(cudaStreamIsCapturing(s, &st));
    if (st == cudaStreamCaptureStatusActive) SF_CUDA(cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal));
    else SF_CUDA(cudaEventRecord(ev, s));
}

template <typename F>
int guarded(F&& f) {
    try {
        set_last_error("");
        return f();
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return SF_CUDA_ERROR;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SF_CUDA_ERROR;
    }
}

// ---- device counters of a volume --------------------------------------------------
struct VolCounters {
    unsigned long long allocated_count;
    unsigned long long free_top;    // size of the free-list stack
    unsigned long long high_water;  // 1 + highest slot ever handed out
    unsigned long long halo_count;  // sharded volume: mirrored blocks of other ranks
};

// Per-frame device counters (zeroed by the frame-setup kernel).
struct FrameCounters {
    uint32_t n_unique;   // CUB unique output count (may include the sentinel)
    uint32_t n_list;     // allocate-list length (valid unique keys)
    uint32_t n_new;      // keys needing a fresh slot
    uint32_t limit;      // processed allocate-list prefix
    uint32_t n_update;   // update-list length
    uint32_t exhausted;  // PoolExhausted raised this frame
    uint32_t skip;       // whole fuse skipped (tracker dead / tracking lost)
    uint32_t exhaust_key;  // smallest allocate-list key that found no free slot (PoolExhausted), else ~0
    uint32_t upd_base;     // work-list index where the update list starts
    uint32_t tickets;      // last-CTA ticket of the allocation pass
    unsigned long long voxels_updated;
    unsigned long long alloc_before;
    unsigned long long alloc_now;
    unsigned long long exact_voxels;  // integrate: voxels decided on the FP64 fallback path
    uint32_t row_chunks;              // integrate: next row chunk (dynamic scheduling)
    uint32_t pad_;
    unsigned long long hw_before;     // slot high-water mark when the frame started
    unsigned long long t_begin;       // integrate: first CTA start (%globaltimer, ns)
    unsigned long long t_end;         // integrate: last CTA end
};

// Device-side aux codec tables (host-computed with the reference's libm).
constexpr int kAuxLut = 1024;  // max buckets of the variance-code lookup
struct AuxTables {
    double tsdf_decode[256];  // dequantize_tsdf(code)        (grid.cpp:25-27), index code+128
    double aux_decode[256];   // AuxQuantization::decode(code) (grid.cpp:48-51)
    double aux_thresh[256];   // variance mode: thresh[k] = min v with encode(v) >= k, k = 1..255
    // FP32 copies (round to nearest) for the certified single-precision integrate path;
    // their rounding error is part of that path's decision margins (sf_fusion.cu).
    float tsdf_decode_f[256], aux_decode_f[256], aux_thresh_f[256];
    int fp32_ok;  // all codec values representable as normal floats (else the FP64 kernel runs)
    // Variance-mode code lookup on the float bits (lut_n > 0): bucket b = (bits(v) >> lut_shift)
    // - lut_base (clamped to [0, lut_n)) holds at most one float threshold; lut[b] = {bits of that
    // threshold (+inf if none), #thresholds below the bucket}, so code = lut[b].y + (v >= T).
    int lut_shift, lut_base, lut_n;
    uint2 lut[kAuxLut];
};
void build_aux_tables(const VolParams& P, AuxTables* t);
uint8_t host_aux_encode(const VolParams& P, double value);  // reference encode (grid.cpp:38-46)

// ---- frame-sized scratch, owned by a volume or a tracker ----------------------------
struct FrameBuffers {
    int w = 0, h = 0, stride = 0;
    int device = 0;
    float* depth = nullptr;    // staged depth for host frames
    float* sigma = nullptr;    // staged sigma plane
    float* normals = nullptr;  // 3*w*h fusion normals
    uint8_t* edge = nullptr;   // w*h
    double* pix_var = nullptr; // w*h per-pixel p_k
    double* pix_w = nullptr;   // w*h per-pixel w_k
    uint8_t* pix_ok = nullptr; // w*h valid && quality >= 0.2
    double* pix_dm = nullptr;  // w*h depth where pix_ok, else 0 (one gather per voxel)
    float2* pix_f = nullptr;   // w*h {depth where pix_ok else 0, (float) p_k or w_k}: FP32 integrate
    double* pix_q = nullptr;   // w*h view quality incl. near-edge halving (refinement path)
    uint32_t key_cap = 0;
    uint32_t* keys = nullptr;
    uint32_t* keys_sorted = nullptr;
    uint32_t* keys_unique = nullptr;
    uint32_t* flags = nullptr;
    uint32_t* ranks = nullptr;
    void* cub_temp = nullptr;
    size_t cub_temp_bytes = 0;
    int2* work = nullptr;  // {slot | fresh<<31, table index}
    uint64_t work_cap = 0;
    FrameCounters* ctr = nullptr;
    FrameConsts* fc = nullptr;
    double* pose = nullptr;  // 12 doubles
    FrameCounters* h_ctr = nullptr;  // pinned mirror
    void release();
    ~FrameBuffers() { release(); }
};


}  // namespace sf

// ---- the opaque volume -------------------------------------------------------------
struct sf_volume {
    int device = 0;
    sf_grid_config cfg{};
    sf_aux_quant aux{};
    sf::VolParams P{};
    int32_t* d_table = nullptr;      // N^3
    uint16_t* d_payload = nullptr;   // capacity * M^3
    float2* d_fpayload = nullptr;    // optional float payload {tsdf, aux}
    int layout = SF_PAYLOAD_CODES;   // sf_payload_layout
    int32_t* d_free_list = nullptr;  // capacity (stack, bottom..top)
    int32_t* d_slot_key = nullptr;   // capacity: table index of the block in each slot, -1 free
    uint32_t* d_occ = nullptr;       // occupancy bitmap, N^3 bits
    uint32_t* d_keybits = nullptr;   // the frame's allocate-list keys, N^3 bits (zero between frames)
    sf::VolCounters* d_vc = nullptr;
    uint32_t* d_sched = nullptr;     // self-resetting work counters of persistent kernels (zero between launches)
    uint32_t* d_patch_order = nullptr;  // ray-bounds patch order for an order_w x order_h image
    int order_w = -1, order_h = -1;
    sf::AuxTables* d_aux = nullptr;
    sf::AuxTables h_aux{};
    sf::FrameBuffers fb;  // scratch for the stand-alone API calls
    unsigned long long host_allocated() const;
};

namespace sf {
using Volume = ::sf_volume;
// Operations that read or write the 2-byte codes fail loudly on a float2-only volume.
inline void require_codes(const Volume& v, const char* what) {
    if (v.layout == SF_PAYLOAD_FLOAT2)
        throw Error(SF_UNSUPPORTED, std::string(what) + ": not available on a float2-payload volume (SF_PAYLOAD_FLOAT2)");
}
void ensure_frame_buffers(Volume& v, FrameBuffers& fb, int w, int h);
void ensure_patch_order(Volume& v, int w, int h);

// Launchers shared between the stand-alone API (sf_integrate, sf_raycast, sf_icp) and the
// tracker. All are asynchronous on `stream`; `dead_flag` (device int, may be NULL) turns
// the launched kernels into no-ops when set (tracker after TrackingLost / PoolExhausted).
struct RayCounters {
    unsigned long long sample_steps, hit_pixels, rays_with_bounds;
    unsigned long long listed;    // length of the active-ray list written by the ray-bounds pass
    unsigned long long brackets;  // rays the stage-1 march bracketed (refine-pass list length)
    // algorithmic work (raycast roofline): cells the reference DDA walks for the
    // rays that reach the occupied box (entry to exit cell within [near, far]), and the secant +
    // gradient samples of stage 2
    unsigned long long dda_cells;
    unsigned long long refine_samples;
};
// A stage-1 bracket [a, b] with TSDF values (va > 0 > vb) of pixel idx (render.cpp:207-208).
struct RayBracket {
    double a, b, va, vb;
    int idx, pad;
};
void launch_consts(const VolParams& P, const Intr& intr, const double* d_pose, FrameConsts* d_fc, cudaStream_t s,
                   uint64_t* launches);
// fuse_frame at the pose in fb.pose (device)
struct FuseEvents {
    cudaEvent_t before_integrate = nullptr, after_integrate = nullptr;
};
// prep_done: launch_fuse_prep already ran for this frame (e.g. on a parallel graph branch).
void launch_fuse(Volume& v, FrameBuffers& fb, const Intr& intr, const float* depth, const float* sigma,
                 const FuseParams& fp, cudaStream_t s, bool export_lists_only, uint64_t* launches,
                 const int* dead_flag, const FuseEvents* events = nullptr, bool prep_done = false,
                 bool caller_brackets = false);
// caller_brackets: the caller ran frame_consts_warp + fuse_begin_body (sf_sample.cuh) before
// and runs fuse_finalize_body after (tracker kernels that merge them with their own work).
void launch_fuse_prep(Volume& v, FrameBuffers& fb, const Intr& intr, const float* depth, const float* sigma,
                      const FuseParams& fp, cudaStream_t s, uint64_t* launches, const int* dead);
// With ray_list (+ list_ctr, depth, normals) the pass also appends every pixel with
// non-empty bounds to ray_list (length in list_ctr->listed, which must start at 0) and
// writes the empty raycast result (0 depth / normal) for the others.
void launch_ray_bounds(Volume& v, const FrameConsts* d_fc, const Intr& intr, float* t_start, float* t_end,
                       cudaStream_t s, uint64_t* launches, const int* dead_flag, int* ray_list = nullptr,
                       RayCounters* list_ctr = nullptr, float* depth = nullptr, float* normals = nullptr);
// Marches the rays of ray_list (from launch_ray_bounds; length in d_stats->listed).
void launch_raycast(Volume& v, const FrameConsts* d_fc, const Intr& intr, const float* t_start, const float* t_end,
                    float* depth, float* normals, RayCounters* d_stats, cudaStream_t s, uint64_t* launches,
                    const int* dead_flag, const int* ray_list, RayBracket* brackets);
void launch_compute_normals(const float* depth, int w, int h, const Intr& intr, double sigma0,
                            double spatial_scale, float* normals, cudaStream_t s, uint64_t* launches,
                            const int* dead_flag);
Intr to_intr(const sf_intrinsics& i);
FuseParams resolve_fuse_params(const Volume& v, const sf_fusion_params& p, bool has_sigma);

}  // namespace sf
