// sf_volume.cu — SparseTsdfGrid storage on the device (grid.hpp:96-193, grid.cpp:53-427).
//
// HBM layout:
//   d_table      int32[N^3]        offset table, z-major / x fastest, -1 = EMPTY (grid.hpp:98)
//   d_payload    uint16[cap*M^3]   {int8 tsdf_code, uint8 aux_code} per voxel, x fastest
//   d_free_list  int32[cap]        free-list stack, lowest slot on top (grid.cpp:68-71)
//   d_slot_key   int32[cap]        inverse map slot -> table index (-1 = free), lets the
//                                  visibility pass walk allocated blocks without an N^3 scan
//   d_occ        uint32[N^3/32]    occupancy bitmap for the ray-bounds DDA (L2 resident), followed
//                                  by a coarse 1-bit-per-16^3-blocks bitmap (shared-memory resident)
//   d_fpayload   float2[cap*M^3]   optional float payload (FloatShadowGrid semantics)
#include <cstdlib>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>
#include <vector>

#include "sf_internal.h"

namespace sf {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

void throw_cuda(cudaError_t e, const char* what, const char* file, int line) {
    throw Error(SF_CUDA_ERROR, std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                                   ") in " + what + " at " + file + ":" + std::to_string(line));
}

Intr to_intr(const sf_intrinsics& i) {
    Intr r;
    r.w = i.width;
    r.h = i.height;
    r.fx = i.fx;
    r.fy = i.fy;
    r.cx = i.cx;
    r.cy = i.cy;
    r.near_plane = i.near_plane;
    r.far_plane = i.far_plane;
    return r;
}

// ---- aux codec (grid.cpp:38-51) ----------------------------------------------------
uint8_t host_aux_encode(const VolParams& P, double value) {
    if (P.aux_mode == 0) {
        const double clamped = std::clamp(value, 0.0, P.aux_w_max);
        return static_cast<uint8_t>(std::lround(clamped / P.aux_w_max * 255.0));
    }
    const double clamped = std::clamp(value, P.aux_p_min, P.aux_p_max);
    const double s = std::log(clamped / P.aux_p_min) / std::log(P.aux_p_max / P.aux_p_min);
    return static_cast<uint8_t>(std::lround(s * 255.0));
}

static double host_aux_decode(const VolParams& P, uint8_t code) {
    if (P.aux_mode == 0) return static_cast<double>(code) / 255.0 * P.aux_w_max;
    return P.aux_p_min * std::exp(static_cast<double>(code) / 255.0 * std::log(P.aux_p_max / P.aux_p_min));
}

static uint64_t dbits(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
}
static double bitsd(uint64_t b) {
    double d;
    std::memcpy(&d, &b, 8);
    return d;
}

// Variance-mode encode is a monotone step function of the value (log is monotone), so
// encode(v) == #{k : v >= thresh[k]}. Each threshold is located by bisection over the
// ordered bit patterns of positive doubles, with the reference's own libm log: exact.
static void build_aux_thresholds(const VolParams& P, AuxTables* t);
static uint32_t f_bits(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    return u;
}
static float bits_f(uint32_t u) {
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}
void build_aux_tables(const VolParams& P, AuxTables* t) {
    for (int c = -128; c < 128; ++c) t->tsdf_decode[c + 128] = dequantize_tsdf(static_cast<int8_t>(c), P.delta);
    for (int c = 0; c < 256; ++c) t->aux_decode[c] = host_aux_decode(P, static_cast<uint8_t>(c));
    t->aux_thresh[0] = -INFINITY;
    for (int k = 1; k < 256; ++k) t->aux_thresh[k] = INFINITY;
    if (P.aux_mode == 1) build_aux_thresholds(P, t);
    // FP32 copies; the single-precision path runs only when every value is a normal float
    // (or 0 / inf) far from the float range limits.
    auto fits = [](double x) { return x == 0.0 || std::isinf(x) || (std::fabs(x) > 1e-30 && std::fabs(x) < 1e30); };
    t->fp32_ok = fits(P.delta) && P.delta > 0.0 ? 1 : 0;
    for (int c = 0; c < 256; ++c) {
        t->tsdf_decode_f[c] = static_cast<float>(t->tsdf_decode[c]);
        t->aux_decode_f[c] = static_cast<float>(t->aux_decode[c]);
        t->aux_thresh_f[c] = static_cast<float>(t->aux_thresh[c]);
        if (!fits(t->tsdf_decode[c]) || !fits(t->aux_decode[c]) || !fits(t->aux_thresh[c])) t->fp32_ok = 0;
    }
    if (P.aux_mode == 0 && !fits(P.aux_w_max)) t->fp32_ok = 0;
    // variance-code lookup over the float thresholds (see AuxTables)
    t->lut_n = 0;
    t->lut_shift = 0;
    t->lut_base = 0;
#ifndef SF_AUX_LUT
#define SF_AUX_LUT 1
#endif
    if (SF_AUX_LUT && P.aux_mode == 1 && t->fp32_ok) {
        std::vector<uint32_t> fin;  // bit patterns of the finite (positive) float thresholds, ascending
        int n_neg = 0;
        bool ok = true;
        for (int k = 1; k < 256; ++k) {
            const float f = t->aux_thresh_f[k];
            if (f == -INFINITY) {
                if (!fin.empty()) ok = false;  // -inf thresholds precede every finite one
                ++n_neg;
            } else if (std::isfinite(f)) {
                if (!(f > 0.0f) || (!fin.empty() && !(f > bits_f(fin.back())))) ok = false;
                fin.push_back(f_bits(f));
            }
        }
        if (ok && !fin.empty()) {
            int sh = 23;
            for (; sh > 0; --sh) {  // coarsest buckets holding at most one threshold each
                bool distinct = true;
                for (size_t i = 1; i < fin.size(); ++i) distinct = distinct && (fin[i] >> sh) != (fin[i - 1] >> sh);
                if (distinct) break;
            }
            const uint32_t base = fin.front() >> sh, n = (fin.back() >> sh) - base + 1;
            bool distinct = true;
            for (size_t i = 1; i < fin.size(); ++i) distinct = distinct && (fin[i] >> sh) != (fin[i - 1] >> sh);
            if (distinct && n <= static_cast<uint32_t>(kAuxLut)) {
                size_t j = 0;  // next finite threshold
                for (uint32_t b = 0; b < n; ++b) {
                    uint2 e = make_uint2(f_bits(INFINITY), static_cast<uint32_t>(n_neg + j));
                    if (j < fin.size() && (fin[j] >> sh) == base + b) e.x = fin[j++];
                    t->lut[b] = e;
                }
                t->lut_shift = sh;
                t->lut_base = static_cast<int>(base);
                t->lut_n = static_cast<int>(n);
            }
        }
    }
}

static void build_aux_thresholds(const VolParams& P, AuxTables* t) {
    const double lo0 = P.aux_p_min, hi0 = P.aux_p_max;
    if (!(lo0 > 0.0) || !(hi0 > lo0)) return;
    for (int k = 1; k < 256; ++k) {
        if (host_aux_encode(P, hi0) < k) break;
        uint64_t lo = dbits(lo0), hi = dbits(hi0);  // enc(lo) < k <= enc(hi)
        if (host_aux_encode(P, lo0) >= k) {
            t->aux_thresh[k] = -INFINITY;
            continue;
        }
        while (hi - lo > 1) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (host_aux_encode(P, bitsd(mid)) >= k) hi = mid;
            else lo = mid;
        }
        t->aux_thresh[k] = bitsd(hi);
    }
}

// ---- frame buffers ---------------------------------------------------------------
void FrameBuffers::release() {
    if (w == 0 && h == 0 && !ctr) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    void* ptrs[] = {depth, sigma, normals, edge, pix_var, pix_w, pix_ok, pix_dm, pix_f, pix_q, keys, keys_sorted, keys_unique,
                    flags, ranks, cub_temp, work, ctr, fc, pose};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h_ctr) cudaFreeHost(h_ctr);
    cudaSetDevice(prev);
    depth = sigma = normals = nullptr;
    edge = pix_ok = nullptr;
    pix_var = pix_w = nullptr;
    pix_dm = nullptr;
    pix_f = nullptr;
    pix_q = nullptr;
    keys = keys_sorted = keys_unique = flags = ranks = nullptr;
    cub_temp = nullptr;
    work = nullptr;
    ctr = nullptr;
    fc = nullptr;
    pose = nullptr;
    h_ctr = nullptr;
    w = h = 0;
}

size_t cub_temp_bytes_needed(uint32_t key_cap);  // sf_fusion.cu

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("SF_PDL");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

void ensure_frame_buffers(Volume& v, FrameBuffers& fb, int w, int h) {
    ensure_patch_order(v, w, h);  // the tracker captures ray bounds into a graph
    if (fb.w == w && fb.h == h && fb.ctr) return;
    fb.release();
    fb.device = v.device;
    fb.w = w;
    fb.h = h;
    const size_t n = static_cast<size_t>(w) * h;
    fb.stride = std::max(1, (v.P.M + 1) / 2);  // fusion.cpp:191
    const uint64_t su = (static_cast<uint64_t>(w) + fb.stride - 1) / fb.stride;
    const uint64_t sv = (static_cast<uint64_t>(h) + fb.stride - 1) / fb.stride;
    fb.key_cap = static_cast<uint32_t>(3 * su * sv);
    SF_CUDA(cudaMalloc(&fb.depth, n * sizeof(float)));
    SF_CUDA(cudaMalloc(&fb.sigma, n * sizeof(float)));
    SF_CUDA(cudaMalloc(&fb.normals, 3 * n * sizeof(float)));
    SF_CUDA(cudaMalloc(&fb.edge, n));
    SF_CUDA(cudaMalloc(&fb.pix_var, n * sizeof(double)));
    SF_CUDA(cudaMalloc(&fb.pix_w, n * sizeof(double)));
    SF_CUDA(cudaMalloc(&fb.pix_ok, n));
    SF_CUDA(cudaMalloc(&fb.pix_dm, n * sizeof(double)));
    SF_CUDA(cudaMalloc(&fb.pix_f, n * sizeof(float2)));
    SF_CUDA(cudaMalloc(&fb.pix_q, n * sizeof(double)));
    SF_CUDA(cudaMalloc(&fb.keys, fb.key_cap * sizeof(uint32_t)));
    SF_CUDA(cudaMalloc(&fb.keys_sorted, fb.key_cap * sizeof(uint32_t)));
    SF_CUDA(cudaMalloc(&fb.keys_unique, fb.key_cap * sizeof(uint32_t)));
    SF_CUDA(cudaMalloc(&fb.flags, fb.key_cap * sizeof(uint32_t)));
    SF_CUDA(cudaMalloc(&fb.ranks, fb.key_cap * sizeof(uint32_t)));
    fb.cub_temp_bytes = cub_temp_bytes_needed(fb.key_cap);
    SF_CUDA(cudaMalloc(&fb.cub_temp, fb.cub_temp_bytes));
    fb.work_cap = static_cast<uint64_t>(fb.key_cap) + v.P.capacity;
    SF_CUDA(cudaMalloc(&fb.work, fb.work_cap * sizeof(int2)));
    SF_CUDA(cudaMalloc(&fb.ctr, sizeof(FrameCounters)));
    SF_CUDA(cudaMemset(fb.ctr, 0, sizeof(FrameCounters)));
    SF_CUDA(cudaMalloc(&fb.fc, sizeof(FrameConsts)));
    SF_CUDA(cudaMalloc(&fb.pose, 12 * sizeof(double)));
    SF_CUDA(cudaMallocHost(&fb.h_ctr, sizeof(FrameCounters)));
    std::memset(fb.h_ctr, 0, sizeof(FrameCounters));
}

// ---- kernels: volume init / structural mutation ------------------------------------
__global__ void k_fill_u16(uint16_t* p, uint64_t n, uint16_t v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}
__global__ void k_fill_f2(float2* p, uint64_t n, float2 v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}
// Free list [cap-1, ..., 0] bottom to top (grid.cpp:68-71).
__global__ void k_init_free_list(int32_t* fl, int32_t* slot_key, uint32_t cap) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < cap; i += gridDim.x * blockDim.x) {
        fl[i] = static_cast<int32_t>(cap - 1 - i);
        slot_key[i] = -1;
    }
}

// allocate_block (grid.cpp:87-100): one block, serial semantics.
__global__ void k_allocate_one(VolParams P, int32_t* table, int32_t* free_list, int32_t* slot_key, uint32_t* occ,
                               uint16_t* payload, float2* fpayload, VolCounters* vc, uint64_t tidx, int32_t* out) {
    __shared__ int32_t s_slot;
    if (threadIdx.x == 0) {
        int32_t slot = table[tidx];
        if (slot == kEmpty) {
            if (vc->free_top == 0) {
                slot = -2;  // PoolExhausted
            } else {
                slot = free_list[vc->free_top - 1];
                vc->free_top -= 1;
                vc->allocated_count += 1;
                if ((unsigned long long)slot + 1 > vc->high_water) vc->high_water = slot + 1;
                table[tidx] = slot;
                slot_key[slot] = static_cast<int32_t>(tidx);
                occ_set(P, occ, tidx);
                out[1] = 1;  // fresh
            }
        }
        out[0] = slot;
        s_slot = slot;
    }
    __syncthreads();
    if (s_slot >= 0 && out[1] == 1) {
        for (int i = threadIdx.x; i < P.M3; i += blockDim.x) payload[(uint64_t)s_slot * P.M3 + i] = kChiPayload;
    }
}

// free_block (grid.cpp:102-119); the float payload is reset to chi like the shadow.
__global__ void k_free_one(VolParams P, int32_t* table, int32_t* free_list, int32_t* slot_key, uint32_t* occ,
                           float2* fpayload, VolCounters* vc, uint64_t tidx) {
    __shared__ int32_t s_slot;
    if (threadIdx.x == 0) {
        const int32_t slot = table[tidx];
        s_slot = slot;
        if (slot != kEmpty) {
            table[tidx] = kEmpty;
            free_list[vc->free_top] = slot;
            vc->free_top += 1;
            vc->allocated_count -= 1;
            slot_key[slot] = -1;
            occ[tidx >> 5] &= ~(1u << (tidx & 31));
        }
    }
    __syncthreads();
    if (s_slot != kEmpty && fpayload) {
        for (int i = threadIdx.x; i < P.M3; i += blockDim.x)
            fpayload[(uint64_t)s_slot * P.M3 + i] = make_float2(INFINITY, 0.0f);
    }
}

// Rebuild slot_key + occupancy from the table (after bulk host writes, e.g. snapshots).
__global__ void k_rebuild_index(VolParams P, const int32_t* table, int32_t* slot_key, uint32_t* occ) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < P.table_size;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int32_t s = table[i];
        if (s != kEmpty) {
            slot_key[s] = static_cast<int32_t>(i);
            occ_set(P, occ, i);
        }
    }
}

}  // namespace sf

using namespace sf;

unsigned long long sf_volume::host_allocated() const {
    VolCounters c;
    SF_CUDA(cudaMemcpy(&c, d_vc, sizeof(c), cudaMemcpyDeviceToHost));
    return c.allocated_count;
}

static VolParams make_params(const sf_grid_config& c, const sf_aux_quant& a, uint32_t capacity) {
    VolParams P{};
    P.N = c.blocks_per_axis;
    P.M = c.voxels_per_block_axis;
    P.M3 = P.M * P.M * P.M;
    P.res = P.N * P.M;
    P.ox = c.box_origin[0];
    P.oy = c.box_origin[1];
    P.oz = c.box_origin[2];
    P.box_side = c.box_side;
    P.voxel = c.box_side / P.res;                      // GridConfig::voxel_size (grid.hpp:36)
    P.inv_voxel = 1.0 / P.voxel;
    P.block_side = P.voxel * P.M;                      // SparseTsdfGrid::block_side (grid.hpp:149)
    P.inv_block_side = 1.0 / P.block_side;
    P.delta = c.truncation > 0.0 ? c.truncation : 4.0 * P.voxel;  // grid.hpp:37
    P.aux_mode = a.mode;
    P.aux_w_max = a.w_max;
    P.aux_p_min = a.p_min;
    P.aux_p_max = a.p_max;
    P.aux_lg_pmin = a.mode == 1 ? std::log2(a.p_min) : 0.0;
    P.aux_lg_scale = a.mode == 1 ? 255.0 / std::log2(a.p_max / a.p_min) : 0.0;
    P.table_size = static_cast<uint64_t>(P.N) * P.N * P.N;
    // table indices travel as int32 (slot -> key map, work items, ray DDA)
    if (P.table_size > 0x7fffffffull) throw Error(SF_INVALID_ARGUMENT, "grid: more than 2^31 blocks (N^3)");
    P.capacity = capacity;
    P.Nc = (P.N + (1 << kCoarseShift) - 1) >> kCoarseShift;
    P.mshift = -1;
    for (int b = 0; b < 16; ++b)
        if ((1 << b) == P.M) P.mshift = b;
    P.nshift = -1;
    for (int b = 0; b < 16; ++b)
        if ((1 << b) == P.N) P.nshift = b;
    P.occ_fine_words = (P.table_size + 31) / 32;
    const uint64_t nc = static_cast<uint64_t>(P.Nc);
    P.occ_coarse_words = (nc * nc * nc + 31) / 32;
    P.shard_rank = 0;
    P.shard_world = 1;
    P.shard_shift = 3;
    return P;
}

static void validate_config(const sf_grid_config& c) {
    // GridConfig::validate (grid.cpp:12-18)
    if (c.blocks_per_axis < 1 || c.voxels_per_block_axis < 1)
        throw Error(SF_INVALID_ARGUMENT, "grid: N and M must be >= 1");
    if (!(c.box_side > 0.0)) throw Error(SF_INVALID_ARGUMENT, "grid: box_side must be positive");
    const double voxel = c.box_side / (c.blocks_per_axis * c.voxels_per_block_axis);
    const double delta = c.truncation > 0.0 ? c.truncation : 4.0 * voxel;
    if (delta < 2.0 * voxel - 1e-12) throw Error(SF_INVALID_ARGUMENT, "grid: truncation must be >= 2 * voxel_size");
    if (static_cast<uint64_t>(c.blocks_per_axis) * c.blocks_per_axis * c.blocks_per_axis >= (1ull << 31))
        throw Error(SF_UNSUPPORTED, "grid: N^3 must be < 2^31 on the device path");
}

static uint64_t table_index_checked(const Volume& v, const int32_t bc[3]) {
    for (int i = 0; i < 3; ++i)
        if (bc[i] < 0 || bc[i] >= v.P.N) throw Error(SF_OUT_OF_RANGE, "grid: block coordinate out of range");
    return table_index(v.P, bc[0], bc[1], bc[2]);
}

static void grid_for(uint64_t n, int& blocks, int threads = 256) {
    const uint64_t b = (n + threads - 1) / threads;
    blocks = static_cast<int>(std::min<uint64_t>(std::max<uint64_t>(b, 1), 148ull * 32));
}

static void volume_init_device(Volume& v) {
    SF_CUDA(cudaSetDevice(v.device));
    const VolParams& P = v.P;
    const uint64_t pool_voxels = static_cast<uint64_t>(P.capacity) * P.M3;
    SF_CUDA(cudaMalloc(&v.d_table, P.table_size * sizeof(int32_t)));
    SF_CUDA(cudaMalloc(&v.d_payload, std::max<uint64_t>(pool_voxels, 1) * sizeof(uint16_t)));
    SF_CUDA(cudaMalloc(&v.d_free_list, std::max<uint32_t>(P.capacity, 1) * sizeof(int32_t)));
    SF_CUDA(cudaMalloc(&v.d_slot_key, std::max<uint32_t>(P.capacity, 1) * sizeof(int32_t)));
    const uint64_t occ_words = P.occ_fine_words + P.occ_coarse_words + 6;  // + bounding box
    SF_CUDA(cudaMalloc(&v.d_occ, occ_words * sizeof(uint32_t)));
    SF_CUDA(cudaMalloc(&v.d_keybits, P.occ_fine_words * sizeof(uint32_t)));
    SF_CUDA(cudaMemset(v.d_keybits, 0, P.occ_fine_words * sizeof(uint32_t)));
    SF_CUDA(cudaMalloc(&v.d_vc, sizeof(VolCounters)));
    SF_CUDA(cudaMalloc(&v.d_sched, 8 * sizeof(uint32_t)));
    SF_CUDA(cudaMemset(v.d_sched, 0, 8 * sizeof(uint32_t)));
    SF_CUDA(cudaMalloc(&v.d_aux, sizeof(AuxTables)));
    SF_CUDA(cudaMemset(v.d_table, 0xFF, P.table_size * sizeof(int32_t)));
    SF_CUDA(cudaMemset(v.d_occ, 0, occ_words * sizeof(uint32_t)));
    {
        const int empty_bb[6] = {INT32_MAX, INT32_MAX, INT32_MAX, -1, -1, -1};
        SF_CUDA(cudaMemcpy(v.d_occ + P.occ_fine_words + P.occ_coarse_words, empty_bb, sizeof(empty_bb),
                           cudaMemcpyHostToDevice));
    }
    int blocks;
    grid_for(pool_voxels, blocks);
    k_fill_u16<<<blocks, 256>>>(v.d_payload, pool_voxels, kChiPayload);
    SF_LAUNCH_CHECK();
    grid_for(P.capacity, blocks);
    k_init_free_list<<<blocks, 256>>>(v.d_free_list, v.d_slot_key, P.capacity);
    SF_LAUNCH_CHECK();
    VolCounters c{};
    c.free_top = P.capacity;
    SF_CUDA(cudaMemcpy(v.d_vc, &c, sizeof(c), cudaMemcpyHostToDevice));
    build_aux_tables(P, &v.h_aux);
    SF_CUDA(cudaMemcpy(v.d_aux, &v.h_aux, sizeof(AuxTables), cudaMemcpyHostToDevice));
    SF_CUDA(cudaDeviceSynchronize());
}

static void volume_free_device(Volume& v) {
    cudaSetDevice(v.device);
    v.fb.release();
    void* ptrs[] = {v.d_table, v.d_payload, v.d_fpayload, v.d_free_list, v.d_slot_key, v.d_occ, v.d_keybits,
                    v.d_vc,    v.d_aux,      v.d_sched, v.d_patch_order};
    for (void* p : ptrs)
        if (p) cudaFree(p);
}

// ---- STSG v1 snapshot (grid.cpp:333-408) -------------------------------------------
template <typename T>
static void put(std::ofstream& o, const T& v) {
    o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
template <typename T>
static T get(std::ifstream& i) {
    T v{};
    i.read(reinterpret_cast<char*>(&v), sizeof(T));
    return v;
}

extern "C" {

const char* sf_last_error(void) { return g_last_error.c_str(); }
const char* sf_version(void) { return "sf_gpu 0.1 sm_100a"; }

int sf_volume_create(const sf_grid_config* config, uint64_t pool_capacity, const sf_aux_quant* aux, int32_t device,
                     sf_volume_t* out) {
    return guarded([&]() -> int {
        if (!config || !out) throw Error(SF_INVALID_ARGUMENT, "sf_volume_create: null argument");
        validate_config(*config);
        sf_aux_quant a{0, 20.0, 1e-8, 1e-2};  // AuxQuantization defaults (grid.hpp:55-63)
        if (aux) a = *aux;
        const uint64_t n = static_cast<uint64_t>(config->blocks_per_axis);
        const uint64_t table = n * n * n;
        if (pool_capacity == 0) pool_capacity = std::max<uint64_t>(1, table / 8);  // grid.cpp:60
        if (pool_capacity > table) throw Error(SF_INVALID_ARGUMENT, "grid: pool_capacity must be <= N^3");
        auto v = std::make_unique<sf_volume>();
        v->device = device;
        v->cfg = *config;
        v->aux = a;
        v->P = make_params(*config, a, static_cast<uint32_t>(pool_capacity));
        volume_init_device(*v);
        *out = v.release();
        return SF_OK;
    });
}

int sf_volume_destroy(sf_volume_t vol) {
    if (!vol) return SF_OK;
    volume_free_device(*vol);
    delete vol;
    return SF_OK;
}

int sf_volume_set_shard(sf_volume_t v, int32_t rank, int32_t world, int32_t brick_shift) {
    return guarded([&]() -> int {
        if (!v) throw Error(SF_INVALID_ARGUMENT, "sf_volume_set_shard: null volume");
        if (world < 1 || rank < 0 || rank >= world || brick_shift < 0 || brick_shift > 16)
            throw Error(SF_INVALID_ARGUMENT, "sf_volume_set_shard: need 0 <= rank < world, 0 <= brick_shift <= 16");
        if (v->host_allocated() != 0)
            throw Error(SF_LOGIC_ERROR, "sf_volume_set_shard: the volume already holds blocks");
        v->P.shard_rank = rank;
        v->P.shard_world = world;
        v->P.shard_shift = brick_shift;
        return SF_OK;
    });
}

int32_t sf_shard_owner(int32_t bx, int32_t by, int32_t bz, int32_t brick_shift, int32_t world) {
    if (world < 1 || brick_shift < 0 || brick_shift > 16) return -1;
    return shard_owner(bx, by, bz, brick_shift, world);
}

int sf_volume_get_info(sf_volume_t v, sf_volume_info* out) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        VolCounters c;
        SF_CUDA(cudaMemcpy(&c, v->d_vc, sizeof(c), cudaMemcpyDeviceToHost));
        out->config = v->cfg;
        out->aux = v->aux;
        out->delta = v->P.delta;
        out->voxel_size = v->P.voxel;
        out->pool_capacity = v->P.capacity;
        out->allocated_count = c.allocated_count;
        // memory_bytes (grid.cpp:156-160)
        const uint64_t n = v->P.N, m = v->P.M;
        out->memory_bytes = 2ull * c.allocated_count * m * m * m + 4ull * n * n * n;
        return SF_OK;
    });
}

int sf_volume_allocate_block(sf_volume_t v, const int32_t bc[3], int32_t* slot_out) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        const uint64_t tidx = table_index_checked(*v, bc);
        int32_t* d_out;
        SF_CUDA(cudaMalloc(&d_out, 2 * sizeof(int32_t)));
        SF_CUDA(cudaMemset(d_out, 0, 2 * sizeof(int32_t)));
        k_allocate_one<<<1, 256>>>(v->P, v->d_table, v->d_free_list, v->d_slot_key, v->d_occ, v->d_payload,
                                   v->d_fpayload, v->d_vc, tidx, d_out);
        SF_LAUNCH_CHECK();
        int32_t h[2];
        SF_CUDA(cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost));
        SF_CUDA(cudaFree(d_out));
        if (h[0] == -2)
            throw Error(SF_POOL_EXHAUSTED, "grid: payload pool exhausted (" + std::to_string(v->P.capacity) +
                                               " blocks); increase pool capacity or lower resolution");
        *slot_out = h[0];
        return SF_OK;
    });
}

int sf_volume_free_block(sf_volume_t v, const int32_t bc[3]) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        const uint64_t tidx = table_index_checked(*v, bc);
        k_free_one<<<1, 256>>>(v->P, v->d_table, v->d_free_list, v->d_slot_key, v->d_occ, v->d_fpayload, v->d_vc,
                               tidx);
        SF_LAUNCH_CHECK();
        SF_CUDA(cudaDeviceSynchronize());
        return SF_OK;
    });
}

int sf_volume_block_slot(sf_volume_t v, const int32_t bc[3], int32_t* slot_out) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        const uint64_t tidx = table_index_checked(*v, bc);
        SF_CUDA(cudaMemcpy(slot_out, v->d_table + tidx, sizeof(int32_t), cudaMemcpyDeviceToHost));
        return SF_OK;
    });
}

// read_voxel (grid.cpp:121-130)
int sf_volume_read_voxel(sf_volume_t v, const int32_t vc[3], int32_t* is_chi, double* tsdf, double* aux) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "read_voxel");
        SF_CUDA(cudaSetDevice(v->device));
        for (int i = 0; i < 3; ++i)
            if (vc[i] < 0 || vc[i] >= v->P.res) throw Error(SF_OUT_OF_RANGE, "grid: voxel coordinate out of range");
        const int M = v->P.M;
        const int32_t bc[3] = {vc[0] / M, vc[1] / M, vc[2] / M};
        const uint64_t tidx = table_index(v->P, bc[0], bc[1], bc[2]);
        int32_t slot;
        SF_CUDA(cudaMemcpy(&slot, v->d_table + tidx, sizeof(slot), cudaMemcpyDeviceToHost));
        *is_chi = 1;
        *tsdf = 0.0;
        *aux = 0.0;
        if (slot == kEmpty) return SF_OK;
        const int lx = vc[0] - bc[0] * M, ly = vc[1] - bc[1] * M, lz = vc[2] - bc[2] * M;
        const uint64_t idx = static_cast<uint64_t>(slot) * v->P.M3 + (static_cast<uint64_t>(lz) * M + ly) * M + lx;
        uint16_t pl;
        SF_CUDA(cudaMemcpy(&pl, v->d_payload + idx, sizeof(pl), cudaMemcpyDeviceToHost));
        const int8_t code = static_cast<int8_t>(pl & 0xFF);
        const uint8_t ac = static_cast<uint8_t>(pl >> 8);
        if (code == kChiCode) return SF_OK;
        *is_chi = 0;
        *tsdf = dequantize_tsdf(code, v->P.delta);
        *aux = v->h_aux.aux_decode[ac];
        return SF_OK;
    });
}

// write_voxel (grid.cpp:132-154)
int sf_volume_write_voxel(sf_volume_t v, const int32_t vc[3], int32_t tsdf_is_chi, double tsdf, double aux) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "write_voxel");
        SF_CUDA(cudaSetDevice(v->device));
        for (int i = 0; i < 3; ++i)
            if (vc[i] < 0 || vc[i] >= v->P.res) throw Error(SF_OUT_OF_RANGE, "grid: voxel coordinate out of range");
        bool chi = tsdf_is_chi != 0;
        if (!chi && std::abs(tsdf) > v->P.delta) chi = true;
        const int M = v->P.M;
        const int32_t bc[3] = {vc[0] / M, vc[1] / M, vc[2] / M};
        const uint64_t tidx = table_index(v->P, bc[0], bc[1], bc[2]);
        int32_t slot;
        SF_CUDA(cudaMemcpy(&slot, v->d_table + tidx, sizeof(slot), cudaMemcpyDeviceToHost));
        if (slot == kEmpty) {
            if (chi) return SF_OK;
            throw Error(SF_LOGIC_ERROR, "grid: write to unallocated block (allocate first)");
        }
        const int lx = vc[0] - bc[0] * M, ly = vc[1] - bc[1] * M, lz = vc[2] - bc[2] * M;
        const uint64_t idx = static_cast<uint64_t>(slot) * v->P.M3 + (static_cast<uint64_t>(lz) * M + ly) * M + lx;
        uint16_t pl = kChiPayload;
        if (!chi) {
            const int8_t code = quantize_tsdf(tsdf, v->P.delta);
            const uint8_t ac = host_aux_encode(v->P, aux);
            pl = static_cast<uint16_t>(static_cast<uint8_t>(code)) | static_cast<uint16_t>(ac << 8);
        }
        SF_CUDA(cudaMemcpy(v->d_payload + idx, &pl, sizeof(pl), cudaMemcpyHostToDevice));
        if (v->d_fpayload) {
            const float2 f = chi ? make_float2(INFINITY, 0.0f)
                                 : make_float2(static_cast<float>(tsdf), static_cast<float>(aux));
            SF_CUDA(cudaMemcpy(v->d_fpayload + idx, &f, sizeof(f), cudaMemcpyHostToDevice));
        }
        return SF_OK;
    });
}

int sf_volume_read_table(sf_volume_t v, int32_t* host_table) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        SF_CUDA(cudaMemcpy(host_table, v->d_table, v->P.table_size * sizeof(int32_t), cudaMemcpyDeviceToHost));
        return SF_OK;
    });
}

int sf_volume_read_payload(sf_volume_t v, uint64_t first, uint64_t count, uint16_t* out) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "read_payload");
        SF_CUDA(cudaSetDevice(v->device));
        if (first + count > v->P.capacity) throw Error(SF_OUT_OF_RANGE, "payload range");
        SF_CUDA(cudaMemcpy(out, v->d_payload + first * v->P.M3, count * v->P.M3 * sizeof(uint16_t),
                           cudaMemcpyDeviceToHost));
        return SF_OK;
    });
}

int sf_volume_write_payload(sf_volume_t v, uint64_t first, uint64_t count, const uint16_t* in) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "write_payload");
        SF_CUDA(cudaSetDevice(v->device));
        if (first + count > v->P.capacity) throw Error(SF_OUT_OF_RANGE, "payload range");
        SF_CUDA(cudaMemcpy(v->d_payload + first * v->P.M3, in, count * v->P.M3 * sizeof(uint16_t),
                           cudaMemcpyHostToDevice));
        return SF_OK;
    });
}

int sf_volume_read_free_list(sf_volume_t v, int32_t* out, uint64_t* count_out) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        VolCounters c;
        SF_CUDA(cudaMemcpy(&c, v->d_vc, sizeof(c), cudaMemcpyDeviceToHost));
        if (out && c.free_top)
            SF_CUDA(cudaMemcpy(out, v->d_free_list, c.free_top * sizeof(int32_t), cudaMemcpyDeviceToHost));
        *count_out = c.free_top;
        return SF_OK;
    });
}

int sf_volume_enable_float_payload(sf_volume_t v) {
    return guarded([&]() -> int {
        if (!v) throw Error(SF_INVALID_ARGUMENT, "sf_volume_enable_float_payload: null volume");
        SF_CUDA(cudaSetDevice(v->device));
        if (v->d_fpayload) return SF_OK;
        v->layout = SF_PAYLOAD_CODES_FLOAT_SHADOW;
        const uint64_t n = static_cast<uint64_t>(v->P.capacity) * v->P.M3;
        SF_CUDA(cudaMalloc(&v->d_fpayload, std::max<uint64_t>(n, 1) * sizeof(float2)));
        int blocks;
        grid_for(n, blocks);
        k_fill_f2<<<blocks, 256>>>(v->d_fpayload, n, make_float2(INFINITY, 0.0f));
        SF_LAUNCH_CHECK();
        SF_CUDA(cudaDeviceSynchronize());
        return SF_OK;
    });
}

int sf_volume_set_payload_layout(sf_volume_t v, int32_t layout) {
    return guarded([&]() -> int {
        if (!v) throw Error(SF_INVALID_ARGUMENT, "sf_volume_set_payload_layout: null volume");
        if (layout < SF_PAYLOAD_CODES || layout > SF_PAYLOAD_FLOAT2)
            throw Error(SF_INVALID_ARGUMENT, "sf_volume_set_payload_layout: unknown layout");
        if (layout == v->layout) return SF_OK;
        if (layout == SF_PAYLOAD_CODES_FLOAT_SHADOW && v->layout == SF_PAYLOAD_CODES)
            return sf_volume_enable_float_payload(v);
        if (v->host_allocated() != 0)
            throw Error(SF_LOGIC_ERROR, "sf_volume_set_payload_layout: the volume must be empty to change layout");
        if (layout == SF_PAYLOAD_CODES) {
            SF_CUDA(cudaSetDevice(v->device));
            if (v->d_fpayload) SF_CUDA(cudaFree(v->d_fpayload));
            v->d_fpayload = nullptr;
            v->layout = SF_PAYLOAD_CODES;
            return SF_OK;
        }
        const int rc = sf_volume_enable_float_payload(v);
        if (rc != SF_OK) return rc;
        v->layout = layout;
        return SF_OK;
    });
}

int sf_volume_get_payload_layout(sf_volume_t v, int32_t* layout) {
    return guarded([&]() -> int {
        if (!v || !layout) throw Error(SF_INVALID_ARGUMENT, "sf_volume_get_payload_layout: null argument");
        *layout = v->layout;
        return SF_OK;
    });
}

int sf_volume_read_float_payload(sf_volume_t v, uint64_t first, uint64_t count, float* out) {
    return guarded([&]() -> int {
        SF_CUDA(cudaSetDevice(v->device));
        if (!v->d_fpayload) throw Error(SF_LOGIC_ERROR, "float payload not enabled");
        if (first + count > v->P.capacity) throw Error(SF_OUT_OF_RANGE, "payload range");
        SF_CUDA(cudaMemcpy(out, v->d_fpayload + first * v->P.M3, count * v->P.M3 * sizeof(float2),
                           cudaMemcpyDeviceToHost));
        return SF_OK;
    });
}

int sf_volume_save_snapshot(sf_volume_t v, const char* path) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "save_snapshot");
        SF_CUDA(cudaSetDevice(v->device));
        std::vector<int32_t> table(v->P.table_size);
        SF_CUDA(cudaMemcpy(table.data(), v->d_table, table.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
        std::ofstream out(path, std::ios::binary);
        if (!out) throw Error(SF_IO_ERROR, std::string("grid: cannot open ") + path + " for writing");
        out.write("STSG", 4);
        put<uint32_t>(out, 1u);
        put<uint32_t>(out, static_cast<uint32_t>(v->cfg.blocks_per_axis));
        put<uint32_t>(out, static_cast<uint32_t>(v->cfg.voxels_per_block_axis));
        for (int i = 0; i < 3; ++i) put<double>(out, v->cfg.box_origin[i]);
        put<double>(out, v->cfg.box_side);
        put<double>(out, v->P.delta);
        put<uint8_t>(out, v->aux.mode == 0 ? 0 : 1);
        put<double>(out, v->aux.w_max);
        put<double>(out, v->aux.p_min);
        put<double>(out, v->aux.p_max);
        out.write(reinterpret_cast<const char*>(table.data()), table.size() * sizeof(int32_t));
        std::vector<int32_t> slots;
        for (int32_t s : table)
            if (s != kEmpty) slots.push_back(s);
        std::sort(slots.begin(), slots.end());
        std::vector<uint16_t> pl(v->P.M3);
        for (int32_t s : slots) {
            SF_CUDA(cudaMemcpy(pl.data(), v->d_payload + static_cast<uint64_t>(s) * v->P.M3,
                               pl.size() * sizeof(uint16_t), cudaMemcpyDeviceToHost));
            out.write(reinterpret_cast<const char*>(pl.data()), pl.size() * sizeof(uint16_t));
        }
        if (!out) throw Error(SF_IO_ERROR, std::string("grid: write failed for ") + path);
        return SF_OK;
    });
}

int sf_volume_load_snapshot(const char* path, uint64_t pool_capacity, int32_t device, sf_volume_t* out) {
    return guarded([&]() -> int {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw Error(SF_IO_ERROR, std::string("grid: cannot open ") + path);
        char magic[4];
        in.read(magic, 4);
        if (!in || std::strncmp(magic, "STSG", 4) != 0)
            throw Error(SF_IO_ERROR, std::string("grid: ") + path + " is not a STSG snapshot");
        if (get<uint32_t>(in) != 1u) throw Error(SF_IO_ERROR, "grid: unsupported STSG version");
        sf_grid_config cfg{};
        cfg.blocks_per_axis = static_cast<int32_t>(get<uint32_t>(in));
        cfg.voxels_per_block_axis = static_cast<int32_t>(get<uint32_t>(in));
        for (int i = 0; i < 3; ++i) cfg.box_origin[i] = get<double>(in);
        cfg.box_side = get<double>(in);
        cfg.truncation = get<double>(in);
        sf_aux_quant aux{};
        aux.mode = get<uint8_t>(in) == 0 ? 0 : 1;
        aux.w_max = get<double>(in);
        aux.p_min = get<double>(in);
        aux.p_max = get<double>(in);
        const uint64_t n = static_cast<uint64_t>(cfg.blocks_per_axis);
        std::vector<int32_t> table(n * n * n);
        in.read(reinterpret_cast<char*>(table.data()), table.size() * sizeof(int32_t));
        std::vector<std::pair<int32_t, uint64_t>> slot_to_table;
        for (uint64_t i = 0; i < table.size(); ++i)
            if (table[i] != kEmpty) slot_to_table.emplace_back(table[i], i);
        std::sort(slot_to_table.begin(), slot_to_table.end());
        if (pool_capacity == 0)
            pool_capacity = std::max<uint64_t>({1, slot_to_table.size(), n * n * n / 8});
        sf_volume_t v = nullptr;
        int st = sf_volume_create(&cfg, pool_capacity, &aux, device, &v);
        if (st != SF_OK) throw Error(st, sf_last_error());
        std::unique_ptr<sf_volume, int (*)(sf_volume_t)> guard(v, sf_volume_destroy);
        // Re-allocation in slot order on a fresh grid hands out slots 0, 1, 2, ... (grid.cpp:398-405).
        const uint64_t count = slot_to_table.size();
        if (count > v->P.capacity)
            throw Error(SF_POOL_EXHAUSTED, "grid: payload pool exhausted (" + std::to_string(v->P.capacity) +
                                               " blocks); increase pool capacity or lower resolution");
        std::vector<int32_t> new_table(table.size(), kEmpty);
        std::vector<uint16_t> payload(count * v->P.M3);
        for (uint64_t k = 0; k < count; ++k) new_table[slot_to_table[k].second] = static_cast<int32_t>(k);
        in.read(reinterpret_cast<char*>(payload.data()), payload.size() * sizeof(uint16_t));
        if (!in) throw Error(SF_IO_ERROR, std::string("grid: truncated STSG snapshot ") + path);
        SF_CUDA(cudaMemcpy(v->d_table, new_table.data(), new_table.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        if (count)
            SF_CUDA(cudaMemcpy(v->d_payload, payload.data(), payload.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
        VolCounters c{};
        c.allocated_count = count;
        c.free_top = v->P.capacity - count;
        c.high_water = count;
        SF_CUDA(cudaMemcpy(v->d_vc, &c, sizeof(c), cudaMemcpyHostToDevice));
        int blocks;
        grid_for(v->P.table_size, blocks);
        k_rebuild_index<<<blocks, 256>>>(v->P, v->d_table, v->d_slot_key, v->d_occ);
        SF_LAUNCH_CHECK();
        SF_CUDA(cudaDeviceSynchronize());
        *out = guard.release();
        return SF_OK;
    });
}

// Bulk import of a host grid's complete state into a FRESH volume (the C++ drop-in layer keeps
// the reference's host SparseTsdfGrid as the source of truth and mirrors it per call):
// offset table, payload slots [0, slot_count), the free-list stack (bottom to top).
int sf_volume_import_state(sf_volume_t v, const int32_t* table, const uint16_t* payload, uint64_t slot_count,
                           const int32_t* free_list, uint64_t free_count) {
    return guarded([&]() -> int {
        if (!v || !table || (slot_count && !payload) || (free_count && !free_list))
            throw Error(SF_INVALID_ARGUMENT, "sf_volume_import_state: null argument");
        SF_CUDA(cudaSetDevice(v->device));
        if (v->host_allocated() != 0) throw Error(SF_LOGIC_ERROR, "sf_volume_import_state: volume not empty");
        if (slot_count > v->P.capacity || free_count > v->P.capacity)
            throw Error(SF_OUT_OF_RANGE, "sf_volume_import_state: more slots than the pool capacity");
        uint64_t allocated = 0, high = 0;
        for (uint64_t i = 0; i < v->P.table_size; ++i)
            if (table[i] != kEmpty) {
                if (table[i] < 0 || static_cast<uint64_t>(table[i]) >= v->P.capacity)
                    throw Error(SF_OUT_OF_RANGE, "sf_volume_import_state: slot out of range");
                ++allocated;
                high = std::max<uint64_t>(high, static_cast<uint64_t>(table[i]) + 1);
            }
        if (allocated + free_count != v->P.capacity)
            throw Error(SF_LOGIC_ERROR, "sf_volume_import_state: allocated + free != capacity");
        SF_CUDA(cudaMemcpy(v->d_table, table, v->P.table_size * sizeof(int32_t), cudaMemcpyHostToDevice));
        if (slot_count)
            SF_CUDA(cudaMemcpy(v->d_payload, payload, slot_count * v->P.M3 * sizeof(uint16_t), cudaMemcpyHostToDevice));
        if (free_count)
            SF_CUDA(cudaMemcpy(v->d_free_list, free_list, free_count * sizeof(int32_t), cudaMemcpyHostToDevice));
        VolCounters c{};
        c.allocated_count = allocated;
        c.free_top = free_count;
        c.high_water = high;
        SF_CUDA(cudaMemcpy(v->d_vc, &c, sizeof(c), cudaMemcpyHostToDevice));
        int blocks;
        grid_for(v->P.table_size, blocks);
        k_rebuild_index<<<blocks, 256>>>(v->P, v->d_table, v->d_slot_key, v->d_occ);
        SF_LAUNCH_CHECK();
        SF_CUDA(cudaDeviceSynchronize());
        return SF_OK;
    });
}

int sf_volume_write_float_payload(sf_volume_t v, uint64_t first, uint64_t count, const float* in) {
    return guarded([&]() -> int {
        if (!v || (count && !in)) throw Error(SF_INVALID_ARGUMENT, "sf_volume_write_float_payload: null argument");
        SF_CUDA(cudaSetDevice(v->device));
        if (!v->d_fpayload) throw Error(SF_LOGIC_ERROR, "float payload not enabled");
        if (first + count > v->P.capacity) throw Error(SF_OUT_OF_RANGE, "payload range");
        SF_CUDA(cudaMemcpy(v->d_fpayload + first * v->P.M3, in, count * v->P.M3 * sizeof(float2),
                           cudaMemcpyHostToDevice));
        return SF_OK;
    });
}

// Host-only introspection of the aux codec tables (used by the CPU test-suite to check the
// threshold encode against the reference's log-based encode without a GPU).
int sf_debug_aux_tables(const sf_aux_quant* aux, double delta, double* tsdf_decode, double* aux_decode,
                        double* aux_thresh) {
    return guarded([&]() -> int {
        VolParams P{};
        P.delta = delta;
        P.aux_mode = aux->mode;
        P.aux_w_max = aux->w_max;
        P.aux_p_min = aux->p_min;
        P.aux_p_max = aux->p_max;
        AuxTables t;
        build_aux_tables(P, &t);
        std::memcpy(tsdf_decode, t.tsdf_decode, sizeof(t.tsdf_decode));
        std::memcpy(aux_decode, t.aux_decode, sizeof(t.aux_decode));
        std::memcpy(aux_thresh, t.aux_thresh, sizeof(t.aux_thresh));
        return SF_OK;
    });
}

}  // extern "C"
