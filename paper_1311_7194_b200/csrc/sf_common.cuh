// sf_common.cuh — shared device/host numerics and POD layouts for the sparse-TSDF path.
//
// PARITY CONTRACT. Every geometric quantity is computed in FP64 with the reference's
// operation order (the order of /root/reference/proj/src/*.cpp evaluated through the
// Eigen-API definition in oracle/shim/Eigen/Dense), and the whole library is compiled
// with -fmad=false (device) / -ffp-contract=off (host), so products and sums are never
// contracted into FMAs. IEEE division and sqrt are correctly rounded in CUDA FP64, so
// the device reproduces the reference's doubles bit for bit. Transcendentals (log/exp in
// the aux codec, cos in MatchParams) are evaluated on the HOST with the same libm as the
// reference and shipped to the device as tables / scalars.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef SF_HD
#define SF_HD __host__ __device__ __forceinline__
#endif

namespace sf {

// Device clock (ns); used for in-kernel span measurements.
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr int32_t kEmpty = -1;          // SparseTsdfGrid::kEmpty (grid.hpp:98)
constexpr int8_t kChiCode = -128;       // grid.hpp:19
constexpr int kTsdfCodeRange = 127;     // grid.hpp:21
constexpr uint16_t kChiPayload = 0x0080; // VoxelPayload{-128, 0}: low byte tsdf, high byte aux

struct d3 {
    double x, y, z;
};

SF_HD d3 mk(double x, double y, double z) { return d3{x, y, z}; }
SF_HD d3 add(d3 a, d3 b) { return d3{a.x + b.x, a.y + b.y, a.z + b.z}; }
SF_HD d3 sub(d3 a, d3 b) { return d3{a.x - b.x, a.y - b.y, a.z - b.z}; }
SF_HD d3 neg(d3 a) { return d3{-a.x, -a.y, -a.z}; }
SF_HD d3 scale(double s, d3 a) { return d3{s * a.x, s * a.y, s * a.z}; }  // Eigen: s * v
SF_HD d3 divs(d3 a, double s) { return d3{a.x / s, a.y / s, a.z / s}; }   // Eigen: v / s
SF_HD d3 cmul(d3 a, d3 b) { return d3{a.x * b.x, a.y * b.y, a.z * b.z}; } // cwiseProduct
SF_HD double dot(d3 a, d3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
SF_HD double sqnorm(d3 a) { return dot(a, a); }
SF_HD d3 cross(d3 a, d3 b) {
    return d3{a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
// Eigen normalized(): v / sqrt(squaredNorm) when squaredNorm > 0.
SF_HD d3 normalized(d3 a) {
    const double z = sqnorm(a);
    if (z > 0.0) return divs(a, sqrt(z));
    return a;
}
SF_HD double dmin(double a, double b) { return (b < a) ? b : a; }  // std::min(a, b)
SF_HD double dmax(double a, double b) { return (a < b) ? b : a; }  // std::max(a, b)
SF_HD double dclamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

// 3x3 matrices, row-major m[r*3+c].
struct m33 {
    double m[9];
};
SF_HD d3 mv(const m33& R, d3 v) {
    return d3{(R.m[0] * v.x + R.m[1] * v.y) + R.m[2] * v.z, (R.m[3] * v.x + R.m[4] * v.y) + R.m[5] * v.z,
              (R.m[6] * v.x + R.m[7] * v.y) + R.m[8] * v.z};
}
SF_HD m33 mt(const m33& R) {
    m33 t;
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) t.m[c * 3 + r] = R.m[r * 3 + c];
    return t;
}
SF_HD m33 mm(const m33& A, const m33& B) {
    m33 r;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j)
            r.m[i * 3 + j] = (A.m[i * 3 + 0] * B.m[0 * 3 + j] + A.m[i * 3 + 1] * B.m[1 * 3 + j]) +
                             A.m[i * 3 + 2] * B.m[2 * 3 + j];
    return r;
}
SF_HD d3 col(const m33& R, int c) { return d3{R.m[c], R.m[3 + c], R.m[6 + c]}; }

// Pose (pose.hpp:9-16): x_w = R x_c + t.
struct Pose {
    m33 R;
    d3 t;
};
SF_HD d3 apply(const Pose& p, d3 x) { return add(mv(p.R, x), p.t); }
// compose (pose.cpp:6-11)
SF_HD Pose compose(const Pose& a, const Pose& b) {
    Pose o;
    o.R = mm(a.R, b.R);
    o.t = add(mv(a.R, b.t), a.t);
    return o;
}
// invert (pose.cpp:13-18)
SF_HD Pose invert(const Pose& a) {
    Pose o;
    o.R = mt(a.R);
    o.t = neg(mv(o.R, a.t));
    return o;
}
SF_HD Pose pose_from12(const double* p) {
    Pose o;
    for (int i = 0; i < 9; ++i) o.R.m[i] = p[i];
    o.t = d3{p[9], p[10], p[11]};
    return o;
}
SF_HD void pose_to12(const Pose& o, double* p) {
    for (int i = 0; i < 9; ++i) p[i] = o.R.m[i];
    p[9] = o.t.x;
    p[10] = o.t.y;
    p[11] = o.t.z;
}

// Intrinsics (camera.hpp:9-24) as a POD.
struct Intr {
    int w, h;
    double fx, fy, cx, cy, near_plane, far_plane;
};
// unproject (camera.cpp:31-33)
SF_HD d3 unproject(const Intr& I, double u, double v, double depth) {
    return d3{(u - I.cx) / I.fx * depth, (v - I.cy) / I.fy * depth, depth};
}
// project (camera.cpp:35-42); returns false when !(z > 0).
SF_HD bool project(const Intr& I, d3 p, double& u, double& v) {
    if (!(p.z > 0.0)) return false;
    u = I.fx * p.x / p.z + I.cx;
    v = I.fy * p.y / p.z + I.cy;
    return true;
}

// static_cast<int>(std::lround(x)) as compiled by g++ on x86-64: glibc lround (half away
// from zero; out-of-range / NaN -> LONG_MIN via cvttsd2si), then truncation to 32 bits.
SF_HD int ref_lround_int(double x) {
    long long r;
    if (!(fabs(x) < 9223372036854775808.0)) r = (long long)0x8000000000000000ULL;
    else r = llround(x);
    return (int)(unsigned int)(unsigned long long)r;
}
// static_cast<int>(double) on x86-64 (cvttsd2si): truncation, INT_MIN when out of range / NaN.
SF_HD int ref_to_int(double x) {
    if (!(x > -2147483649.0 && x < 2147483648.0)) return (int)0x80000000u;
    return (int)x;
}
SF_HD int ref_floor_int(double x) { return ref_to_int(floor(x)); }

// ---- conversion-free exact helpers (device hot loops) --------------------------------
// FP64 <-> integer conversions and floor/round run on the SM's low-rate XU pipe; these
// equivalents use the FP64 add pipe and integer ALU only (magic number 1.5 * 2^52).
constexpr double kMagic52 = 6755399441055744.0;
// (double)n, exact for |n| < 2^51
__device__ __forceinline__ double i2d_exact(long long n) {
    return __longlong_as_double(__double_as_longlong(kMagic52) + n) - kMagic52;
}
// floor(x) as (double, int), exact for |x| < 2^30 (caller checks the range)
__device__ __forceinline__ double floor_exact(double x, int& xi) {
    const double t = x + kMagic52;  // round to nearest integer (ties to even)
    double n = t - kMagic52;
    int ni = static_cast<int>(static_cast<unsigned int>(__double_as_longlong(t)));
    if (n > x) {
        n -= 1.0;
        ni -= 1;
    }
    xi = ni;
    return n;
}
// static_cast<int>(std::floor(x)) (ref_floor_int) via floor_exact when |x| < 2^30.
__device__ __forceinline__ int ref_floor_int_fast(double x) {
    if (!(fabs(x) < 1073741824.0)) return ref_floor_int(x);
    int xi;
    floor_exact(x, xi);
    return xi;
}
// std::lround(a) when it is certain under the margin e (a not within e of k + 1/2).
__device__ __forceinline__ bool certain_lround_fast(double a, double e, int& out) {
    if (!(fabs(a) < 1e9)) return false;
    const double t = a + kMagic52;
    const double n = t - kMagic52;  // nearest integer
    const double d = a - n;          // exact, |d| <= 1/2
    out = static_cast<int>(static_cast<unsigned int>(__double_as_longlong(t)));
    return fabs(d) < 0.5 - e;
}

// Quantizers (grid.cpp:20-27): lround(clamp(d,-delta,delta) / delta * 127).
SF_HD int8_t quantize_tsdf(double d, double delta) {
    const double clamped = dclamp(d, -delta, delta);
    return (int8_t)(long long)llround(clamped / delta * (double)kTsdfCodeRange);
}
SF_HD double dequantize_tsdf(int8_t code, double delta) { return (double)code / (double)kTsdfCodeRange * delta; }

// Volume parameters shared by every kernel (by value).
struct VolParams {
    int N, M, M3, res;  // blocks/axis, voxels/block axis, M^3, N*M
    double ox, oy, oz;  // box origin
    double box_side, voxel, block_side, delta;
    int aux_mode;  // 0 weight, 1 variance
    double aux_w_max, aux_p_min, aux_p_max;
    uint64_t table_size;  // N^3
    uint32_t capacity;
    int mshift;               // log2(M) when M is a power of two, else -1
    int Nc;                   // coarse occupancy lattice: ceil(N / 16) super-blocks per axis
    uint64_t occ_fine_words;    // uint32 words of the fine (per-block) bitmap; coarse bits follow
    uint64_t occ_coarse_words;  // uint32 words of the coarse bitmap; 6 ints of bounding box follow
    double inv_voxel;           // RN(1 / voxel): Markstein-corrected division by voxel (sf_render.cu)
    double inv_block_side;      // RN(1 / block_side): the same for block keys (sf_fusion.cu)
    double aux_lg_pmin, aux_lg_scale;
    int nshift;  // log2(N) when N is a power of two, else -1  // variance codes: log2(p_min), 255 / log2(p_max / p_min) (code guess)
    // Spatial sharding: this volume allocates only the blocks it owns,
    // owner = hash of the (2^shard_shift)^3-block brick % shard_world. world 1 = owns all.
    int shard_rank, shard_world, shard_shift;
};

// Owner rank of block (bx, by, bz) under brick sharding (identical on host and device).
SF_HD int shard_owner(int bx, int by, int bz, int shift, int world) {
    const uint32_t x = static_cast<uint32_t>(bx) >> shift, y = static_cast<uint32_t>(by) >> shift,
                   z = static_cast<uint32_t>(bz) >> shift;
    uint32_t hsh = x * 0x9E3779B1u ^ y * 0x85EBCA77u ^ z * 0xC2B2AE3Du;
    hsh ^= hsh >> 15;
    hsh *= 0x2C1B3C6Du;
    hsh ^= hsh >> 12;
    return static_cast<int>(hsh % static_cast<uint32_t>(world));
}
SF_HD bool shard_owns(const VolParams& P, int bx, int by, int bz) {
    return P.shard_world <= 1 || shard_owner(bx, by, bz, P.shard_shift, P.shard_world) == P.shard_rank;
}

constexpr int kCoarseShift = 4;  // super-block = 16^3 blocks

// Occupancy bitmaps (fine: 1 bit per block; coarse: 1 bit per 16^3 super-block, set when
// any block in it was ever allocated — a conservative filter, never cleared on free).
// Block-coordinate bounding box of every block ever allocated: {xlo, ylo, zlo, xhi, yhi, zhi}
// (empty: lo > hi). Grown on allocation, never shrunk: a conservative filter like the coarse bits.
SF_HD const int* occ_bbox(const VolParams& P, const uint32_t* occ) {
    return reinterpret_cast<const int*>(occ + P.occ_fine_words + P.occ_coarse_words);
}
__device__ __forceinline__ void occ_set(const VolParams& P, uint32_t* occ, uint64_t key) {
    atomicOr(&occ[key >> 5], 1u << (key & 31));
    const uint64_t x = key % P.N, y = (key / P.N) % P.N, z = key / ((uint64_t)P.N * P.N);
    const uint64_t c = ((z >> kCoarseShift) * P.Nc + (y >> kCoarseShift)) * P.Nc + (x >> kCoarseShift);
    atomicOr(&occ[P.occ_fine_words + (c >> 5)], 1u << (c & 31));
    int* bb = reinterpret_cast<int*>(occ + P.occ_fine_words + P.occ_coarse_words);
    atomicMin(&bb[0], (int)x);
    atomicMin(&bb[1], (int)y);
    atomicMin(&bb[2], (int)z);
    atomicMax(&bb[3], (int)x);
    atomicMax(&bb[4], (int)y);
    atomicMax(&bb[5], (int)z);
}

// voxel_center (grid.cpp:271-273): origin + (vc + 0.5) * voxel_size
SF_HD d3 voxel_center(const VolParams& P, int x, int y, int z) {
    return d3{P.ox + ((double)x + 0.5) * P.voxel, P.oy + ((double)y + 0.5) * P.voxel,
              P.oz + ((double)z + 0.5) * P.voxel};
}
// the same values without int->double conversions (exact for |coordinate| < 2^51)
__device__ __forceinline__ d3 voxel_center_fast(const VolParams& P, int x, int y, int z) {
    return d3{P.ox + (i2d_exact(x) + 0.5) * P.voxel, P.oy + (i2d_exact(y) + 0.5) * P.voxel,
              P.oz + (i2d_exact(z) + 0.5) * P.voxel};
}
// block_min_corner (grid.cpp:275-277): origin + bc * block_side
SF_HD d3 block_min_corner(const VolParams& P, int x, int y, int z) {
    return d3{P.ox + (double)x * P.block_side, P.oy + (double)y * P.block_side, P.oz + (double)z * P.block_side};
}
SF_HD uint64_t table_index(const VolParams& P, int x, int y, int z) {
    return ((uint64_t)z * (uint64_t)P.N + (uint64_t)y) * (uint64_t)P.N + (uint64_t)x;
}

// Per-frame constants derived from (pose, intrinsics), computed on the device by one
// thread (so a device-resident ICP pose never round-trips to the host).
constexpr int kSatAxes = 26;  // 3 box + 5 frustum + 6x3 edge crosses (grid.cpp:208-216)
struct FrameConsts {
    Pose pose;        // camera -> world
    Pose inv;         // world -> camera (invert(pose))
    Intr intr;
    double delta;     // grid delta (fusion params.delta := grid.delta(), fusion.cpp:278)
    // Frustum SAT (grid.cpp:228-269): axis vector, frustum projection interval, validity.
    d3 sat_axis[kSatAxes];
    double sat_lo[kSatAxes], sat_hi[kSatAxes];
    int sat_valid[kSatAxes];
    // Inward unit normals (camera frame) of the four side faces of the frustum pyramid: a
    // conservative "block strictly inside" test that skips the SAT for most blocks.
    d3 side_n[4];
};

// Fusion parameters (fusion.hpp:18-31) resolved on the host.
struct FuseParams {
    int mode;  // 0 simple, 1 weighted, 2 kalman
    double w_fixed, w_max, q, sigma0, min_variance;
    int downweight;
    int has_sigma;
    int refine;  // refinement_steps (fusion.hpp:25): sub-pixel descent (generic kernel)
};

}  // namespace sf
