/*
 * sf_oracle.c — plain-C restatement of the reference hot path (TEST INFRASTRUCTURE ONLY;
 * see sf_oracle.h). Every function cites the reference lines it follows; paths are relative
 * to /root/reference/proj. Sequential, single-threaded, FP64, -ffp-contract=off.
 */
#define _GNU_SOURCE
#include "sf_oracle.h"

#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------------------------------
 * errors
 * ------------------------------------------------------------------------------------- */
static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* sfo_last_error(void) { return g_err; }

/* ---------------------------------------------------------------------------------------
 * vectors / poses (Eigen-shim evaluation order: left-to-right sums)
 * ------------------------------------------------------------------------------------- */
typedef struct {
    double x, y, z;
} v3;
typedef struct {
    double R[9]; /* row-major */
    v3 t;
} pose_t;

static v3 V(double x, double y, double z) {
    v3 r = {x, y, z};
    return r;
}
static v3 vadd(v3 a, v3 b) { return V(a.x + b.x, a.y + b.y, a.z + b.z); }
static v3 vsub(v3 a, v3 b) { return V(a.x - b.x, a.y - b.y, a.z - b.z); }
static v3 vscale(double s, v3 a) { return V(s * a.x, s * a.y, s * a.z); }
static v3 vdivs(v3 a, double s) { return V(a.x / s, a.y / s, a.z / s); }
static v3 vmul(v3 a, v3 b) { return V(a.x * b.x, a.y * b.y, a.z * b.z); }
static double vdot(v3 a, v3 b) { return (a.x * b.x + a.y * b.y) + a.z * b.z; }
static v3 vcross(v3 a, v3 b) { return V(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x); }
static v3 vnormalized(v3 a) { /* Eigen normalized() */
    const double z = vdot(a, a);
    return z > 0.0 ? vdivs(a, sqrt(z)) : a;
}
static double dmin(double a, double b) { return (b < a) ? b : a; } /* std::min */
static double dmax(double a, double b) { return (a < b) ? b : a; } /* std::max */
static double dclamp(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

static v3 mv(const double* R, v3 v) {
    return V((R[0] * v.x + R[1] * v.y) + R[2] * v.z, (R[3] * v.x + R[4] * v.y) + R[5] * v.z,
             (R[6] * v.x + R[7] * v.y) + R[8] * v.z);
}
static void mm(const double* A, const double* B, double* out) {
    double r[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r[i * 3 + j] = (A[i * 3] * B[j] + A[i * 3 + 1] * B[3 + j]) + A[i * 3 + 2] * B[6 + j];
    memcpy(out, r, sizeof r);
}
static void mtrans(const double* A, double* out) {
    double r[9];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) r[j * 3 + i] = A[i * 3 + j];
    memcpy(out, r, sizeof r);
}
static pose_t pose_from(const double* p) {
    pose_t o;
    memcpy(o.R, p, 9 * sizeof(double));
    o.t = V(p[9], p[10], p[11]);
    return o;
}
static void pose_to(pose_t o, double* p) {
    memcpy(p, o.R, 9 * sizeof(double));
    p[9] = o.t.x;
    p[10] = o.t.y;
    p[11] = o.t.z;
}
static v3 papply(const pose_t* p, v3 x) { return vadd(mv(p->R, x), p->t); } /* pose.hpp:12 */
static pose_t compose(const pose_t* a, const pose_t* b) {                    /* pose.cpp:6-11 */
    pose_t o;
    mm(a->R, b->R, o.R);
    o.t = vadd(mv(a->R, b->t), a->t);
    return o;
}
static pose_t invert(const pose_t* a) { /* pose.cpp:13-18 */
    pose_t o;
    mtrans(a->R, o.R);
    v3 t = mv(o.R, a->t);
    o.t = V(-t.x, -t.y, -t.z);
    return o;
}

/* static_cast<int>(std::lround(x)) / static_cast<int>(std::floor(x)) on x86-64 g++ */
static int ref_lround_int(double x) {
    long long r;
    if (!(fabs(x) < 9223372036854775808.0)) r = (long long)0x8000000000000000ULL;
    else r = llround(x);
    return (int)(unsigned int)(unsigned long long)r;
}
static int ref_to_int(double x) {
    if (!(x > -2147483649.0 && x < 2147483648.0)) return INT_MIN;
    return (int)x;
}
static int ref_floor_int(double x) { return ref_to_int(floor(x)); }

/* ---------------------------------------------------------------------------------------
 * camera (camera.cpp)
 * ------------------------------------------------------------------------------------- */
static int validate_intr(const sf_intrinsics* i) { /* camera.cpp:9-14 */
    if (i->width <= 0 || i->height <= 0) return fail(SF_INVALID_ARGUMENT, "intrinsics: non-positive image size");
    if (i->fx <= 0.0 || i->fy <= 0.0) return fail(SF_INVALID_ARGUMENT, "intrinsics: non-positive focal length");
    if (!(i->near_plane > 0.0) || !(i->near_plane < i->far_plane))
        return fail(SF_INVALID_ARGUMENT, "intrinsics: need 0 < near < far");
    return SF_OK;
}
static v3 unproject(const sf_intrinsics* I, double u, double v, double d) { /* camera.cpp:31-33 */
    return V((u - I->cx) / I->fx * d, (v - I->cy) / I->fy * d, d);
}
static int project(const sf_intrinsics* I, v3 p, double* u, double* v) { /* camera.cpp:35-42 */
    if (!(p.z > 0.0)) return 0;
    *u = I->fx * p.x / p.z + I->cx;
    *v = I->fy * p.y / p.z + I->cy;
    return 1;
}
static int px_valid(const float* d, int w, int h, int u, int v) { /* camera.hpp:49-54 */
    return u >= 0 && v >= 0 && u < w && v < h && d[(size_t)v * w + u] > 0.0f;
}
static int nvalid(const float* n, size_t i) { /* camera.hpp:72, float squaredNorm */
    return (n[3 * i] * n[3 * i] + n[3 * i + 1] * n[3 * i + 1]) + n[3 * i + 2] * n[3 * i + 2] > 0.0f;
}

/* compute_normals (camera.cpp:44-76) */
static void normals_impl(const float* depth, const sf_intrinsics* I, double sigma0, double spatial, float* out) {
    const int w = I->width, h = I->height;
    memset(out, 0, sizeof(float) * 3 * (size_t)w * h);
    for (int v = 1; v + 1 < h; ++v)
        for (int u = 1; u + 1 < w; ++u) {
            const float z = px_valid(depth, w, h, u, v) ? depth[(size_t)v * w + u] : 0.0f;
            if (z <= 0.0f) continue;
            const float zl = depth[(size_t)v * w + u - 1], zr = depth[(size_t)v * w + u + 1];
            const float zu = depth[(size_t)(v - 1) * w + u], zd = depth[(size_t)(v + 1) * w + u];
            if (zl <= 0.0f || zr <= 0.0f || zu <= 0.0f || zd <= 0.0f) continue;
            const double thr = 3.0 * sigma0 * (double)z * (double)z + 2.0 * spatial;
            if (fabsf(zl - z) > thr || fabsf(zr - z) > thr || fabsf(zu - z) > thr || fabsf(zd - z) > thr) continue;
            const v3 du = vsub(unproject(I, u + 1, v, zr), unproject(I, u - 1, v, zl));
            const v3 dv = vsub(unproject(I, u, v + 1, zd), unproject(I, u, v - 1, zu));
            v3 n = vcross(du, dv);
            const double len = sqrt(vdot(n, n));
            if (!(len > 0.0)) continue;
            n = vdivs(n, len);
            if (vdot(n, unproject(I, u, v, z)) > 0.0) n = V(-n.x, -n.y, -n.z);
            float* o = out + 3 * ((size_t)v * w + u);
            o[0] = (float)n.x;
            o[1] = (float)n.y;
            o[2] = (float)n.z;
        }
}

int sfo_compute_normals(const sf_frame* f, double sigma0, double spatial, float* out, int32_t on_dev, void* s) {
    (void)on_dev;
    (void)s;
    int st = validate_intr(&f->intrinsics);
    if (st) return st;
    normals_impl(f->depth, &f->intrinsics, sigma0, spatial, out);
    return SF_OK;
}

/* ---------------------------------------------------------------------------------------
 * grid (grid.cpp)
 * ------------------------------------------------------------------------------------- */
typedef struct sfo_volume {
    sf_grid_config cfg;
    sf_aux_quant aux;
    int N, M, M3, res;
    double voxel, block_side, delta;
    uint64_t table_size, capacity, allocated, free_top;
    int32_t* table;
    uint16_t* payload;
    int32_t* free_list;
} vol_t;

/* quantize_tsdf / dequantize_tsdf (grid.cpp:20-27) */
static int8_t quantize_tsdf(double d, double delta) {
    const double c = dclamp(d, -delta, delta);
    return (int8_t)lround(c / delta * 127);
}
static double dequantize_tsdf(int8_t code, double delta) { return (double)code / 127 * delta; }
/* AuxQuantization::encode / decode (grid.cpp:38-51) */
static uint8_t aux_encode(const sf_aux_quant* a, double value) {
    if (a->mode == 0) {
        const double c = dclamp(value, 0.0, a->w_max);
        return (uint8_t)lround(c / a->w_max * 255.0);
    }
    const double c = dclamp(value, a->p_min, a->p_max);
    const double s = log(c / a->p_min) / log(a->p_max / a->p_min);
    return (uint8_t)lround(s * 255.0);
}
static double aux_decode(const sf_aux_quant* a, uint8_t code) {
    if (a->mode == 0) return (double)code / 255.0 * a->w_max;
    return a->p_min * exp((double)code / 255.0 * log(a->p_max / a->p_min));
}

static uint64_t tindex(const vol_t* g, int x, int y, int z) {
    return ((uint64_t)z * g->N + (uint64_t)y) * g->N + (uint64_t)x;
}
static int block_in_range(const vol_t* g, int x, int y, int z) {
    return x >= 0 && y >= 0 && z >= 0 && x < g->N && y < g->N && z < g->N;
}
static v3 voxel_center(const vol_t* g, int x, int y, int z) { /* grid.cpp:271-273 */
    return V(g->cfg.box_origin[0] + ((double)x + 0.5) * g->voxel, g->cfg.box_origin[1] + ((double)y + 0.5) * g->voxel,
             g->cfg.box_origin[2] + ((double)z + 0.5) * g->voxel);
}
static v3 block_min_corner(const vol_t* g, int x, int y, int z) { /* grid.cpp:275-277 */
    return V(g->cfg.box_origin[0] + (double)x * g->block_side, g->cfg.box_origin[1] + (double)y * g->block_side,
             g->cfg.box_origin[2] + (double)z * g->block_side);
}

/* SparseTsdfGrid ctor (grid.cpp:53-72) with GridConfig::validate (grid.cpp:12-18) */
int sfo_volume_create(const sf_grid_config* c, uint64_t cap, const sf_aux_quant* aux, int32_t dev, vol_t** out) {
    (void)dev;
    if (c->blocks_per_axis < 1 || c->voxels_per_block_axis < 1)
        return fail(SF_INVALID_ARGUMENT, "grid: N and M must be >= 1");
    if (!(c->box_side > 0.0)) return fail(SF_INVALID_ARGUMENT, "grid: box_side must be positive");
    const double voxel = c->box_side / (c->blocks_per_axis * c->voxels_per_block_axis);
    const double delta = c->truncation > 0.0 ? c->truncation : 4.0 * voxel;
    if (delta < 2.0 * voxel - 1e-12) return fail(SF_INVALID_ARGUMENT, "grid: truncation must be >= 2 * voxel_size");
    const uint64_t n = (uint64_t)c->blocks_per_axis, table = n * n * n;
    if (cap == 0) cap = table / 8 > 1 ? table / 8 : 1;
    if (cap > table) return fail(SF_INVALID_ARGUMENT, "grid: pool_capacity must be <= N^3");
    vol_t* g = calloc(1, sizeof *g);
    g->cfg = *c;
    sf_aux_quant def = {0, 20.0, 1e-8, 1e-2};
    g->aux = aux ? *aux : def;
    g->N = c->blocks_per_axis;
    g->M = c->voxels_per_block_axis;
    g->M3 = g->M * g->M * g->M;
    g->res = g->N * g->M;
    g->voxel = voxel;
    g->block_side = voxel * g->M;
    g->delta = delta;
    g->table_size = table;
    g->capacity = cap;
    g->table = malloc(table * sizeof(int32_t));
    for (uint64_t i = 0; i < table; ++i) g->table[i] = -1;
    g->payload = malloc(cap * g->M3 * sizeof(uint16_t));
    for (uint64_t i = 0; i < cap * g->M3; ++i) g->payload[i] = 0x0080;
    g->free_list = malloc(cap * sizeof(int32_t));
    for (uint64_t i = 0; i < cap; ++i) g->free_list[i] = (int32_t)(cap - 1 - i);
    g->free_top = cap;
    *out = g;
    return SF_OK;
}

int sfo_volume_destroy(vol_t* g) {
    if (!g) return SF_OK;
    free(g->table);
    free(g->payload);
    free(g->free_list);
    free(g);
    return SF_OK;
}

int sfo_volume_get_info(vol_t* g, sf_volume_info* o) {
    memset(o, 0, sizeof *o);
    o->config = g->cfg;
    o->aux = g->aux;
    o->delta = g->delta;
    o->voxel_size = g->voxel;
    o->pool_capacity = g->capacity;
    o->allocated_count = g->allocated;
    const uint64_t n = g->N, m = g->M;
    o->memory_bytes = 2ull * g->allocated * m * m * m + 4ull * n * n * n; /* grid.cpp:156-160 */
    return SF_OK;
}

/* allocate_block (grid.cpp:87-100) */
static int allocate_block(vol_t* g, int x, int y, int z, int32_t* slot_out) {
    const uint64_t ti = tindex(g, x, y, z);
    if (g->table[ti] != -1) {
        *slot_out = g->table[ti];
        return SF_OK;
    }
    if (g->free_top == 0)
        return fail(SF_POOL_EXHAUSTED,
                    "grid: payload pool exhausted (%llu blocks); increase pool capacity or lower resolution",
                    (unsigned long long)g->capacity);
    const int32_t slot = g->free_list[--g->free_top];
    g->table[ti] = slot;
    ++g->allocated;
    for (int i = 0; i < g->M3; ++i) g->payload[(size_t)slot * g->M3 + i] = 0x0080;
    *slot_out = slot;
    return SF_OK;
}

int sfo_volume_allocate_block(vol_t* g, const int32_t* bc, int32_t* slot) {
    if (!block_in_range(g, bc[0], bc[1], bc[2])) return fail(SF_OUT_OF_RANGE, "grid: block coordinate out of range");
    return allocate_block(g, bc[0], bc[1], bc[2], slot);
}

int sfo_volume_free_block(vol_t* g, const int32_t* bc) { /* grid.cpp:102-119 */
    if (!block_in_range(g, bc[0], bc[1], bc[2])) return fail(SF_OUT_OF_RANGE, "grid: block coordinate out of range");
    const uint64_t ti = tindex(g, bc[0], bc[1], bc[2]);
    const int32_t slot = g->table[ti];
    if (slot == -1) return SF_OK;
    g->table[ti] = -1;
    g->free_list[g->free_top++] = slot;
    --g->allocated;
    return SF_OK;
}

int sfo_volume_block_slot(vol_t* g, const int32_t* bc, int32_t* slot) { /* grid.cpp:82-85 */
    if (!block_in_range(g, bc[0], bc[1], bc[2])) return fail(SF_OUT_OF_RANGE, "grid: block coordinate out of range");
    *slot = g->table[tindex(g, bc[0], bc[1], bc[2])];
    return SF_OK;
}

static uint16_t* voxel_ptr(vol_t* g, const int32_t* vc, int32_t* slot_out) {
    const int M = g->M;
    const int bx = vc[0] / M, by = vc[1] / M, bz = vc[2] / M;
    const int32_t slot = g->table[tindex(g, bx, by, bz)];
    *slot_out = slot;
    if (slot == -1) return NULL;
    const int lx = vc[0] - bx * M, ly = vc[1] - by * M, lz = vc[2] - bz * M;
    return g->payload + (size_t)slot * g->M3 + ((size_t)lz * M + ly) * M + lx;
}

int sfo_volume_read_voxel(vol_t* g, const int32_t* vc, int32_t* is_chi, double* tsdf, double* aux) { /* grid.cpp:121-130 */
    for (int i = 0; i < 3; ++i)
        if (vc[i] < 0 || vc[i] >= g->res) return fail(SF_OUT_OF_RANGE, "grid: voxel coordinate out of range");
    int32_t slot;
    uint16_t* p = voxel_ptr(g, vc, &slot);
    *is_chi = 1;
    *tsdf = 0.0;
    *aux = 0.0;
    if (!p) return SF_OK;
    const int8_t code = (int8_t)(*p & 0xFF);
    if (code == -128) return SF_OK;
    *is_chi = 0;
    *tsdf = dequantize_tsdf(code, g->delta);
    *aux = aux_decode(&g->aux, (uint8_t)(*p >> 8));
    return SF_OK;
}

int sfo_volume_write_voxel(vol_t* g, const int32_t* vc, int32_t chi, double tsdf, double aux) { /* grid.cpp:132-154 */
    for (int i = 0; i < 3; ++i)
        if (vc[i] < 0 || vc[i] >= g->res) return fail(SF_OUT_OF_RANGE, "grid: voxel coordinate out of range");
    if (!chi && fabs(tsdf) > g->delta) chi = 1;
    int32_t slot;
    uint16_t* p = voxel_ptr(g, vc, &slot);
    if (!p) {
        if (chi) return SF_OK;
        return fail(SF_LOGIC_ERROR, "grid: write to unallocated block (allocate first)");
    }
    *p = chi ? 0x0080
             : (uint16_t)((uint8_t)quantize_tsdf(tsdf, g->delta) | ((uint16_t)aux_encode(&g->aux, aux) << 8));
    return SF_OK;
}

int sfo_volume_read_table(vol_t* g, int32_t* t) {
    memcpy(t, g->table, g->table_size * sizeof(int32_t));
    return SF_OK;
}
int sfo_volume_read_payload(vol_t* g, uint64_t first, uint64_t count, uint16_t* out) {
    if (first + count > g->capacity) return fail(SF_OUT_OF_RANGE, "payload range");
    memcpy(out, g->payload + first * g->M3, count * g->M3 * sizeof(uint16_t));
    return SF_OK;
}
int sfo_volume_write_payload(vol_t* g, uint64_t first, uint64_t count, const uint16_t* in) {
    if (first + count > g->capacity) return fail(SF_OUT_OF_RANGE, "payload range");
    memcpy(g->payload + first * g->M3, in, count * g->M3 * sizeof(uint16_t));
    return SF_OK;
}
int sfo_volume_save_snapshot(vol_t* g, const char* path) {
    (void)g;
    (void)path;
    return fail(SF_UNSUPPORTED, "oracle: snapshots are checked against the reference build");
}
int sfo_volume_load_snapshot(const char* path, uint64_t cap, int32_t dev, vol_t** out) {
    (void)path;
    (void)cap;
    (void)dev;
    (void)out;
    return fail(SF_UNSUPPORTED, "oracle: snapshots are checked against the reference build");
}

/* ---------------------------------------------------------------------------------------
 * fusion (fusion.cpp)
 * ------------------------------------------------------------------------------------- */
typedef struct {
    const sf_frame* frame;
    pose_t cfw; /* camera_from_world */
    float* normals;
    uint8_t* near_edge;
    int downweight;
} mctx_t;

/* MeasurementContext::make (fusion.cpp:25-72) */
static void mctx_make(mctx_t* c, const sf_frame* f, const pose_t* pose, const sf_fusion_params* p, double delta) {
    const sf_intrinsics* I = &f->intrinsics;
    const int w = I->width, h = I->height;
    const size_t n = (size_t)w * h;
    c->frame = f;
    c->cfw = invert(pose);
    c->downweight = p->edge_downweight;
    c->normals = NULL;
    c->near_edge = NULL;
    if (!c->downweight) return;
    c->normals = malloc(3 * n * sizeof(float));
    normals_impl(f->depth, I, p->sigma0, 0.25 * delta, c->normals);
    uint8_t* edge = calloc(n, 1);
    c->near_edge = calloc(n, 1);
    const float* d = f->depth;
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) {
            if (!px_valid(d, w, h, u, v)) {
                edge[(size_t)v * w + u] = 1;
                continue;
            }
            const float z = d[(size_t)v * w + u];
            const double jump = 3.0 * p->sigma0 * (double)z * (double)z + 0.02 * (double)z;
            int is_edge = u == 0 || v == 0 || u == w - 1 || v == h - 1;
            for (int k = 0; !is_edge && k < 4; ++k) {
                const int nu = u + (k == 0 ? 1 : k == 1 ? -1 : 0);
                const int nv = v + (k == 2 ? 1 : k == 3 ? -1 : 0);
                if (!px_valid(d, w, h, nu, nv) || fabsf(d[(size_t)nv * w + nu] - z) > jump) is_edge = 1;
            }
            if (is_edge) edge[(size_t)v * w + u] = 1;
        }
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) {
            int near = 0;
            for (int dv = -2; !near && dv <= 2; ++dv)
                for (int du = -2; !near && du <= 2; ++du) {
                    const int nu = u + du, nv = v + dv;
                    if (nu >= 0 && nv >= 0 && nu < w && nv < h && edge[(size_t)nv * w + nu]) near = 1;
                }
            if (near) c->near_edge[(size_t)v * w + u] = 1;
        }
    free(edge);
}

static void mctx_free(mctx_t* c) {
    free(c->normals);
    free(c->near_edge);
}

typedef struct {
    int valid;
    double tsdf, variance, weight;
} sample_t;

/* depth_interp of the refinement path (fusion.cpp:107-117) */
static double depth_interp(const sf_frame* f, double uu, double vv) {
    const int w = f->intrinsics.width, h = f->intrinsics.height;
    const int u0 = (int)floor(uu), v0 = (int)floor(vv);
    if (!(u0 >= 0 && v0 >= 0 && u0 < w && v0 < h) || !(u0 + 1 >= 0 && v0 + 1 >= 0 && u0 + 1 < w && v0 + 1 < h))
        return 0.0;
    const float d00 = f->depth[(size_t)v0 * w + u0], d10 = f->depth[(size_t)v0 * w + u0 + 1];
    const float d01 = f->depth[(size_t)(v0 + 1) * w + u0], d11 = f->depth[(size_t)(v0 + 1) * w + u0 + 1];
    if (d00 <= 0.0f || d10 <= 0.0f || d01 <= 0.0f || d11 <= 0.0f) return 0.0;
    const double fu = uu - u0, fv = vv - v0;
    return (d00 * (1.0 - fu) + d10 * fu) * (1.0 - fv) + (d01 * (1.0 - fu) + d11 * fu) * fv;
}
static double dist_sq(const sf_frame* f, double uu, double vv, v3 xc) {
    const double d = depth_interp(f, uu, vv);
    if (d <= 0.0) return INFINITY;
    const v3 r = vsub(unproject(&f->intrinsics, uu, vv, d), xc);
    return vdot(r, r);
}

/* estimate_measurement (fusion.cpp:81-173) */
static sample_t estimate(const mctx_t* c, v3 x, const sf_fusion_params* p, double delta) {
    sample_t out = {0, 0, 0, 0};
    const sf_frame* f = c->frame;
    const sf_intrinsics* I = &f->intrinsics;
    const int w = I->width, h = I->height;
    const v3 xc = papply(&c->cfw, x);
    double pu, pv;
    if (!project(I, xc, &pu, &pv)) return out;
    int u = ref_lround_int(pu), v = ref_lround_int(pv);
    if (!px_valid(f->depth, w, h, u, v)) return out;
    double measured = f->depth[(size_t)v * w + u];
    double tsdf_k = measured - xc.z;
    if (p->refinement_steps > 0) { /* fusion.cpp:99-143 */
        double cu = pu, cv = pv;
        double best = dist_sq(f, cu, cv, xc);
        if (isfinite(best)) {
            const double hh = 0.5;
            for (int step = 0; step < p->refinement_steps; ++step) {
                const double gu = dist_sq(f, cu + hh, cv, xc) - dist_sq(f, cu - hh, cv, xc);
                const double gv = dist_sq(f, cu, cv + hh, xc) - dist_sq(f, cu, cv - hh, xc);
                const double norm = hypot(gu, gv);
                if (!isfinite(norm) || norm == 0.0) break;
                const double nu = cu - hh * gu / norm;
                const double nv = cv - hh * gv / norm;
                const double cand = dist_sq(f, nu, nv, xc);
                if (!(cand < best)) break;
                best = cand;
                cu = nu;
                cv = nv;
            }
            const double d_here = depth_interp(f, cu, cv);
            if (d_here > 0.0) {
                u = ref_lround_int(cu);
                v = ref_lround_int(cv);
                measured = d_here;
                tsdf_k = (d_here >= xc.z ? 1.0 : -1.0) * sqrt(best);
            }
        }
    }
    if (fabs(tsdf_k) > delta) return out;
    const size_t pix = (size_t)v * w + u;
    const double sigma = (f->sigma && f->sigma[pix] > 0.0f) ? (double)f->sigma[pix] : p->sigma0 * measured * measured;
    out.valid = 1;
    out.tsdf = tsdf_k;
    out.variance = dmax(sigma * sigma, p->min_variance);
    out.weight = p->w_fixed;
    if (c->downweight) {
        double quality = 0.3;
        if (nvalid(c->normals, pix)) {
            const v3 ray = vnormalized(unproject(I, u, v, 1.0));
            const float* n = c->normals + 3 * pix;
            quality = fabs(vdot(V(n[0], n[1], n[2]), ray));
        }
        if (c->near_edge[pix]) quality *= 0.5;
        if (quality < 0.2) {
            out.valid = 0;
            return out;
        }
        out.weight *= quality;
        out.variance /= quality;
    }
    return out;
}

/* occupied_blocks_in_frustum's separating-axis test (grid.cpp:174-269) */
typedef struct {
    v3 pts[8];
    v3 axes[5];
    v3 edges[6];
} frustum_t;

static void frustum_make(frustum_t* fr, const pose_t* pose, const sf_intrinsics* I) {
    const double us[2] = {-0.5, I->width - 0.5}, vs[2] = {-0.5, I->height - 0.5};
    const double zs[2] = {I->near_plane, I->far_plane};
    int k = 0;
    for (int iz = 0; iz < 2; ++iz)
        for (int iv = 0; iv < 2; ++iv)
            for (int iu = 0; iu < 2; ++iu) fr->pts[k++] = papply(pose, unproject(I, us[iu], vs[iv], zs[iz]));
#define CORNER(u, v) vnormalized(mv(pose->R, unproject(I, u, v, 1.0)))
    const v3 r00 = CORNER(us[0], vs[0]), r10 = CORNER(us[1], vs[0]), r01 = CORNER(us[0], vs[1]),
             r11 = CORNER(us[1], vs[1]);
#undef CORNER
    fr->axes[0] = V(pose->R[2], pose->R[5], pose->R[8]);
    fr->axes[1] = vcross(r00, r10);
    fr->axes[2] = vcross(r11, r01);
    fr->axes[3] = vcross(r01, r00);
    fr->axes[4] = vcross(r10, r11);
    fr->edges[0] = r00;
    fr->edges[1] = r10;
    fr->edges[2] = r01;
    fr->edges[3] = r11;
    fr->edges[4] = V(pose->R[0], pose->R[3], pose->R[6]);
    fr->edges[5] = V(pose->R[1], pose->R[4], pose->R[7]);
}

static void hull_project(const v3* pts, v3 axis, double* lo, double* hi) {
    *lo = INFINITY;
    *hi = -INFINITY;
    for (int i = 0; i < 8; ++i) {
        const double d = vdot(axis, pts[i]);
        *lo = dmin(*lo, d);
        *hi = dmax(*hi, d);
    }
}

static int separated(const frustum_t* fr, const v3* box, v3 axis) {
    if (vdot(axis, axis) < 1e-18) return 0;
    double alo, ahi, blo, bhi;
    hull_project(fr->pts, axis, &alo, &ahi);
    hull_project(box, axis, &blo, &bhi);
    return ahi < blo || bhi < alo;
}

static int frustum_intersects(const frustum_t* fr, v3 lo, v3 hi) {
    v3 box[8];
    for (int i = 0; i < 8; ++i) box[i] = V(i & 1 ? hi.x : lo.x, i & 2 ? hi.y : lo.y, i & 4 ? hi.z : lo.z);
    const v3 ba[3] = {V(1, 0, 0), V(0, 1, 0), V(0, 0, 1)};
    for (int i = 0; i < 3; ++i)
        if (separated(fr, box, ba[i])) return 0;
    for (int i = 0; i < 5; ++i)
        if (separated(fr, box, fr->axes[i])) return 0;
    for (int e = 0; e < 6; ++e)
        for (int i = 0; i < 3; ++i)
            if (separated(fr, box, vcross(fr->edges[e], ba[i]))) return 0;
    return 1;
}

static int cmp_u64(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

typedef struct {
    uint64_t* alloc;
    size_t n_alloc;
    uint64_t* update;
    size_t n_update;
} lists_t;

static int sorted_contains(const uint64_t* a, size_t n, uint64_t k) {
    size_t lo = 0, hi = n;
    while (lo < hi) {
        const size_t mid = (lo + hi) / 2;
        if (a[mid] < k) lo = mid + 1;
        else hi = mid;
    }
    return lo < n && a[lo] == k;
}

/* select_update_blocks (fusion.cpp:187-235); a (z,y,x)-ordered std::set == sorted unique
 * table indices. */
static void select_lists(vol_t* g, const sf_frame* f, const pose_t* pose, lists_t* L) {
    const sf_intrinsics* I = &f->intrinsics;
    const int w = I->width, h = I->height;
    const double delta = g->delta;
    const int stride = (g->M + 1) / 2 > 1 ? (g->M + 1) / 2 : 1;
    size_t cap = 3 * (size_t)((w + stride - 1) / stride) * ((h + stride - 1) / stride) + 1, n = 0;
    uint64_t* keys = malloc(cap * sizeof(uint64_t));
    for (int v = 0; v < h; v += stride)
        for (int u = 0; u < w; u += stride) {
            if (!px_valid(f->depth, w, h, u, v)) continue;
            const v3 dir_cam = vnormalized(unproject(I, u, v, 1.0));
            const v3 dir = mv(pose->R, dir_cam);
            const double t_hit = f->depth[(size_t)v * w + u] / dir_cam.z;
            const double offs[3] = {-delta, 0.0, delta};
            for (int k = 0; k < 3; ++k) {
                const v3 x = vadd(pose->t, vscale(t_hit + offs[k], dir));
                const int bx = ref_floor_int((x.x - g->cfg.box_origin[0]) / g->block_side);
                const int by = ref_floor_int((x.y - g->cfg.box_origin[1]) / g->block_side);
                const int bz = ref_floor_int((x.z - g->cfg.box_origin[2]) / g->block_side);
                if (block_in_range(g, bx, by, bz)) keys[n++] = tindex(g, bx, by, bz);
            }
        }
    qsort(keys, n, sizeof(uint64_t), cmp_u64);
    size_t m = 0;
    for (size_t i = 0; i < n; ++i)
        if (m == 0 || keys[m - 1] != keys[i]) keys[m++] = keys[i];
    L->alloc = keys;
    L->n_alloc = m;
    /* visible allocated blocks (grid.cpp:228-269, fusion.cpp:211-233), table order */
    frustum_t fr;
    frustum_make(&fr, pose, I);
    const pose_t inv = invert(pose);
    const double side = g->block_side;
    L->update = malloc((g->allocated + 1) * sizeof(uint64_t));
    L->n_update = 0;
    for (uint64_t ti = 0; ti < g->table_size; ++ti) {
        if (g->table[ti] == -1) continue;
        const int bx = (int)(ti % g->N), by = (int)((ti / g->N) % g->N), bz = (int)(ti / ((uint64_t)g->N * g->N));
        const v3 lo = block_min_corner(g, bx, by, bz);
        const v3 hi = vadd(lo, V(side, side, side));
        if (!frustum_intersects(&fr, lo, hi)) continue;
        if (sorted_contains(L->alloc, L->n_alloc, ti)) continue;
        int visible = 0;
        for (int i = 0; i < 9 && !visible; ++i) {
            const v3 probe = i == 8 ? vadd(lo, V(0.5 * side, 0.5 * side, 0.5 * side))
                                    : vadd(lo, V(i & 1 ? side : 0.0, i & 2 ? side : 0.0, i & 4 ? side : 0.0));
            const v3 xc = papply(&inv, probe);
            double pu, pv;
            if (!project(I, xc, &pu, &pv)) continue;
            const int u = ref_lround_int(pu), v = ref_lround_int(pv);
            if (!(u >= 0 && v >= 0 && u < w && v < h)) continue;
            const float d = f->depth[(size_t)v * w + u];
            if (!(d > 0.0f) || xc.z <= d + delta) visible = 1;
        }
        if (visible) L->update[L->n_update++] = ti;
    }
}

int sfo_select_update_blocks(vol_t* g, const sf_frame* f, const double* pose12, int32_t* axyz, uint64_t* na,
                             int32_t* uxyz, uint64_t* nu, void* s) {
    (void)s;
    int st = validate_intr(&f->intrinsics);
    if (st) return st;
    const pose_t pose = pose_from(pose12);
    lists_t L;
    select_lists(g, f, &pose, &L);
    if (L.n_alloc > *na || L.n_update > *nu) {
        free(L.alloc);
        free(L.update);
        return fail(SF_OUT_OF_RANGE, "select_update_blocks: output capacity");
    }
    for (size_t i = 0; i < L.n_alloc; ++i) {
        axyz[3 * i] = (int32_t)(L.alloc[i] % g->N);
        axyz[3 * i + 1] = (int32_t)((L.alloc[i] / g->N) % g->N);
        axyz[3 * i + 2] = (int32_t)(L.alloc[i] / ((uint64_t)g->N * g->N));
    }
    for (size_t i = 0; i < L.n_update; ++i) {
        uxyz[3 * i] = (int32_t)(L.update[i] % g->N);
        uxyz[3 * i + 1] = (int32_t)((L.update[i] / g->N) % g->N);
        uxyz[3 * i + 2] = (int32_t)(L.update[i] / ((uint64_t)g->N * g->N));
    }
    *na = L.n_alloc;
    *nu = L.n_update;
    free(L.alloc);
    free(L.update);
    return SF_OK;
}

/* fuse_frame (fusion.cpp:274-376) */
int sfo_integrate(vol_t* g, const sf_frame* f, const double* pose12, const sf_fusion_params* pin,
                  sf_fusion_stats* stats, void* s) {
    (void)s;
    /* FusionParams::validate (fusion.cpp:12-17), mode/aux checks (fusion.cpp:279-283) */
    if (!(pin->w_fixed > 0.0) || pin->w_fixed > 1.0) return fail(SF_INVALID_ARGUMENT, "fusion: w_fixed must be in (0, 1]");
    if (!(pin->w_max > 0.0)) return fail(SF_INVALID_ARGUMENT, "fusion: w_max must be positive");
    if (pin->sigma0 < 0.0) return fail(SF_INVALID_ARGUMENT, "fusion: sigma0 must be >= 0");
    if (pin->refinement_steps < 0) return fail(SF_INVALID_ARGUMENT, "fusion: negative refinement_steps");
    if (pin->mode == 2 && g->aux.mode != 1)
        return fail(SF_INVALID_ARGUMENT, "fusion: Kalman mode needs a variance-mode grid");
    if (pin->mode != 2 && g->aux.mode != 0)
        return fail(SF_INVALID_ARGUMENT, "fusion: weight-mode grid required for this fusion mode");
    int st = validate_intr(&f->intrinsics);
    if (st) return st;
    sf_fusion_params p = *pin;
    p.delta = g->delta;
    const double delta = g->delta;
    const pose_t pose = pose_from(pose12);
    lists_t L;
    select_lists(g, f, &pose, &L);
    const uint64_t before = g->allocated;
    mctx_t ctx;
    mctx_make(&ctx, f, &pose, &p, delta);
    double q; /* resolved_q (fusion.cpp:19-23) */
    if (p.process_variance >= 0.0) q = p.process_variance;
    else {
        const double step = 0.1 * delta / 127;
        q = step * step;
    }
    const int M = g->M;
    uint64_t updated = 0;
    int status = SF_OK;
    for (int pass = 0; pass < 2 && status == SF_OK; ++pass) {
        const uint64_t* list = pass == 0 ? L.alloc : L.update;
        const size_t cnt = pass == 0 ? L.n_alloc : L.n_update;
        for (size_t b = 0; b < cnt; ++b) {
            const uint64_t ti = list[b];
            const int bx = (int)(ti % g->N), by = (int)((ti / g->N) % g->N), bz = (int)(ti / ((uint64_t)g->N * g->N));
            int32_t slot = g->table[ti];
            if (slot == -1) {
                if (pass == 1) continue;
                status = allocate_block(g, bx, by, bz, &slot);
                if (status != SF_OK) break;
            }
            uint16_t* pl = g->payload + (size_t)slot * g->M3;
            for (int z = 0; z < M; ++z)
                for (int y = 0; y < M; ++y)
                    for (int x = 0; x < M; ++x) {
                        const sample_t smp = estimate(&ctx, voxel_center(g, bx * M + x, by * M + y, bz * M + z), &p, delta);
                        if (!smp.valid) continue;
                        uint16_t* cell = pl + ((size_t)z * M + y) * M + x;
                        const int8_t code = (int8_t)(*cell & 0xFF);
                        const int has = code != -128;
                        const double pt = has ? dequantize_tsdf(code, delta) : 0.0;
                        const double pa = has ? aux_decode(&g->aux, (uint8_t)(*cell >> 8)) : 0.0;
                        double nt, na;
                        if (p.mode == 0) { /* fuse_simple (fusion.cpp:237-242) */
                            nt = has ? (1.0 - smp.weight) * pt + smp.weight * smp.tsdf : smp.tsdf;
                            na = smp.weight;
                        } else if (p.mode == 1) { /* fuse_weighted (fusion.cpp:244-256) */
                            if (!has) {
                                nt = smp.tsdf;
                                na = smp.weight;
                            } else {
                                nt = (pa * pt + smp.weight * smp.tsdf) / (pa + smp.weight);
                                na = dmin(pa + smp.weight, p.w_max);
                            }
                        } else { /* fuse_kalman (fusion.cpp:258-272) */
                            if (!has) {
                                nt = smp.tsdf;
                                na = smp.variance;
                            } else {
                                const double predicted = pa + q;
                                const double gain = predicted / (predicted + smp.variance);
                                nt = pt + gain * (smp.tsdf - pt);
                                na = (1.0 - gain) * predicted;
                            }
                        }
                        if (fabs(nt) > delta) *cell = 0x0080;
                        else *cell = (uint16_t)((uint8_t)quantize_tsdf(nt, delta) | ((uint16_t)aux_encode(&g->aux, na) << 8));
                        ++updated;
                    }
        }
    }
    mctx_free(&ctx);
    free(L.alloc);
    free(L.update);
    if (stats) {
        const uint64_t n = g->N, m = g->M;
        stats->voxels_updated = updated;
        stats->blocks_allocated_now = g->allocated - before;
        stats->blocks_total = g->allocated;
        stats->memory_bytes = 2ull * g->allocated * m * m * m + 4ull * n * n * n;
    }
    return status;
}

/* ---------------------------------------------------------------------------------------
 * raycast (render.cpp)
 * ------------------------------------------------------------------------------------- */
static int voxel_code(const vol_t* g, int x, int y, int z, double* out) { /* render.cpp:12-21 */
    const int M = g->M;
    const int bx = x / M, by = y / M, bz = z / M;
    const int32_t slot = g->table[tindex(g, bx, by, bz)];
    if (slot == -1) return 0;
    const uint16_t pl = g->payload[(size_t)slot * g->M3 + ((size_t)(z - bz * M) * M + (y - by * M)) * M + (x - bx * M)];
    const int8_t c = (int8_t)(pl & 0xFF);
    if (c == -128) return 0;
    *out = dequantize_tsdf(c, g->delta);
    return 1;
}

static int sample_tsdf(const vol_t* g, v3 p, double* out) { /* render.cpp:25-48 */
    const double gx = (p.x - g->cfg.box_origin[0]) / g->voxel - 0.5;
    const double gy = (p.y - g->cfg.box_origin[1]) / g->voxel - 0.5;
    const double gz = (p.z - g->cfg.box_origin[2]) / g->voxel - 0.5;
    const int bx = ref_floor_int(gx), by = ref_floor_int(gy), bz = ref_floor_int(gz);
    if (bx < 0 || by < 0 || bz < 0 || bx + 1 >= g->res || by + 1 >= g->res || bz + 1 >= g->res) return 0;
    const double fx = gx - bx, fy = gy - by, fz = gz - bz;
    double c[8];
    for (int i = 0; i < 8; ++i)
        if (!voxel_code(g, bx + (i & 1), by + ((i >> 1) & 1), bz + ((i >> 2) & 1), &c[i])) return 0;
    const double x0 = c[0] + (c[1] - c[0]) * fx, x1 = c[2] + (c[3] - c[2]) * fx;
    const double x2 = c[4] + (c[5] - c[4]) * fx, x3 = c[6] + (c[7] - c[6]) * fx;
    const double y0 = x0 + (x1 - x0) * fy, y1 = x2 + (x3 - x2) * fy;
    *out = y0 + (y1 - y0) * fz;
    return 1;
}

static int sample_gradient(const vol_t* g, v3 p, double h, v3* out) { /* render.cpp:50-63 */
    double gv[3];
    for (int i = 0; i < 3; ++i) {
        v3 dp = p, dm = p;
        double* a = i == 0 ? &dp.x : i == 1 ? &dp.y : &dp.z;
        double* b = i == 0 ? &dm.x : i == 1 ? &dm.y : &dm.z;
        *a += h;
        *b -= h;
        double va, vb;
        if (!sample_tsdf(g, dp, &va) || !sample_tsdf(g, dm, &vb)) return 0;
        gv[i] = (va - vb) / (2.0 * h);
    }
    *out = V(gv[0], gv[1], gv[2]);
    return 1;
}

/* compute_ray_bounds (render.cpp:65-153) */
static void bounds_impl(const vol_t* g, const pose_t* pose, const sf_intrinsics* I, float* ts, float* te) {
    const int w = I->width, h = I->height;
    for (size_t i = 0; i < (size_t)w * h; ++i) {
        ts[i] = INFINITY;
        te[i] = -INFINITY;
    }
    if (g->allocated == 0) return;
    const int n = g->N;
    const double side = g->block_side;
    const double blo[3] = {g->cfg.box_origin[0], g->cfg.box_origin[1], g->cfg.box_origin[2]};
    const double bhi[3] = {blo[0] + g->cfg.box_side, blo[1] + g->cfg.box_side, blo[2] + g->cfg.box_side};
    const double org[3] = {pose->t.x, pose->t.y, pose->t.z};
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) {
            const v3 dc = vnormalized(unproject(I, u, v, 1.0));
            const v3 d3 = mv(pose->R, dc);
            const double dir[3] = {d3.x, d3.y, d3.z};
            double lo = I->near_plane / dc.z, hi = I->far_plane / dc.z;
            for (int a = 0; a < 3; ++a) {
                if (fabs(dir[a]) < 1e-15) {
                    if (org[a] < blo[a] || org[a] > bhi[a]) {
                        lo = 1.0;
                        hi = 0.0;
                        break;
                    }
                    continue;
                }
                double t0 = (blo[a] - org[a]) / dir[a], t1 = (bhi[a] - org[a]) / dir[a];
                if (t0 > t1) {
                    const double tmp = t0;
                    t0 = t1;
                    t1 = tmp;
                }
                lo = dmax(lo, t0);
                hi = dmin(hi, t1);
            }
            if (!(lo <= hi)) continue;
            const double entry[3] = {org[0] + lo * dir[0], org[1] + lo * dir[1], org[2] + lo * dir[2]};
            int cell[3], step[3];
            double tmax[3], tdelta[3];
            for (int a = 0; a < 3; ++a) {
                int c = ref_floor_int((entry[a] - blo[a]) / side);
                cell[a] = c < 0 ? 0 : (n - 1 < c ? n - 1 : c);
            }
            for (int a = 0; a < 3; ++a) {
                if (dir[a] > 1e-15) {
                    step[a] = 1;
                    tmax[a] = lo + (blo[a] + (cell[a] + 1) * side - entry[a]) / dir[a];
                    tdelta[a] = side / dir[a];
                } else if (dir[a] < -1e-15) {
                    step[a] = -1;
                    tmax[a] = lo + (blo[a] + cell[a] * side - entry[a]) / dir[a];
                    tdelta[a] = -side / dir[a];
                } else {
                    step[a] = 0;
                    tmax[a] = INFINITY;
                    tdelta[a] = INFINITY;
                }
            }
            double first = INFINITY, last = -INFINITY, t_in = lo;
            while (t_in <= hi) {
                const int axis = tmax[0] <= tmax[1] ? (tmax[0] <= tmax[2] ? 0 : 2) : (tmax[1] <= tmax[2] ? 1 : 2);
                const double t_out = dmin(tmax[axis], hi);
                if (g->table[tindex(g, cell[0], cell[1], cell[2])] != -1) {
                    first = dmin(first, t_in);
                    last = dmax(last, t_out);
                }
                t_in = tmax[axis];
                cell[axis] += step[axis];
                if (cell[axis] < 0 || cell[axis] >= n) break;
                tmax[axis] += tdelta[axis];
            }
            if (first <= last) {
                ts[(size_t)v * w + u] = (float)dmax(first, lo);
                te[(size_t)v * w + u] = (float)dmin(last, hi);
            }
        }
}

int sfo_ray_bounds(vol_t* g, const double* pose12, const sf_intrinsics* I, float* ts, float* te, int32_t od, void* s) {
    (void)od;
    (void)s;
    int st = validate_intr(I);
    if (st) return st;
    const pose_t pose = pose_from(pose12);
    bounds_impl(g, &pose, I, ts, te);
    return SF_OK;
}

/* raycast (render.cpp:155-250) */
int sfo_raycast(vol_t* g, const double* pose12, const sf_intrinsics* I, float* depth, float* normals, int32_t od,
                sf_raycast_stats* stats, void* s) {
    (void)od;
    (void)s;
    int st = validate_intr(I);
    if (st) return st;
    const pose_t pose = pose_from(pose12);
    const int w = I->width, h = I->height;
    const size_t n = (size_t)w * h;
    float* ts = malloc(n * sizeof(float));
    float* te = malloc(n * sizeof(float));
    bounds_impl(g, &pose, I, ts, te);
    memset(depth, 0, n * sizeof(float));
    memset(normals, 0, 3 * n * sizeof(float));
    sf_raycast_stats rs = {0, 0, 0};
    const double vox = g->voxel, coarse = 0.5 * g->delta, fine_tol = 0.01 * vox;
    double w2c[9];
    mtrans(pose.R, w2c);
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) {
            const size_t idx = (size_t)v * w + u;
            if (!(ts[idx] <= te[idx])) continue;
            ++rs.rays_with_bounds;
            const v3 dc = vnormalized(unproject(I, u, v, 1.0));
            const v3 dir = mv(pose.R, dc);
            const double t0 = ts[idx], t1 = te[idx];
            double prev_t = 0.0, prev_val = 0.0, ha = 0.0, hb = 0.0, va = 0.0, vb = 0.0;
            int have_prev = 0, bracketed = 0;
            for (double t = t0;; t += coarse) {
                const int final_sample = t >= t1;
                if (final_sample) t = t1;
                ++rs.sample_steps;
                double val;
                if (sample_tsdf(g, vadd(pose.t, vscale(t, dir)), &val)) {
                    if (have_prev && prev_val > 0.0 && val < 0.0) {
                        ha = prev_t;
                        va = prev_val;
                        hb = t;
                        vb = val;
                        bracketed = 1;
                        break;
                    }
                    have_prev = 1;
                    prev_t = t;
                    prev_val = val;
                }
                if (final_sample) break;
            }
            if (!bracketed) continue;
            double root = hb;
            for (int iter = 0; iter < 48 && hb - ha > fine_tol; ++iter) {
                double tn = hb - vb * (hb - ha) / (vb - va);
                if (!(tn > ha) || !(tn < hb)) tn = 0.5 * (ha + hb);
                double val;
                if (!sample_tsdf(g, vadd(pose.t, vscale(tn, dir)), &val)) {
                    ha = tn;
                    va = dmax(va, 1e-12);
                    continue;
                }
                if (val > 0.0) {
                    ha = tn;
                    va = val;
                } else {
                    hb = tn;
                    vb = val;
                }
            }
            if (vb != va) root = dclamp(hb - vb * (hb - ha) / (vb - va), ha, hb);
            else root = 0.5 * (ha + hb);
            const double d = root * dc.z;
            if (d < I->near_plane || d > I->far_plane) continue;
            depth[idx] = (float)d;
            ++rs.hit_pixels;
            v3 gr;
            if (sample_gradient(g, vadd(pose.t, vscale(root, dir)), vox, &gr) && vdot(gr, gr) > 0.0) {
                const v3 nc = mv(w2c, vnormalized(gr));
                normals[3 * idx] = (float)nc.x;
                normals[3 * idx + 1] = (float)nc.y;
                normals[3 * idx + 2] = (float)nc.z;
            }
        }
    free(ts);
    free(te);
    if (stats) *stats = rs;
    return SF_OK;
}

/* ---------------------------------------------------------------------------------------
 * registration (registration.cpp) and pose.cpp
 * ------------------------------------------------------------------------------------- */
/* Eigen JacobiSVD<Matrix3d> as restated in oracle/shim/Eigen/Dense */
typedef struct {
    double c, s;
} rot2;
static rot2 rmul(rot2 a, rot2 b) {
    rot2 r = {a.c * b.c - a.s * b.s, a.c * b.s + a.s * b.c};
    return r;
}
static rot2 rtr(rot2 a) {
    rot2 r = {a.c, -a.s};
    return r;
}
static void make_jacobi(double x, double y, double z, rot2* j) {
    const double deno = 2.0 * fabs(y);
    if (deno < DBL_MIN) {
        j->c = 1.0;
        j->s = 0.0;
        return;
    }
    const double tau = (x - z) / deno;
    const double w = sqrt(tau * tau + 1.0);
    const double t = tau > 0.0 ? 1.0 / (tau + w) : 1.0 / (tau - w);
    const double sign_t = t > 0.0 ? 1.0 : -1.0;
    const double n = 1.0 / sqrt(t * t + 1.0);
    j->s = -sign_t * (y / fabs(y)) * fabs(t) * n;
    j->c = n;
}
static void jsvd_2x2(double m[3][3], int p, int q, rot2* jl, rot2* jr) {
    double m00 = m[p][p], m01 = m[p][q], m10 = m[q][p], m11 = m[q][q];
    rot2 r1;
    const double t = m00 + m11, d = m10 - m01;
    if (fabs(d) < DBL_MIN) {
        r1.s = 0.0;
        r1.c = 1.0;
    } else {
        const double u = t / d, tmp = sqrt(1.0 + u * u);
        r1.s = 1.0 / tmp;
        r1.c = u / tmp;
    }
    const double a0 = m00, a1 = m01, b0 = m10, b1 = m11;
    m00 = r1.c * a0 + r1.s * b0;
    m01 = r1.c * a1 + r1.s * b1;
    m11 = -r1.s * a1 + r1.c * b1;
    (void)b0;
    make_jacobi(m00, m01, m11, jr);
    *jl = rmul(r1, rtr(*jr));
}
static void apply_left(double m[3][3], int p, int q, rot2 j) {
    for (int k = 0; k < 3; ++k) {
        const double x = m[p][k], y = m[q][k];
        m[p][k] = j.c * x + j.s * y;
        m[q][k] = -j.s * x + j.c * y;
    }
}
static void apply_right(double m[3][3], int p, int q, rot2 j) {
    for (int k = 0; k < 3; ++k) {
        const double x = m[k][p], y = m[k][q];
        m[k][p] = j.c * x - j.s * y;
        m[k][q] = j.s * x + j.c * y;
    }
}
/* nearest_rotation (pose.cpp:20-29) */
static void nearest_rotation(const double* A, double* R) {
    double scale = fabs(A[0]);
    for (int c = 0; c < 3; ++c)
        for (int r = 0; r < 3; ++r) {
            const double x = fabs(A[r * 3 + c]);
            scale = scale < x ? x : scale;
        }
    if (scale == 0.0) scale = 1.0;
    double wk[3][3], u[3][3], v[3][3];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            wk[r][c] = A[r * 3 + c] / scale;
            u[r][c] = v[r][c] = r == c ? 1.0 : 0.0;
        }
    const double precision = 2.0 * DBL_EPSILON;
    double maxd = dmax(dmax(fabs(wk[0][0]), fabs(wk[1][1])), fabs(wk[2][2]));
    int finished = 0, sweeps = 0;
    while (!finished && sweeps < 64) {
        finished = 1;
        ++sweeps;
        for (int p = 1; p < 3; ++p)
            for (int q = 0; q < p; ++q) {
                const double thr = dmax(DBL_MIN, precision * maxd);
                if (fabs(wk[p][q]) > thr || fabs(wk[q][p]) > thr) {
                    finished = 0;
                    rot2 jl, jr;
                    jsvd_2x2(wk, p, q, &jl, &jr);
                    apply_left(wk, p, q, jl);
                    apply_right(u, p, q, rtr(jl));
                    apply_right(wk, p, q, jr);
                    apply_right(v, p, q, jr);
                    maxd = dmax(maxd, dmax(fabs(wk[p][p]), fabs(wk[q][q])));
                }
            }
    }
    double sv[3];
    for (int i = 0; i < 3; ++i) {
        sv[i] = fabs(wk[i][i]);
        if (wk[i][i] < 0.0)
            for (int k = 0; k < 3; ++k) u[k][i] = -u[k][i];
    }
    for (int i = 0; i < 3; ++i) {
        int pos = i;
        for (int k = i + 1; k < 3; ++k)
            if (sv[k] > sv[pos]) pos = k;
        if (pos != i) {
            double t = sv[i];
            sv[i] = sv[pos];
            sv[pos] = t;
            for (int k = 0; k < 3; ++k) {
                t = u[k][i];
                u[k][i] = u[k][pos];
                u[k][pos] = t;
                t = v[k][i];
                v[k][i] = v[k][pos];
                v[k][pos] = t;
            }
        }
    }
    double U[9], Vt[9];
    for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c) {
            U[r * 3 + c] = u[r][c];
            Vt[c * 3 + r] = v[r][c];
        }
    mm(U, Vt, R);
    const double det = R[0] * (R[4] * R[8] - R[7] * R[5]) - R[3] * (R[1] * R[8] - R[7] * R[2]) +
                       R[6] * (R[1] * R[5] - R[4] * R[2]);
    if (det < 0.0) {
        const double flip[9] = {1, 0, 0, 0, 1, 0, 0, 0, -1};
        double tmp[9];
        mm(U, flip, tmp);
        mm(tmp, Vt, R);
    }
}
/* apply_motion (pose.cpp:31-43) */
static pose_t apply_motion(const pose_t* pose, v3 r, v3 t) {
    const double lin[9] = {1.0, -r.z, r.y, r.z, 1.0, -r.x, -r.y, r.x, 1.0};
    pose_t corr;
    nearest_rotation(lin, corr.R);
    corr.t = t;
    return compose(&corr, pose);
}

/* eigendecompose_sym6 (registration.cpp:125-165): dense rot^T m rot products, naive order */
static void mat6_mul(const double* A, const double* B, double* out) { /* (i,j) = sum_k A(i,k) B(k,j), k ascending */
    double r[36];
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
            double s = A[i * 6] * B[j];
            for (int k = 1; k < 6; ++k) s = s + A[i * 6 + k] * B[k * 6 + j];
            r[i * 6 + j] = s;
        }
    memcpy(out, r, sizeof r);
}
static void eigen6(const double* a, double* values, double* vectors /* col-major [c*6+r] */) {
    double m[36], v[36];
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
            m[i * 6 + j] = 0.5 * (a[i * 6 + j] + a[j * 6 + i]);
            v[i * 6 + j] = i == j ? 1.0 : 0.0;
        }
    double sq = m[0] * m[0];
    for (int c = 0; c < 6; ++c)
        for (int r = 0; r < 6; ++r)
            if (c || r) sq = sq + m[r * 6 + c] * m[r * 6 + c];
    const double scl = dmax(1.0, sqrt(sq)), tol = 1e-12 * scl;
    for (int sweep = 0; sweep < 64; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < 6; ++p)
            for (int q = p + 1; q < 6; ++q) off += m[p * 6 + q] * m[p * 6 + q];
        if (sqrt(off) <= tol) break;
        for (int p = 0; p < 6; ++p)
            for (int q = p + 1; q < 6; ++q) {
                const double apq = m[p * 6 + q];
                if (fabs(apq) <= tol / 30.0) continue;
                const double theta = (m[q * 6 + q] - m[p * 6 + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
                double rot[36], rt[36];
                for (int i = 0; i < 36; ++i) rot[i] = (i % 7 == 0) ? 1.0 : 0.0;
                rot[p * 6 + p] = c;
                rot[q * 6 + q] = c;
                rot[p * 6 + q] = s;
                rot[q * 6 + p] = -s;
                for (int i = 0; i < 6; ++i)
                    for (int j = 0; j < 6; ++j) rt[j * 6 + i] = rot[i * 6 + j];
                mat6_mul(rt, m, m);
                mat6_mul(m, rot, m);
                mat6_mul(v, rot, v);
            }
    }
    int order[6] = {0, 1, 2, 3, 4, 5};
    for (int i = 1; i < 6; ++i) { /* stable insertion sort == libstdc++ std::sort for n <= 16 */
        const int val = order[i];
        int j = i;
        while (j > 0 && m[val * 6 + val] < m[order[j - 1] * 6 + order[j - 1]]) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = val;
    }
    for (int i = 0; i < 6; ++i) {
        values[i] = m[order[i] * 6 + order[i]];
        for (int r = 0; r < 6; ++r) vectors[i * 6 + r] = v[r * 6 + order[i]];
    }
}

typedef struct {
    v3 p, q, n;
} match_t;

/* Kahan-compensated accumulator (registration.cpp:79-89) */
typedef struct {
    double sum, carry;
} kahan_t;
static void kadd(kahan_t* k, double value) {
    const double y = value - k->carry;
    const double t = k->sum + y;
    k->carry = (t - k->sum) - y;
    k->sum = t;
}

int sfo_icp(const sf_frame* src, const float* src_n_in, const sf_frame* tgt, const float* tgt_n,
            const double* initial, const sf_match_params* mp, sf_icp_result* res, void* s) {
    (void)s;
    const sf_intrinsics* si = &src->intrinsics;
    const sf_intrinsics* ti = &tgt->intrinsics;
    if (si->width != ti->width || si->height != ti->height)
        return fail(SF_INVALID_ARGUMENT, "match: frames must share intrinsics");
    const int w = si->width, h = si->height;
    const size_t npx = (size_t)w * h;
    float* sn_owned = NULL;
    const float* sn = src_n_in;
    if (!sn) { /* registration.cpp:216-220 */
        sn_owned = malloc(3 * npx * sizeof(float));
        normals_impl(src->depth, si, mp->normal_sigma0, mp->normal_spatial_scale, sn_owned);
        sn = sn_owned;
    }
    const double cos_max = cos(mp->max_normal_angle), max_dist_sq = mp->max_distance * mp->max_distance;
    memset(res, 0, sizeof *res);
    pose_t delta = pose_from(initial);
    match_t* mt = malloc(npx * sizeof(match_t));
    int status = SF_OK;
    for (int iter = 0; iter < mp->max_iterations; ++iter) {
        /* match_points (registration.cpp:17-50) */
        size_t nm = 0;
        for (int v = 0; v < h; ++v)
            for (int u = 0; u < w; ++u) {
                const size_t i = (size_t)v * w + u;
                if (!px_valid(src->depth, w, h, u, v) || !nvalid(sn, i)) continue;
                const v3 p = papply(&delta, unproject(si, u, v, src->depth[i]));
                double pu, pv;
                if (!project(ti, p, &pu, &pv)) continue;
                const int tu = ref_lround_int(pu), tv = ref_lround_int(pv);
                if (!(tu >= 0 && tv >= 0 && tu < w && tv < h)) continue;
                const size_t j = (size_t)tv * w + tu;
                if (!(tgt->depth[j] > 0.0f) || !nvalid(tgt_n, j)) continue;
                const v3 q = unproject(ti, tu, tv, tgt->depth[j]);
                const v3 dq = vsub(p, q);
                if (vdot(dq, dq) > max_dist_sq) continue;
                const v3 n = V(tgt_n[3 * j], tgt_n[3 * j + 1], tgt_n[3 * j + 2]);
                const v3 ns = mv(delta.R, V(sn[3 * i], sn[3 * i + 1], sn[3 * i + 2]));
                if (vdot(ns, n) < cos_max) continue;
                mt[nm].p = p;
                mt[nm].q = q;
                mt[nm].n = n;
                ++nm;
            }
        if (nm < 10) {
            status = fail(SF_TRACKING_LOST, "icp: only %zu correspondences", nm);
            break;
        }
        res->matches = nm;
        /* shrink (registration.cpp:52-74) */
        v3 lo = mt[0].p, hi = mt[0].p;
        for (size_t k = 0; k < nm; ++k) {
            lo = V(dmin(dmin(lo.x, mt[k].p.x), mt[k].q.x), dmin(dmin(lo.y, mt[k].p.y), mt[k].q.y),
                   dmin(dmin(lo.z, mt[k].p.z), mt[k].q.z));
            hi = V(dmax(dmax(hi.x, mt[k].p.x), mt[k].q.x), dmax(dmax(hi.y, mt[k].p.y), mt[k].q.y),
                   dmax(dmax(hi.z, mt[k].p.z), mt[k].q.z));
        }
        const v3 center = vscale(0.5, vadd(lo, hi));
        const v3 ext = vsub(hi, lo);
        const v3 scale = V(dmax(ext.x, mp->shrink_floor), dmax(ext.y, mp->shrink_floor), dmax(ext.z, mp->shrink_floor));
        const v3 inv = V(1.0 / scale.x, 1.0 / scale.y, 1.0 / scale.z);
        /* assemble (registration.cpp:93-123) */
        kahan_t up[21], rhs[6], rsq;
        memset(up, 0, sizeof up);
        memset(rhs, 0, sizeof rhs);
        memset(&rsq, 0, sizeof rsq);
        for (size_t k = 0; k < nm; ++k) {
            const v3 ph = vmul(inv, vsub(mt[k].p, center)), qh = vmul(inv, vsub(mt[k].q, center));
            const v3 ch = vmul(inv, vsub(vcross(mt[k].p, mt[k].n), vcross(center, mt[k].n)));
            const double row[6] = {ch.x, ch.y, ch.z, mt[k].n.x, mt[k].n.y, mt[k].n.z};
            const double d = vdot(vmul(scale, vsub(ph, qh)), mt[k].n);
            int kk = 0;
            for (int a = 0; a < 6; ++a)
                for (int b = a; b < 6; ++b, ++kk) kadd(&up[kk], row[a] * row[b]);
            for (int a = 0; a < 6; ++a) kadd(&rhs[a], -row[a] * d);
            kadd(&rsq, d * d);
        }
        double A[36], bvec[6];
        int kk = 0;
        for (int a = 0; a < 6; ++a)
            for (int b = a; b < 6; ++b, ++kk) A[a * 6 + b] = A[b * 6 + a] = up[kk].sum;
        for (int a = 0; a < 6; ++a) bvec[a] = rhs[a].sum;
        /* solve_gated (registration.cpp:175-193) */
        res->pair_count = nm;
        res->residual_rms = sqrt(dmax(0.0, rsq.sum) / (double)nm);
        eigen6(A, res->eigenvalues, res->eigenvectors);
        double x[6] = {0, 0, 0, 0, 0, 0};
        for (int i = 0; i < 6; ++i) {
            res->gated_mask[i] = res->eigenvalues[i] / (double)nm > mp->eigen_threshold;
            if (!res->gated_mask[i]) continue;
            const double* vc = res->eigenvectors + i * 6;
            double vb = vc[0] * bvec[0];
            for (int r = 1; r < 6; ++r) vb = vb + vc[r] * bvec[r];
            const double sc = vb / res->eigenvalues[i];
            for (int r = 0; r < 6; ++r) x[r] = x[r] + vc[r] * sc;
        }
        double xn = x[0] * x[0];
        for (int r = 1; r < 6; ++r) xn = xn + x[r] * x[r];
        res->shrunk_motion_norm = sqrt(xn);
        /* unshrink_motion (registration.cpp:167-173) */
        const v3 mr = V((1.0 / scale.x) * x[0], (1.0 / scale.y) * x[1], (1.0 / scale.z) * x[2]);
        const v3 mtv = vsub(V(x[3], x[4], x[5]), vcross(mr, center));
        res->motion_r[0] = mr.x;
        res->motion_r[1] = mr.y;
        res->motion_r[2] = mr.z;
        res->motion_t[0] = mtv.x;
        res->motion_t[1] = mtv.y;
        res->motion_t[2] = mtv.z;
        delta = apply_motion(&delta, mr, mtv);
        res->iterations = iter + 1;
        if (res->shrunk_motion_norm < mp->convergence_epsilon) break;
    }
    pose_to(delta, res->delta);
    free(mt);
    free(sn_owned);
    return status;
}

/* ---------------------------------------------------------------------------------------
 * synthetic depth, noise-free (scene.cpp:13-147); noisy frames come from the reference build
 * ------------------------------------------------------------------------------------- */
int sfo_render_synthetic_depth(const sf_scene* sc, const double* pose12, const sf_intrinsics* I, double sigma0,
                               uint64_t seed, int32_t max_steps, double tol_scale, double domain, float* depth,
                               float* sigma) {
    (void)seed;
    int st = validate_intr(I);
    if (st) return st;
    if (sigma0 > 0.0) return fail(SF_UNSUPPORTED, "oracle: noisy frames are checked against the reference build");
    const int w = I->width, h = I->height;
    memset(depth, 0, sizeof(float) * (size_t)w * h);
    if (sigma) memset(sigma, 0, sizeof(float) * (size_t)w * h);
    if (sc->sphere_count + sc->plane_count + sc->box_count == 0) return SF_OK;
    double* pl = malloc((size_t)(4 * sc->plane_count + 1) * sizeof(double));
    for (int i = 0; i < sc->plane_count; ++i) { /* AnalyticScene::add_plane (scene.cpp:53-57) */
        const double* p = sc->planes + 4 * i;
        const double len = sqrt((p[0] * p[0] + p[1] * p[1]) + p[2] * p[2]);
        for (int k = 0; k < 4; ++k) pl[4 * i + k] = p[k] / len;
    }
    const pose_t pose = pose_from(pose12);
    const double tolerance = tol_scale * domain;
    for (int v = 0; v < h; ++v)
        for (int u = 0; u < w; ++u) {
            const v3 dc = vnormalized(unproject(I, u, v, 1.0));
            const v3 dir = mv(pose.R, dc);
            const double t_near = I->near_plane / dc.z, t_far = I->far_plane / dc.z;
            double t = t_near, d_out = 0.0;
            for (int step = 0; step < max_steps && t <= t_far; ++step) {
                const v3 x = vadd(pose.t, vscale(t, dir));
                double best = INFINITY;
                for (int i = 0; i < sc->sphere_count; ++i) {
                    const double* s = sc->spheres + 4 * i;
                    const v3 r = vsub(x, V(s[0], s[1], s[2]));
                    best = dmin(best, sqrt(vdot(r, r)) - s[3]);
                }
                for (int i = 0; i < sc->plane_count; ++i)
                    best = dmin(best, vdot(V(pl[4 * i], pl[4 * i + 1], pl[4 * i + 2]), x) - pl[4 * i + 3]);
                for (int i = 0; i < sc->box_count; ++i) {
                    const double* b = sc->boxes + 6 * i;
                    const v3 local = vsub(x, V(b[0], b[1], b[2])); /* identity rotation */
                    const v3 q = vsub(V(fabs(local.x), fabs(local.y), fabs(local.z)), V(b[3], b[4], b[5]));
                    const v3 o = V(dmax(q.x, 0.0), dmax(q.y, 0.0), dmax(q.z, 0.0));
                    double mx = q.x;
                    mx = mx < q.y ? q.y : mx;
                    mx = mx < q.z ? q.z : mx;
                    best = dmin(best, sqrt(vdot(o, o)) + dmin(mx, 0.0));
                }
                if (best < tolerance) {
                    d_out = t * dc.z;
                    break;
                }
                t += best;
            }
            if (d_out <= 0.0) continue;
            if (d_out < I->near_plane || d_out > I->far_plane) continue;
            depth[(size_t)v * w + u] = (float)d_out;
        }
    free(pl);
    return SF_OK;
}
