// sf_mesh.cu — sparse marching cubes on the device (marching_cubes.cpp:74-196).
//
// Same mesh as the reference, vertex for vertex and triangle for triangle:
//   block list   allocated blocks in table order (or the frustum-filtered ones,
//                grid.cpp:162-172, 222-269): slot index -> keys, radix sort, stable filter
//   count        one CTA per block, a thread per cube: the 8 corner codes, the case index,
//                the triangle count (marching_cubes.cpp:36-59, 85-95)
//   batches      the greedy memory-budget grouping of blocks (:97-108), on the host over
//                the per-block counts; it scopes vertex welding
//   offsets      exclusive scan of the per-cube counts: every triangle's position in the
//                reference's emission order (block, z, y, x, table order)
//   corners      each triangle corner -> (batch, cube-edge id) (:61-72); a hash table keeps
//                the first position that names each edge: the reference creates a vertex at
//                the first reference to its edge in a batch (:118-126), so vertex numbers are
//                the ranks of those first positions (scan)
//   vertices     position from the first-referencing cube's corner values (:127-138, the
//                edge direction of that cube matters for the rounding), normal from the
//                TSDF gradient at h = voxel, then 0.5 voxel (:140-143)
//   triangles    winding flipped to (0, 2, 1), degenerate ones (|cross| <= 1e-12) dropped
//                (:150-158); vertices without a gradient normal take the normalised sum of
//                their faces' cross products in float, accumulated in triangle order (:165-180)
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <vector>

#include "sf_internal.h"
#include "sf_sample.cuh"

namespace sf {

// Canonical marching-cubes triangle table (Lorensen & Cline case set in P. Bourke's
// numbering, as used by marching_cubes.cpp): case c, entry i = nibble i of kTri[c]
// (0..11 = cube edge, 15 = end of list).
__constant__ unsigned long long kTri[256] = {
    0xffffffffffffffffull, 0xfffffffffffff380ull, 0xfffffffffffff910ull, 0xffffffffff189381ull,
    0xfffffffffffffa21ull, 0xffffffffffa21380ull, 0xffffffffff920a29ull, 0xfffffff89a8a2382ull,
    0xfffffffffffff2b3ull, 0xffffffffff0b82b0ull, 0xffffffffffb32091ull, 0xfffffffb89b912b1ull,
    0xffffffffff3ab1a3ull, 0xfffffffab8a801a0ull, 0xfffffff9ab9b3093ull, 0xffffffffffb8aa89ull,
    0xfffffffffffff874ull, 0xffffffffff437034ull, 0xffffffffff748910ull, 0xfffffff137174914ull,
    0xffffffffff748a21ull, 0xfffffffa21403743ull, 0xfffffff748209a29ull, 0xffff4973727929a2ull,
    0xffffffffff2b3748ull, 0xfffffff40242b74bull, 0xfffffffb32748109ull, 0xffff1292b9b49b74ull,
    0xfffffff487ab31a3ull, 0xffff4b7401b41ab1ull, 0xffff30bab9b09874ull, 0xfffffffab99b4b74ull,
    0xfffffffffffff459ull, 0xffffffffff380459ull, 0xffffffffff051450ull, 0xfffffff513538458ull,
    0xffffffffff459a21ull, 0xfffffff594a21803ull, 0xfffffff204245a25ull, 0xffff8434535235a2ull,
    0xffffffffffb32459ull, 0xfffffff594b802b0ull, 0xfffffffb32510450ull, 0xffff584b82852512ull,
    0xfffffff45931ab3aull, 0xffffab81a8180594ull, 0xffff30bab5b05045ull, 0xfffffffb8aa85845ull,
    0xffffffffff975879ull, 0xfffffff375359039ull, 0xfffffff751710870ull, 0xffffffffff753351ull,
    0xfffffff21a759879ull, 0xffff37503505921aull, 0xffff25a758528208ull, 0xfffffff7533525a2ull,
    0xfffffff2b3987597ull, 0xffffb72029279759ull, 0xffff751871810b32ull, 0xfffffff51771b12bull,
    0xffffb3a31a758859ull, 0xf0aba010b7905075ull, 0xf07570805a30b0abull, 0xffffffffff5b75abull,
    0xfffffffffffff56aull, 0xffffffffff6a5380ull, 0xffffffffff6a5109ull, 0xfffffff6a5891381ull,
    0xffffffffff162561ull, 0xfffffff803621561ull, 0xfffffff620609569ull, 0xffff823625285895ull,
    0xffffffffff56ab32ull, 0xfffffff56a02b80bull, 0xfffffff6a5b32910ull, 0xffffb892b92916a5ull,
    0xfffffff315356b36ull, 0xffff6b51505b0b80ull, 0xffff9505606306b3ull, 0xfffffff89bb96956ull,
    0xffffffffff8746a5ull, 0xfffffffa56374034ull, 0xfffffff7486a5091ull, 0xffff49737179156aull,
    0xfffffff874156216ull, 0xffff743403625521ull, 0xffff620560509748ull, 0xf962695923497937ull,
    0xfffffff56a4872b3ull, 0xffffb720242746a5ull, 0xffff6a5b32874910ull, 0xf6a54b7b492b9129ull,
    0xffff6b51535b3748ull, 0xfb404b7b016b5b15ull, 0xf74836b630560950ull, 0xffff9b7974b96956ull,
    0xffffffffffa4694aull, 0xfffffff380a946a4ull, 0xfffffff04606a10aull, 0xffffa16468618138ull,
    0xfffffff462421941ull, 0xffff462942921803ull, 0xffffffffff624420ull, 0xfffffff624428238ull,
    0xfffffff32b46a94aull, 0xffff6a4a94b82280ull, 0xffffa164606102b3ull, 0xf1b8b12184a16146ull,
    0xffff36b319639469ull, 0xf14641916b0181b8ull, 0xfffffff4600636b3ull, 0xffffffffff86b846ull,
    0xfffffffa98a876a7ull, 0xffffa76a907a0370ull, 0xffff0818717a176aull, 0xfffffff37117a76aull,
    0xffff768981861621ull, 0xf937390976192962ull, 0xfffffff206607087ull, 0xffffffffff276237ull,
    0xffff76898a86ab32ull, 0xf7a9a76790b72702ull, 0xfb32a767a1871081ull, 0xffff17616a71b12bull,
    0xf63136b619768698ull, 0xffffffffff76b190ull, 0xffff06b0b3607087ull, 0xfffffffffffff6b7ull,
    0xfffffffffffffb67ull, 0xffffffffff67b803ull, 0xffffffffff67b910ull, 0xfffffff67b138918ull,
    0xffffffffff7b621aull, 0xfffffff7b6803a21ull, 0xfffffff7b69a2092ull, 0xffff89a38a3a27b6ull,
    0xffffffffff726327ull, 0xfffffff026067807ull, 0xfffffff910732672ull, 0xffff678891681261ull,
    0xfffffff73171a67aull, 0xffff801781a7167aull, 0xffff7a69a0a70730ull, 0xfffffff9a88a7a67ull,
    0xffffffffff68b486ull, 0xfffffff640603b63ull, 0xfffffff109648b68ull, 0xffff63b139369649ull,
    0xfffffff1a28b6486ull, 0xffff640b60b03a21ull, 0xffff9a2920b648b4ull, 0xf36463b34923a39aull,
    0xfffffff264248328ull, 0xffffffffff264240ull, 0xffff834642432091ull, 0xfffffff642241491ull,
    0xffff1a6648168318ull, 0xfffffff40660a01aull, 0xf39a9303a6834364ull, 0xffffffffff4a649aull,
    0xffffffffffb67594ull, 0xfffffff67b594380ull, 0xfffffffb67045105ull, 0xffff51345343867bull,
    0xfffffffb6721a459ull, 0xffff594380a217b6ull, 0xffff204a24a45b67ull, 0xf67b25a523453843ull,
    0xfffffff945267327ull, 0xffff786260680459ull, 0xffff045051673263ull, 0xf851584812786826ull,
    0xffff73167161a459ull, 0xf459078701671a61ull, 0xfa737a6a305a4a04ull, 0xffffa84a458a7a67ull,
    0xfffffff98b9b6596ull, 0xffff590650360b63ull, 0xffffb65510b508b0ull, 0xfffffff1355363b6ull,
    0xffff65b8b9b59a21ull, 0xfa21965690b603b0ull, 0xf52025a50865b58bull, 0xffff35a3a25363b6ull,
    0xffff283265825985ull, 0xfffffff260069659ull, 0xf826283865081851ull, 0xffffffffff612651ull,
    0xf698965683a61631ull, 0xffff06505960a01aull, 0xffffffffffa65830ull, 0xfffffffffffff65aull,
    0xffffffffffb57a5bull, 0xfffffff03857ba5bull, 0xfffffff091ba57b5ull, 0xffff1381897ba57aull,
    0xfffffff15717b21bull, 0xffffb27571721380ull, 0xffff7b2209729579ull, 0xf289823295b27257ull,
    0xfffffff573532a52ull, 0xffff52a578258028ull, 0xffff2a37353a5109ull, 0xf25752a278129289ull,
    0xffffffffff573531ull, 0xfffffff571170780ull, 0xfffffff735539309ull, 0xffffffffff795789ull,
    0xfffffff8ba8a5485ull, 0xffff03bba50b5405ull, 0xffff54aba8a48910ull, 0xf41314943b54a4baull,
    0xffff8548b2582152ull, 0xfb151b2b543b0b40ull, 0xf58b8545b2950520ull, 0xffffffffff3b2549ull,
    0xffff483543253a52ull, 0xfffffff0244252a5ull, 0xf910854583a532a3ull, 0xffff2492914252a5ull,
    0xfffffff153358548ull, 0xffffffffff501540ull, 0xffff530509358548ull, 0xfffffffffffff549ull,
    0xfffffffba9b947b4ull, 0xffffba97b9794380ull, 0xffffb470414b1ba1ull, 0xf4bab474a1843413ull,
    0xffff219b294b97b4ull, 0xf3801b2b197b9479ull, 0xfffffff04224b47bull, 0xffff42343824b47bull,
    0xffff947732972a92ull, 0xf70207872a4797a9ull, 0xfa040a1a472a3a73ull, 0xffffffffff4782a1ull,
    0xfffffff317714194ull, 0xffff178180714194ull, 0xffffffffff347304ull, 0xfffffffffffff784ull,
    0xffffffffff8ba8a9ull, 0xfffffffa9bb93903ull, 0xfffffffba88a0a10ull, 0xffffffffffa3ba13ull,
    0xfffffff8b99b1b21ull, 0xffff9b2921b93903ull, 0xffffffffffb08b20ull, 0xfffffffffffffb23ull,
    0xfffffff98aa82832ull, 0xffffffffff2902a9ull, 0xffff8a1810a82832ull, 0xfffffffffffff2a1ull,
    0xffffffffff819831ull, 0xfffffffffffff190ull, 0xfffffffffffff830ull, 0xffffffffffffffffull,};
__device__ __forceinline__ int tri_entry(int c, int i) { return static_cast<int>((kTri[c] >> (4 * i)) & 0xF); }

// Corner numbering (marching_cubes.cpp:14-19): 0 (0,0,0), 1 (1,0,0), 2 (1,1,0), 3 (0,1,0), then
// z + 1 for 4..7; edge e joins corners kEdge[e][0] -> kEdge[e][1].
__constant__ int kCorner[8][3] = {{0, 0, 0}, {1, 0, 0}, {1, 1, 0}, {0, 1, 0}, {0, 0, 1}, {1, 0, 1}, {1, 1, 1}, {0, 1, 1}};
__constant__ int kEdge[12][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 0}, {4, 5}, {5, 6}, {6, 7}, {7, 4}, {0, 4}, {1, 5}, {2, 6}, {3, 7}};

constexpr unsigned long long kHashEmpty = ~0ull;

// fetch_tsdf (marching_cubes.cpp:21-30): false for an EMPTY block or a chi voxel.
__device__ __forceinline__ bool mc_fetch(const VolParams& P, const int32_t* __restrict__ table,
                                         const uint16_t* __restrict__ payload, const double* tdec, int x, int y,
                                         int z, double& out) {
    const int M = P.M;
    const int bx = x / M, by = y / M, bz = z / M;
    const int32_t slot = __ldg(&table[table_index(P, bx, by, bz)]);
    if (slot == kEmpty) return false;
    const uint16_t pl = __ldg(&payload[(size_t)slot * P.M3 + ((z - bz * M) * M + (y - by * M)) * M + (x - bx * M)]);
    const int8_t c = static_cast<int8_t>(pl & 0xFF);
    if (c == kChiCode) return false;
    out = tdec[(int)c + 128];
    return true;
}

// sample_cube (marching_cubes.cpp:38-49): case index, or -1 when not usable.
__device__ int mc_cube(const VolParams& P, const int32_t* __restrict__ table, const uint16_t* __restrict__ payload,
                       const double* tdec, int x, int y, int z, double v[8]) {
    int idx = 0;
    for (int i = 0; i < 8; ++i) {
        if (!mc_fetch(P, table, payload, tdec, x + kCorner[i][0], y + kCorner[i][1], z + kCorner[i][2], v[i]))
            return -1;
        if (v[i] < 0.0) idx |= 1 << i;
    }
    return (idx != 0 && idx != 255) ? idx : -1;
}

__device__ __forceinline__ int mc_count(int idx) {  // cube_triangle_count (:51-56)
    if (idx < 0) return 0;
    int n = 0;
    while (n < 5 && tri_entry(idx, 3 * n) != 15) ++n;
    return n;
}

// edge_key (marching_cubes.cpp:61-72)
__device__ __forceinline__ unsigned long long mc_edge_key(int x, int y, int z, int edge, int res) {
    const int* ca = kCorner[kEdge[edge][0]];
    const int* cb = kCorner[kEdge[edge][1]];
    const int a[3] = {x + ca[0], y + ca[1], z + ca[2]}, b[3] = {x + cb[0], y + cb[1], z + cb[2]};
    int axis = 0;
    for (int i = 0; i < 3; ++i)
        if (a[i] != b[i]) axis = i;
    const int* lo = a[axis] < b[axis] ? a : b;
    return ((static_cast<unsigned long long>(lo[2]) * res + lo[1]) * res + lo[0]) * 3 + axis;
}

__device__ __forceinline__ unsigned long long mix64(unsigned long long k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdull;
    k ^= k >> 33;
    k *= 0xc4ceb9fe1a85ec53ull;
    k ^= k >> 33;
    return k;
}

// Cube (block i of the list, local cube l) -> voxel coordinates of its base corner.
__device__ __forceinline__ void mc_base(const VolParams& P, const uint32_t* __restrict__ blocks, uint32_t cube, int& x,
                                        int& y, int& z) {
    const int M = P.M;
    const uint32_t bi = cube / P.M3, l = cube % P.M3;
    const uint32_t key = blocks[bi];
    const int bx = key % P.N, by = (key / P.N) % P.N, bz = key / (P.N * P.N);
    x = bx * M + static_cast<int>(l % M);
    y = by * M + static_cast<int>((l / M) % M);
    z = bz * M + static_cast<int>(l / (M * M));
}

__device__ __forceinline__ uint32_t warp_push(bool pred, uint32_t* counter) {
    const unsigned am = __activemask();
    const unsigned bal = __ballot_sync(am, pred);
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (bal) {
        const int leader = __ffs(bal) - 1;
        if (lane == leader) base = atomicAdd(counter, static_cast<uint32_t>(__popc(bal)));
        base = __shfl_sync(am, base, leader);
    }
    return base + __popc(bal & ((1u << lane) - 1u));
}

// Allocated blocks (slot -> table index), any order.
__global__ void k_mc_collect(const int32_t* __restrict__ slot_key, const VolCounters* __restrict__ vc,
                             uint32_t* __restrict__ keys, uint32_t* count) {
    const unsigned long long hw = vc->high_water;
    for (unsigned long long s = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; s < hw;
         s += (unsigned long long)gridDim.x * blockDim.x) {
        const int32_t key = slot_key[s];
        const uint32_t j = warp_push(key >= 0, count);
        if (key >= 0) keys[j] = static_cast<uint32_t>(key);
    }
}

// occupied_blocks_in_frustum (grid.cpp:228-269): the region's SAT test per listed block.
__global__ void k_mc_frustum(VolParams P, const FrameConsts* __restrict__ fc, const uint32_t* __restrict__ keys,
                             const uint32_t* count, uint8_t* __restrict__ keep) {
    const uint32_t n = *count;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t key = keys[i];
        const int bx = key % P.N, by = (key / P.N) % P.N, bz = key / (P.N * P.N);
        const d3 lo = block_min_corner(P, bx, by, bz);
        const double side = P.block_side;
        keep[i] = frustum_intersects_block(P, fc, lo, add(lo, mk(side, side, side))) ? 1 : 0;
    }
}

// Count pass: triangles per cube and per block.
__global__ void k_mc_count(VolParams P, const int32_t* __restrict__ table, const uint16_t* __restrict__ payload,
                           const AuxTables* __restrict__ aux, const uint32_t* __restrict__ blocks,
                           uint32_t* __restrict__ cube_tris, uint32_t* __restrict__ block_tris) {
    __shared__ double s_tdec[256];
    __shared__ uint32_t s_sum;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_tdec[i] = aux->tsdf_decode[i];
    if (threadIdx.x == 0) s_sum = 0;
    __syncthreads();
    const uint32_t bi = blockIdx.x;
    uint32_t local = 0;
    for (int l = threadIdx.x; l < P.M3; l += blockDim.x) {
        int x, y, z;
        mc_base(P, blocks, bi * P.M3 + l, x, y, z);
        int c = 0;
        if (x + 1 < P.res && y + 1 < P.res && z + 1 < P.res) {
            double v[8];
            c = mc_count(mc_cube(P, table, payload, s_tdec, x, y, z, v));
        }
        cube_tris[(size_t)bi * P.M3 + l] = c;
        local += c;
    }
    for (int off = 16; off > 0; off >>= 1) local += __shfl_down_sync(0xffffffffu, local, off);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(&s_sum, local);
    __syncthreads();
    if (threadIdx.x == 0) block_tris[bi] = s_sum;
}

// Corners: (batch, edge id) of every triangle corner at its reference position, and the
// first position naming each edge (hash table, atomicMin).
__global__ void k_mc_corners(VolParams P, const int32_t* __restrict__ table, const uint16_t* __restrict__ payload,
                             const AuxTables* __restrict__ aux, const uint32_t* __restrict__ blocks, uint64_t n_cubes,
                             const uint32_t* __restrict__ cube_tris, const uint32_t* __restrict__ tri_off,
                             const uint32_t* __restrict__ block_batch, unsigned long long* __restrict__ corner_key,
                             uint32_t* __restrict__ corner_cube, unsigned long long* __restrict__ hkeys,
                             uint32_t* __restrict__ hvals, unsigned long long hmask) {
    __shared__ double s_tdec[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_tdec[i] = aux->tsdf_decode[i];
    __syncthreads();
    for (uint64_t cube = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; cube < n_cubes;
         cube += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t c = cube_tris[cube];
        if (!c) continue;
        int x, y, z;
        mc_base(P, blocks, static_cast<uint32_t>(cube), x, y, z);
        double v[8];
        const int idx = mc_cube(P, table, payload, s_tdec, x, y, z, v);
        const unsigned long long batch = block_batch[cube / P.M3];
        for (uint32_t k = 0; k < c; ++k)
            for (int e = 0; e < 3; ++e) {
                const unsigned long long key = mc_edge_key(x, y, z, tri_entry(idx, 3 * k + e), P.res) | (batch << 42);
                const uint32_t pos = 3 * (tri_off[cube] + k) + e;
                corner_key[pos] = key;
                corner_cube[pos] = static_cast<uint32_t>(cube);
                unsigned long long h = mix64(key) & hmask;
                for (;;) {
                    const unsigned long long prev = atomicCAS(&hkeys[h], kHashEmpty, key);
                    if (prev == kHashEmpty || prev == key) {
                        atomicMin(&hvals[h], pos);
                        break;
                    }
                    h = (h + 1) & hmask;
                }
            }
    }
}

__global__ void k_mc_first(const unsigned long long* __restrict__ corner_key, uint64_t n_corners,
                           const unsigned long long* __restrict__ hkeys, const uint32_t* __restrict__ hvals,
                           unsigned long long hmask, uint32_t* __restrict__ corner_slot, uint32_t* __restrict__ first) {
    for (uint64_t pos = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; pos < n_corners;
         pos += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long key = corner_key[pos];
        unsigned long long h = mix64(key) & hmask;
        while (hkeys[h] != key) h = (h + 1) & hmask;
        corner_slot[pos] = static_cast<uint32_t>(h);
        first[pos] = hvals[h] == pos ? 1u : 0u;
    }
}

// Vertices, created where their edge is first named (marching_cubes.cpp:118-146).
__global__ void k_mc_vertices(VolParams P, const int32_t* __restrict__ table, const uint16_t* __restrict__ payload,
                              const uint32_t* __restrict__ occ, const AuxTables* __restrict__ aux,
                              const uint32_t* __restrict__ blocks, uint64_t n_corners,
                              const uint32_t* __restrict__ first, const uint32_t* __restrict__ vnum,
                              const uint32_t* __restrict__ corner_slot, const uint32_t* __restrict__ corner_cube,
                              const uint32_t* __restrict__ tri_off, uint32_t* __restrict__ slot_vidx,
                              float* __restrict__ vert, float* __restrict__ nrm, uint8_t* __restrict__ pending) {
    __shared__ double s_tdec[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) s_tdec[i] = aux->tsdf_decode[i];
    __syncthreads();
    const Sampler S{P, table, payload, occ, s_tdec};
    const double vox = P.voxel;
    for (uint64_t pos = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; pos < n_corners;
         pos += (uint64_t)gridDim.x * blockDim.x) {
        if (!first[pos]) continue;
        const uint32_t vi = vnum[pos];
        slot_vidx[corner_slot[pos]] = vi;
        const uint32_t cube = corner_cube[pos];
        int x, y, z;
        mc_base(P, blocks, cube, x, y, z);
        double v[8];
        const int idx = mc_cube(P, table, payload, s_tdec, x, y, z, v);
        const uint32_t k = static_cast<uint32_t>(pos / 3) - tri_off[cube];
        const int edge = tri_entry(idx, 3 * k + static_cast<int>(pos % 3));
        const int a = kEdge[edge][0], b = kEdge[edge][1];
        const double va = v[a], vb = v[b];
        const double t = va / (va - vb);  // zero crossing
        const d3 pa = voxel_center(P, x + kCorner[a][0], y + kCorner[a][1], z + kCorner[a][2]);
        const d3 pb = voxel_center(P, x + kCorner[b][0], y + kCorner[b][1], z + kCorner[b][2]);
        const d3 p = add(pa, scale(t, sub(pb, pa)));
        float nx = 0.f, ny = 0.f, nz = 0.f;
        d3 g;
        int64_t ckey = -1;  // block-slot cache of the near-surface sampler (same values as sample())
        int32_t cslot = kEmpty;
        bool ok = S.gradient_near(p, vox, g, ckey, cslot);
        if (!ok) ok = S.gradient_near(p, 0.5 * vox, g, ckey, cslot);
        if (ok && sqnorm(g) > 0.0) {
            const d3 n = normalized(g);
            nx = (float)n.x;
            ny = (float)n.y;
            nz = (float)n.z;
        }
        vert[3 * vi] = (float)p.x;
        vert[3 * vi + 1] = (float)p.y;
        vert[3 * vi + 2] = (float)p.z;
        // no gradient normal: the face-normal fallback overwrites this; a vertex in no kept
        // triangle keeps UnitZ (marching_cubes.cpp:176-178)
        const bool pend = (nx * nx + ny * ny) + nz * nz == 0.0f;
        nrm[3 * vi] = nx;
        nrm[3 * vi + 1] = ny;
        nrm[3 * vi + 2] = pend ? 1.0f : nz;
        pending[vi] = pend ? 1 : 0;
    }
}

// Triangles: winding (0, 2, 1); degenerate ones dropped (marching_cubes.cpp:147-158).
__global__ void k_mc_keep(uint64_t n_tris, const uint32_t* __restrict__ corner_slot,
                          const uint32_t* __restrict__ slot_vidx, const float* __restrict__ vert,
                          uint32_t* __restrict__ keep, uint3* __restrict__ tri_v) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_tris;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i0 = slot_vidx[corner_slot[3 * t]], i1 = slot_vidx[corner_slot[3 * t + 1]],
                       i2 = slot_vidx[corner_slot[3 * t + 2]];
        const d3 v0 = mk(vert[3 * i0], vert[3 * i0 + 1], vert[3 * i0 + 2]);
        const d3 v1 = mk(vert[3 * i2], vert[3 * i2 + 1], vert[3 * i2 + 2]);
        const d3 v2 = mk(vert[3 * i1], vert[3 * i1 + 1], vert[3 * i1 + 2]);
        const double nn = sqrt(sqnorm(cross(sub(v1, v0), sub(v2, v0))));
        keep[t] = nn <= 1e-12 ? 0u : 1u;
        tri_v[t] = make_uint3(i0, i2, i1);
    }
}

__global__ void k_mc_emit(uint64_t n_tris, const uint32_t* __restrict__ keep, const uint32_t* __restrict__ out_pos,
                          const uint3* __restrict__ tri_v, uint3* __restrict__ tris) {
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n_tris;
         t += (uint64_t)gridDim.x * blockDim.x)
        if (keep[t]) tris[out_pos[t]] = tri_v[t];
}

// Face-normal fallback (marching_cubes.cpp:162-180): records (vertex, triangle) of pending
// vertices, sorted, then each vertex sums its faces in triangle order (float).
__global__ void k_mc_pending_records(uint64_t n_out, const uint3* __restrict__ tris, const uint8_t* __restrict__ pending,
                                     unsigned long long* __restrict__ rec) {
    for (uint64_t o = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; o < n_out;
         o += (uint64_t)gridDim.x * blockDim.x) {
        const uint3 t = tris[o];
        const uint32_t v[3] = {t.x, t.y, t.z};
        for (int j = 0; j < 3; ++j)
            rec[3 * o + j] = pending[v[j]] ? ((static_cast<unsigned long long>(v[j]) << 32) | o) : ~0ull;
    }
}
__device__ __forceinline__ float3 fsub(float3 a, float3 b) { return make_float3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ float3 fcross(float3 a, float3 b) {
    return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__global__ void k_mc_pending_normals(uint64_t n_rec, const unsigned long long* __restrict__ rec,
                                     const uint3* __restrict__ tris, const float* __restrict__ vert,
                                     float* __restrict__ nrm) {
    auto V = [&](uint32_t i) { return make_float3(vert[3 * i], vert[3 * i + 1], vert[3 * i + 2]); };
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_rec;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const unsigned long long r = rec[i];
        if (r == ~0ull) continue;
        const uint32_t vtx = static_cast<uint32_t>(r >> 32);
        if (i > 0 && static_cast<uint32_t>(rec[i - 1] >> 32) == vtx && rec[i - 1] != ~0ull) continue;
        float3 acc = make_float3(0.f, 0.f, 0.f);
        for (uint64_t j = i; j < n_rec && rec[j] != ~0ull && static_cast<uint32_t>(rec[j] >> 32) == vtx; ++j) {
            const uint3 t = tris[static_cast<uint32_t>(rec[j])];
            const float3 a = V(t.x);
            const float3 f = fcross(fsub(V(t.y), a), fsub(V(t.z), a));
            acc = make_float3(acc.x + f.x, acc.y + f.y, acc.z + f.z);
        }
        const float len = sqrtf((acc.x * acc.x + acc.y * acc.y) + acc.z * acc.z);
        if (len > 0.0f) {
            nrm[3 * vtx] = acc.x / len;
            nrm[3 * vtx + 1] = acc.y / len;
            nrm[3 * vtx + 2] = acc.z / len;
        } else {
            nrm[3 * vtx] = 0.0f;
            nrm[3 * vtx + 1] = 0.0f;
            nrm[3 * vtx + 2] = 1.0f;
        }
    }
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf(size_t n, cudaStream_t st) : s(st) {
        if (n) SF_CUDA(cudaMallocAsync(&p, n * sizeof(T), s));
    }
    ~DevBuf() {
        if (p) cudaFreeAsync(p, s);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

template <typename In, typename Out>
static void exclusive_sum(const In* in, Out* out, uint64_t n, cudaStream_t s) {
    size_t tb = 0;
    SF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, (int64_t)n, s));
    DevBuf<char> tmp(tb, s);
    SF_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, tb, in, out, (int64_t)n, s));
}

}  // namespace sf

struct sf_mesh {
    int device = 0;
    uint64_t nv = 0, nt = 0;
    float* vert = nullptr;
    float* nrm = nullptr;
    uint32_t* tris = nullptr;
    ~sf_mesh() {
        cudaSetDevice(device);
        if (vert) cudaFree(vert);
        if (nrm) cudaFree(nrm);
        if (tris) cudaFree(tris);
    }
};

using namespace sf;

extern "C" {

int sf_marching_cubes(sf_volume_t v, const double region_pose[12], const sf_intrinsics* region_intrinsics,
                      uint64_t batch_memory_budget, sf_mesh_t* out, void* stream) {
    return guarded([&]() -> int {
        if (v) require_codes(*v, "marching_cubes");
        if (!v || !out) throw Error(SF_INVALID_ARGUMENT, "sf_marching_cubes: null argument");
        if ((region_pose == nullptr) != (region_intrinsics == nullptr))
            throw Error(SF_INVALID_ARGUMENT, "sf_marching_cubes: region needs both pose and intrinsics");
        SF_CUDA(cudaSetDevice(v->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const VolParams& P = v->P;
        const uint64_t budget = batch_memory_budget ? batch_memory_budget : (64ull << 20);  // marching_cubes.hpp:42
        // ---- block list in table order (allocated_blocks / occupied_blocks_in_frustum)
        const uint64_t cap = P.capacity;
        DevBuf<uint32_t> keys(cap + 1, s), keys_sorted(cap + 1, s), counters(2, s);
        SF_CUDA(cudaMemsetAsync(counters.p, 0, 2 * sizeof(uint32_t), s));
        k_mc_collect<<<148 * 4, 256, 0, s>>>(v->d_slot_key, v->d_vc, keys.p, counters.p);
        SF_LAUNCH_CHECK();
        uint32_t nb = 0;
        SF_CUDA(cudaMemcpyAsync(&nb, counters.p, sizeof(nb), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        uint32_t* blocks = keys_sorted.p;
        if (nb) {
            size_t tb = 0;
            SF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, keys.p, keys_sorted.p, (int)nb, 0, 32, s));
            DevBuf<char> tmp(tb, s);
            SF_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, keys.p, keys_sorted.p, (int)nb, 0, 32, s));
        }
        if (nb && region_pose) {
            if (region_intrinsics->width <= 0 || region_intrinsics->height <= 0 || region_intrinsics->fx <= 0.0 ||
                region_intrinsics->fy <= 0.0 || !(region_intrinsics->near_plane > 0.0) ||
                !(region_intrinsics->near_plane < region_intrinsics->far_plane))
                throw Error(SF_INVALID_ARGUMENT, "intrinsics: invalid region camera");
            DevBuf<double> d_pose(12, s);
            DevBuf<FrameConsts> fc(1, s);
            DevBuf<uint8_t> flag(nb, s);
            SF_CUDA(cudaMemcpyAsync(d_pose.p, region_pose, 12 * sizeof(double), cudaMemcpyHostToDevice, s));
            SF_CUDA(cudaMemcpyAsync(counters.p, &nb, sizeof(nb), cudaMemcpyHostToDevice, s));
            launch_consts(P, to_intr(*region_intrinsics), d_pose.p, fc.p, s, nullptr);
            k_mc_frustum<<<148 * 4, 256, 0, s>>>(P, fc.p, keys_sorted.p, counters.p, flag.p);
            SF_LAUNCH_CHECK();
            size_t tb = 0;
            SF_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, keys_sorted.p, flag.p, keys.p, counters.p + 1, (int)nb, s));
            DevBuf<char> tmp(tb, s);
            SF_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, keys_sorted.p, flag.p, keys.p, counters.p + 1, (int)nb, s));
            SF_CUDA(cudaMemcpyAsync(&nb, counters.p + 1, sizeof(nb), cudaMemcpyDeviceToHost, s));
            SF_CUDA(cudaStreamSynchronize(s));
            blocks = keys.p;
        }
        auto mesh = std::make_unique<sf_mesh>();
        mesh->device = v->device;
        if (nb == 0) {
            *out = mesh.release();
            return SF_OK;
        }
        // ---- count pass
        const uint64_t n_cubes = (uint64_t)nb * P.M3;
        DevBuf<uint32_t> cube_tris(n_cubes, s), tri_off(n_cubes, s), block_tris(nb, s), block_batch(nb, s);
        k_mc_count<<<nb, 256, 0, s>>>(P, v->d_table, v->d_payload, v->d_aux, blocks, cube_tris.p, block_tris.p);
        SF_LAUNCH_CHECK();
        std::vector<uint32_t> h_bt(nb), h_batch(nb);
        SF_CUDA(cudaMemcpyAsync(h_bt.data(), block_tris.p, nb * sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        // ---- batches: greedy grouping under the memory budget (marching_cubes.cpp:97-108)
        constexpr uint64_t kBytesPerTriangle = 3 * (2 * 3 * sizeof(float)) + 12;
        uint64_t batch_bytes = 0, total = 0;
        uint32_t batch = 0;
        for (uint32_t bi = 0; bi < nb; ++bi) {
            const uint64_t bytes = (uint64_t)h_bt[bi] * kBytesPerTriangle;
            if (batch_bytes > 0 && batch_bytes + bytes > budget) {
                ++batch;
                batch_bytes = 0;
            }
            batch_bytes += bytes;
            h_batch[bi] = batch;
            total += h_bt[bi];
        }
        if (total == 0) {
            *out = mesh.release();
            return SF_OK;
        }
        if (3 * total >= (1ull << 32)) throw Error(SF_OUT_OF_RANGE, "marching_cubes: mesh too large");
        SF_CUDA(cudaMemcpyAsync(block_batch.p, h_batch.data(), nb * sizeof(uint32_t), cudaMemcpyHostToDevice, s));
        exclusive_sum(cube_tris.p, tri_off.p, n_cubes, s);
        // ---- corners and first references
        const uint64_t n_corners = 3 * total;
        uint64_t hcap = 1024;
        while (hcap < 2 * n_corners) hcap <<= 1;
        DevBuf<unsigned long long> corner_key(n_corners, s), hkeys(hcap, s);
        DevBuf<uint32_t> corner_cube(n_corners, s), hvals(hcap, s), corner_slot(n_corners, s), first(n_corners, s),
            vnum(n_corners, s), slot_vidx(hcap, s);
        SF_CUDA(cudaMemsetAsync(hkeys.p, 0xff, hcap * sizeof(unsigned long long), s));
        SF_CUDA(cudaMemsetAsync(hvals.p, 0xff, hcap * sizeof(uint32_t), s));
        k_mc_corners<<<148 * 8, 256, 0, s>>>(P, v->d_table, v->d_payload, v->d_aux, blocks, n_cubes, cube_tris.p,
                                             tri_off.p, block_batch.p, corner_key.p, corner_cube.p, hkeys.p, hvals.p,
                                             hcap - 1);
        SF_LAUNCH_CHECK();
        k_mc_first<<<148 * 8, 256, 0, s>>>(corner_key.p, n_corners, hkeys.p, hvals.p, hcap - 1, corner_slot.p,
                                           first.p);
        SF_LAUNCH_CHECK();
        exclusive_sum(first.p, vnum.p, n_corners, s);
        uint32_t last_v = 0, last_f = 0;
        SF_CUDA(cudaMemcpyAsync(&last_v, vnum.p + n_corners - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaMemcpyAsync(&last_f, first.p + n_corners - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        const uint64_t nv = (uint64_t)last_v + last_f;
        // ---- vertices
        SF_CUDA(cudaMalloc(&mesh->vert, nv * 3 * sizeof(float)));
        SF_CUDA(cudaMalloc(&mesh->nrm, nv * 3 * sizeof(float)));
        DevBuf<uint8_t> pending(nv, s);
        k_mc_vertices<<<148 * 8, 256, 0, s>>>(P, v->d_table, v->d_payload, v->d_occ, v->d_aux, blocks, n_corners,
                                              first.p, vnum.p, corner_slot.p, corner_cube.p, tri_off.p, slot_vidx.p,
                                              mesh->vert, mesh->nrm, pending.p);
        SF_LAUNCH_CHECK();
        // ---- triangles
        DevBuf<uint32_t> keep(total, s), out_pos(total, s);
        DevBuf<uint3> tri_v(total, s);
        k_mc_keep<<<148 * 8, 256, 0, s>>>(total, corner_slot.p, slot_vidx.p, mesh->vert, keep.p, tri_v.p);
        SF_LAUNCH_CHECK();
        exclusive_sum(keep.p, out_pos.p, total, s);
        uint32_t last_o = 0, last_k = 0;
        SF_CUDA(cudaMemcpyAsync(&last_o, out_pos.p + total - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaMemcpyAsync(&last_k, keep.p + total - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        SF_CUDA(cudaStreamSynchronize(s));
        const uint64_t nt = (uint64_t)last_o + last_k;
        SF_CUDA(cudaMalloc(&mesh->tris, std::max<uint64_t>(nt, 1) * 3 * sizeof(uint32_t)));
        k_mc_emit<<<148 * 8, 256, 0, s>>>(total, keep.p, out_pos.p, tri_v.p, reinterpret_cast<uint3*>(mesh->tris));
        SF_LAUNCH_CHECK();
        // ---- face-normal fallback for vertices without a gradient normal
        if (nt) {
            const uint64_t nrec = 3 * nt;
            DevBuf<unsigned long long> rec(nrec, s), rec_sorted(nrec, s);
            k_mc_pending_records<<<148 * 8, 256, 0, s>>>(nt, reinterpret_cast<const uint3*>(mesh->tris), pending.p,
                                                         rec.p);
            SF_LAUNCH_CHECK();
            size_t tb = 0;
            SF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, rec.p, rec_sorted.p, (int64_t)nrec, 0, 64, s));
            DevBuf<char> tmp(tb, s);
            SF_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tb, rec.p, rec_sorted.p, (int64_t)nrec, 0, 64, s));
            k_mc_pending_normals<<<148 * 8, 256, 0, s>>>(nrec, rec_sorted.p,
                                                         reinterpret_cast<const uint3*>(mesh->tris), mesh->vert,
                                                         mesh->nrm);
            SF_LAUNCH_CHECK();
        }
        SF_CUDA(cudaStreamSynchronize(s));
        mesh->nv = nv;
        mesh->nt = nt;
        *out = mesh.release();
        return SF_OK;
    });
}

int sf_mesh_counts(sf_mesh_t m, uint64_t* vertices, uint64_t* triangles) {
    return guarded([&]() -> int {
        if (!m) throw Error(SF_INVALID_ARGUMENT, "sf_mesh_counts: null mesh");
        if (vertices) *vertices = m->nv;
        if (triangles) *triangles = m->nt;
        return SF_OK;
    });
}

int sf_mesh_read(sf_mesh_t m, float* vertices_xyz, float* normals_xyz, uint32_t* triangles, int32_t out_on_device,
                 void* stream) {
    return guarded([&]() -> int {
        if (!m) throw Error(SF_INVALID_ARGUMENT, "sf_mesh_read: null mesh");
        SF_CUDA(cudaSetDevice(m->device));
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        const cudaMemcpyKind kind = out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        if (vertices_xyz && m->nv)
            SF_CUDA(cudaMemcpyAsync(vertices_xyz, m->vert, m->nv * 3 * sizeof(float), kind, s));
        if (normals_xyz && m->nv) SF_CUDA(cudaMemcpyAsync(normals_xyz, m->nrm, m->nv * 3 * sizeof(float), kind, s));
        if (triangles && m->nt) SF_CUDA(cudaMemcpyAsync(triangles, m->tris, m->nt * 3 * sizeof(uint32_t), kind, s));
        SF_CUDA(cudaStreamSynchronize(s));
        return SF_OK;
    });
}

int sf_mesh_destroy(sf_mesh_t m) {
    delete m;
    return SF_OK;
}

}  // extern "C"
