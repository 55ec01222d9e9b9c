// kernels_svf.cu — stationary-velocity-field (SVF) mode: exp_map and its
// discrete adjoint svf_pullback (diffeo.cpp:66-167).
//
// exp_map is M self-compositions of v/2^M (k_compose of kernels_point.cu).
// svf_pullback pushes a cotangent w back through the M squarings.  Per level
// k (reverse order) the reference computes
//   wn = w + J(u_k)(x + u_k(x))^T w          voxel-parallel
//   wn[node] += wt * w[i]                    serial scatter, voxel order
// where the scatter spreads w at voxel i onto the 8 corners of the cell its
// sample x_i + u_k(x_i) fell in.  A float-atomic scatter would make the result
// depend on thread timing; here the scatter is a deterministic GATHER instead:
//   1. k_svf_jt writes, per voxel, the pair (cell base node, voxel) and the
//      lerp weights of its 8 corners;
//   2. a stable radix sort by base (CUB) keeps each base's voxels in
//      increasing order (n pairs, not 8n: the corners are base + fixed offsets);
//   3. k_svf_offsets turns the sorted keys into per-base segment starts;
//   4. k_svf_gather, for node q, merges the segments of the 8 bases q - off_k
//      by voxel index (ties: corner order) — the reference's serial order —
//      and accumulates.
// Results are bit-stable run to run and the per-node summation order is the
// reference's own.
#include <cmath>
#include <cstdint>

#include <cub/device/device_radix_sort.cuh>

#include "dfm_device.cuh"
#include "dfm_kernels.cuh"

namespace dfm {

namespace {

constexpr int kNS = 256;

inline unsigned grid_n(int64_t n) { return static_cast<unsigned>((n + kNS - 1) / kNS); }

__device__ __forceinline__ void voxel_of(const Dims& d, int64_t i, int& x, int& y, int& z) {
    x = static_cast<int>(i % d.nx);
    const int64_t r = i / d.nx;
    y = static_cast<int>(r % d.ny);
    z = static_cast<int>(r / d.ny);
}

template <class T>
__global__ void k_scale3(const T* __restrict__ in, T* __restrict__ out, int64_t n3, T s,
                         const LoopState* st) {
    if (st && st->done) return;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kNS) + threadIdx.x;
    if (i < n3) out[i] = in[i] * s;
}

// the lerp weight of corner k of voxel i's cell (diffeo.cpp:140-156 order)
template <class T>
__device__ __forceinline__ T corner_wt(const Cell3<T>& c, int k) {
    const int cx = k & 1, cy = (k >> 1) & 1, cz = k >> 2;
    return (cx ? c.fx : T(1) - c.fx) * (cy ? c.fy : T(1) - c.fy) *
           (c.three ? (cz ? c.fz : T(1) - c.fz) : T(1));
}

// terms (a)+(b) of one level: wn = w + J^T w; and the (node, 8i+corner) pairs
template <class T>
__global__ void k_svf_jt(const T* __restrict__ uk, const T* __restrict__ w, Dims d,
                         T* __restrict__ wn, int32_t* __restrict__ keys,
                         int32_t* __restrict__ vals, T* __restrict__ wts, const LoopState* st) {
    if (st && st->done) return;
    const int64_t i = blockIdx.x * static_cast<int64_t>(kNS) + threadIdx.x;
    if (i >= d.n) return;
    int x, y, z;
    voxel_of(d, i, x, y, z);
    const int64_t n = d.n;
    const bool three = d.ndim == 3;
    const Cell3<T> c = locate3<T>(d, x, y, z, uk[i], uk[n + i], three ? uk[2 * n + i] : T(0));
    // J[comp][a] = d u_k[comp] / d x_a at the sample (interp.cpp:205-227)
    T J[3][3];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
        if (comp < d.ndim) {
            const Corners<T> k = fetch_corners<T, T, false>(uk + comp * n, c);
            lerp_grad(c, k, d.ndim, J[comp]);
        } else {
            J[comp][0] = J[comp][1] = J[comp][2] = T(0);
        }
    }
    const T wi[3] = {w[i], w[n + i], three ? w[2 * n + i] : T(0)};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (a >= d.ndim) {
            wn[a * n + i] = T(0);
            continue;
        }
        T acc = T(0);
#pragma unroll
        for (int comp = 0; comp < 3; ++comp)
            if (comp < d.ndim) acc += J[comp][a] * wi[comp];
        wn[a * n + i] = wi[a] + acc;
    }
    const int ncorner = three ? 8 : 4;
    // (cell base, voxel) for the sort; the corners' lerp weights for the gather
    keys[i] = static_cast<int32_t>(c.base);
    vals[i] = static_cast<int32_t>(i);
#pragma unroll
    for (int k = 0; k < 8; ++k) wts[8 * i + k] = k < ncorner ? corner_wt(c, k) : T(0);
}

// segment start of every node q in [0, n]: start[q] = first j with key[j] >= q
__global__ void k_svf_offsets(const int32_t* __restrict__ keys, int64_t m, int32_t n,
                              int32_t* __restrict__ start, const LoopState* st) {
    if (st && st->done) return;
    const int64_t j = blockIdx.x * static_cast<int64_t>(kNS) + threadIdx.x;
    if (j >= m) return;
    const int32_t key = keys[j];
    const int32_t prev = j == 0 ? -1 : keys[j - 1];
    for (int32_t q = prev + 1; q <= key && q <= n; ++q) start[q] = static_cast<int32_t>(j);
    // nodes past the last key keep the value k_svf_fill set (m): the tail after
    // the last cell base spans a whole plane, too long for one thread
}

__global__ void k_svf_fill(int32_t* __restrict__ start, int64_t count, int32_t v,
                           const LoopState* st) {
    if (st && st->done) return;
    const int64_t q = blockIdx.x * static_cast<int64_t>(kNS) + threadIdx.x;
    if (q < count) start[q] = v;
}

// term (c) as a gather: node q adds wt * w[i] of its contributors in voxel
// order.  Voxel i contributes to q through corner k when its cell base is
// q - off_k; the voxels of each base are consecutive in the sorted pairs, in
// increasing order, so node q merges the (usually one-element) segments of its
// 8 candidate bases by voxel index, ties in corner order (flat axes make
// corners coincide) — exactly the order of the serial scatter.
template <class T>
__global__ void k_svf_gather(const T* __restrict__ w, Dims d, const int32_t* __restrict__ vals,
                             const T* __restrict__ wts, const int32_t* __restrict__ start,
                             T* __restrict__ wn, const LoopState* st) {
    if (st && st->done) return;
    const int64_t q = blockIdx.x * static_cast<int64_t>(kNS) + threadIdx.x;
    if (q >= d.n) return;
    const int64_t n = d.n;
    const bool three = d.ndim == 3;
    const int sx = d.nx > 1 ? 1 : 0, sy = d.ny > 1 ? d.nx : 0;
    const int sz = three ? d.nx * d.ny : 0;
    const int ncorner = three ? 8 : 4;
    int lo[8], hi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int cx = k & 1, cy = (k >> 1) & 1, cz = k >> 2;
        const int64_t b = q - (cx * sx + cy * sy + cz * sz);
        lo[k] = hi[k] = 0;
        if (k < ncorner && b >= 0) {
            lo[k] = start[b];
            hi[k] = start[b + 1];
        }
    }
    T acc[3] = {wn[q], wn[n + q], three ? wn[2 * n + q] : T(0)};
    for (;;) {
        int bk = -1;
        int32_t best = 0x7fffffff;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (lo[k] < hi[k]) {
                const int32_t vi = vals[lo[k]];
                if (vi < best) {  // strict: ties keep the lower corner
                    best = vi;
                    bk = k;
                }
            }
        if (bk < 0) break;
#pragma unroll
        for (int k = 0; k < 8; ++k) lo[k] += (k == bk);
        const int64_t i = best;
        const T wt = wts[8 * i + bk];
        if (wt == T(0)) continue;  // diffeo.cpp:147-148
        acc[0] += wt * w[i];
        acc[1] += wt * w[n + i];
        if (three) acc[2] += wt * w[2 * n + i];
    }
    wn[q] = acc[0];
    wn[n + q] = acc[1];
    if (three) wn[2 * n + q] = acc[2];
}

int key_bits(int64_t n) {
    int b = 1;
    while ((int64_t(1) << b) <= n) ++b;
    return b;
}

}  // namespace

size_t svf_sort_temp_bytes(int64_t n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr),
                                    static_cast<const int32_t*>(nullptr),
                                    static_cast<int32_t*>(nullptr), static_cast<int>(n), 0,
                                    key_bits(n));
    return bytes;
}

template <class T>
void launch_exp_map(const Launch& L, const T* v, Dims d, int M, T* levels, const LoopState* st) {
    const int64_t n3 = 3 * d.n;
    const T s = static_cast<T>(std::ldexp(1.0, -M));
    k_scale3<T><<<grid_n(n3), kNS, 0, L.stream>>>(v, levels, n3, s, st);
    L.bump();
    // self-composition u <- u + u(x + u); 3-D grids without flat axes take the
    // loop's pointwise compose (one clamped cell search, 24 gathers, fma form)
    const bool fast3 = d.ndim == 3 && d.nx > 1 && d.ny > 1 && d.nz > 1 && d.zoff == 0 &&
                       d.gnz == 0;
    for (int k = 0; k < M; ++k) {
        const T* a = levels + k * n3;
        T* b = levels + (k + 1) * n3;
        if (fast3)
            launch_compose_pointwise<T>(L, a, a, 1e30, d, b, nullptr);
        else
            launch_compose<T>(L, CPlanes3<T>{{a, a + d.n, a + 2 * d.n}},
                              CPlanes3<T>{{a, a + d.n, a + 2 * d.n}}, d,
                              Planes3<T>{{b, b + d.n, b + 2 * d.n}});
    }
}

template <class T>
void launch_svf_pullback(const Launch& L, const T* levels, Dims d, int M, const T* grad_phi,
                         T* out, const SvfWork<T>& ws, const LoopState* st) {
    const int64_t n = d.n, n3 = 3 * n, m = n;  // one (base, voxel) pair per voxel
    const T* w = grad_phi;
    T* bufs[2] = {ws.wa, ws.wb};
    for (int k = M - 1; k >= 0; --k) {
        const T* uk = levels + k * n3;
        T* wn = bufs[k & 1];
        k_svf_jt<T><<<grid_n(n), kNS, 0, L.stream>>>(uk, w, d, wn, ws.keys[0], ws.vals[0], ws.wts,
                                                    st);
        L.bump();
        size_t tb = ws.temp_bytes;
        cub::DeviceRadixSort::SortPairs(ws.temp, tb, ws.keys[0], ws.keys[1], ws.vals[0],
                                        ws.vals[1], static_cast<int>(m), 0, key_bits(n),
                                        L.stream);  // library kernels: not counted
        k_svf_fill<<<grid_n(n + 1), kNS, 0, L.stream>>>(ws.start, n + 1,
                                                        static_cast<int32_t>(m), st);
        L.bump();
        k_svf_offsets<<<grid_n(m), kNS, 0, L.stream>>>(ws.keys[1], m, static_cast<int32_t>(n),
                                                       ws.start, st);
        L.bump();
        k_svf_gather<T><<<grid_n(n), kNS, 0, L.stream>>>(w, d, ws.vals[1], ws.wts, ws.start, wn,
                                                        st);
        L.bump();
        w = wn;
    }
    const T s = static_cast<T>(std::ldexp(1.0, -M));
    k_scale3<T><<<grid_n(n3), kNS, 0, L.stream>>>(w, out, n3, s, st);
    L.bump();
}

#define DFM_INST_SVF(T)                                                                       \
    template void launch_exp_map<T>(const Launch&, const T*, Dims, int, T*, const LoopState*); \
    template void launch_svf_pullback<T>(const Launch&, const T*, Dims, int, const T*, T*,    \
                                         const SvfWork<T>&, const LoopState*);

DFM_INST_SVF(float)
DFM_INST_SVF(double)

}  // namespace dfm
