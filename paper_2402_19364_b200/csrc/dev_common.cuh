// dev_common.cuh -- device helpers shared by the sm_100a kernels (kernels.cu, seg_kernel.cu):
// per-lane row fragments, 16-byte loads/stores, vector L2 reductions, launch-shape helpers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <initializer_list>

namespace arrow {
namespace dev {

template <typename T, int VEC> struct VecT;
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<double, 2> { using type = double2; };
template <> struct VecT<double, 1> { using type = double; };

// VEC consecutive elements of one row held by one lane
template <typename T, int VEC> struct Frag {
    T v[VEC];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < VEC; ++i) v[i] = T(0);
    }
};

template <typename T, int VEC>
__device__ __forceinline__ Frag<T, VEC> ld_x(const T *p) {  // read-only (L1-allocating) path
    using V = typename VecT<T, VEC>::type;
    V r = __ldg(reinterpret_cast<const V *>(p));
    Frag<T, VEC> f;
    static_assert(sizeof(V) == sizeof(f), "frag size");
    memcpy(&f, &r, sizeof(V));
    return f;
}

template <typename T, int VEC>
__device__ __forceinline__ Frag<T, VEC> ld_plain(const T *p) {
    using V = typename VecT<T, VEC>::type;
    V r = *reinterpret_cast<const V *>(p);
    Frag<T, VEC> f;
    memcpy(&f, &r, sizeof(V));
    return f;
}

template <typename T, int VEC>
__device__ __forceinline__ void st_stream(T *p, const Frag<T, VEC> &f) {  // evict-first: Y is write-once
    using V = typename VecT<T, VEC>::type;
    V r;
    memcpy(&r, &f, sizeof(V));
    __stcs(reinterpret_cast<V *>(p), r);
}

template <typename T, int VEC>
__device__ __forceinline__ void st_plain(T *p, const Frag<T, VEC> &f) {
    using V = typename VecT<T, VEC>::type;
    V r;
    memcpy(&r, &f, sizeof(V));
    *reinterpret_cast<V *>(p) = r;
}

// fire-and-forget L2 reduction (red.global.add.v4.f32 for a 16-byte fp32 fragment)
template <typename T, int VEC>
__device__ __forceinline__ void atomic_add_frag(T *p, const Frag<T, VEC> &f) {
    if constexpr (sizeof(T) == 4 && VEC == 4) {
        atomicAdd(reinterpret_cast<float4 *>(p), make_float4(f.v[0], f.v[1], f.v[2], f.v[3]));
    } else if constexpr (sizeof(T) == 4 && VEC == 2) {
        atomicAdd(reinterpret_cast<float2 *>(p), make_float2(f.v[0], f.v[1]));
    } else {
#pragma unroll
        for (int i = 0; i < VEC; ++i) atomicAdd(p + i, f.v[i]);
    }
}

}  // namespace dev

// widest vector (16 bytes at most) that divides k and every pointer's alignment
inline int pick_vec(int dtype, int64_t k, std::initializer_list<const void *> ptrs) {
    const int es = dtype == 1 ? 8 : 4;
    int vec = 16 / es;
    while (vec > 1) {
        bool ok = (k % vec) == 0;
        for (const void *p : ptrs) ok = ok && ((reinterpret_cast<uintptr_t>(p) % (vec * es)) == 0);
        if (ok) break;
        vec >>= 1;
    }
    return vec;
}

// lanes per row slab: the smallest power of two covering ceil(k / vec), at most a warp
inline int pick_lpe(int64_t k, int vec) {
    const int64_t need = (k + vec - 1) / vec;
    int lpe = 1;
    while (lpe < 32 && lpe < need) lpe <<= 1;
    return lpe;
}

// grid for an elementwise pass of `total` thread items: 16 blocks of 256 per SM at most
inline unsigned grid_for(int64_t total, int num_sms) {
    int64_t g = (total + 255) / 256;
    if (g > (int64_t)num_sms * 16) g = (int64_t)num_sms * 16;
    if (g < 1) g = 1;
    return (unsigned)g;
}

}  // namespace arrow
