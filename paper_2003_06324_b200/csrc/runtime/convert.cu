// Device element conversion fp32 -> storage type. The f16 path is IEEE RNE,
// which equals anvil::round_to_f16 (proj/include/anvil/matrix.hpp:67-80) for
// |x| < 65504; bf16 is IEEE RNE.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace fireiron::rt {

template <typename T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half cvt<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

template <typename T>
__global__ void convert_kernel(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
    int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * 4;
    for (; i + 3 < n; i += stride) {
        float4 v = *reinterpret_cast<const float4*>(src + i);
        dst[i] = cvt<T>(v.x);
        dst[i + 1] = cvt<T>(v.y);
        dst[i + 2] = cvt<T>(v.z);
        dst[i + 3] = cvt<T>(v.w);
    }
    for (; i < n; ++i) dst[i] = cvt<T>(src[i]);
}

// storage -> fp32 (used to hand results back through the fp32 host boundary)
template <typename T>
__device__ __forceinline__ float widen(T v);
template <>
__device__ __forceinline__ float widen<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float widen<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__global__ void widen_kernel(const T* __restrict__ src, float* __restrict__ dst, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        dst[i] = widen<T>(src[i]);
}

static int grid_for(int64_t n) {
    int64_t blocks = (n / 4 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    return static_cast<int>(blocks);
}

// elem: 0 f32, 1 f16, 2 bf16. src must be 16B aligned for the vector path.
cudaError_t convert_f32(const float* src, void* dst, int64_t n, int elem, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (elem == 0) return cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToDevice, s);
    if ((reinterpret_cast<uintptr_t>(src) & 15) != 0) return cudaErrorMisalignedAddress;
    const int g = grid_for(n);
    switch (elem) {
        case 1: convert_kernel<__half><<<g, 256, 0, s>>>(src, static_cast<__half*>(dst), n); break;
        case 2:
            convert_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(src, static_cast<__nv_bfloat16*>(dst), n);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t widen_to_f32(const void* src, float* dst, int64_t n, int elem, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    int g = grid_for(n * 4);
    switch (elem) {
        case 0: return cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToDevice, s);
        case 1: widen_kernel<__half><<<g, 256, 0, s>>>(static_cast<const __half*>(src), dst, n); break;
        case 2:
            widen_kernel<__nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src), dst, n);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace fireiron::rt
