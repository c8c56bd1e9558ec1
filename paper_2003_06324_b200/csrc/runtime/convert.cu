// Device element conversion fp32 -> storage type. The f16 path is IEEE RNE
// with the reference's saturation above 2^16, which equals anvil::round_to_f16
// (proj/include/anvil/matrix.hpp:67-80) except on [65520, 65536), where the
// reference yields 65536 (not an f16 value) and this gives inf; bf16 is IEEE RNE.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace fireiron::rt {

template <typename T>
__device__ __forceinline__ T cvt(float v);
template <>
__device__ __forceinline__ float cvt<float>(float v) { return v; }
// round_to_f16 (matrix.hpp:76) saturates finite |x| >= 2^16 to +-65504 where
// IEEE RNE gives +-inf; infinities and NaN pass through (matrix.hpp:68)
template <>
__device__ __forceinline__ __half cvt<__half>(float v) {
    const float a = fabsf(v);
    return __float2half_rn(a >= 65536.0f && a <= 3.40282347e38f ? copysignf(65504.0f, v) : v);
}
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

// Pitched regions (width contiguous elements x height lines, `pitch` elements
// apart; source and destination share the pitch): the blocked host pipeline
// converts each operand panel and widens each C block where it lands.
template <typename T, bool kVec>
__global__ void convert_2d_kernel(const float* __restrict__ src, T* __restrict__ dst, int64_t width, int64_t height,
                                  int64_t pitch) {
    constexpr int V = kVec ? 4 : 1;
    const int64_t per_line = width / V;
    const int64_t n = per_line * height;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t y = i / per_line, x = (i - y * per_line) * V;
        const int64_t o = y * pitch + x;
        if constexpr (kVec) {
            const float4 v = *reinterpret_cast<const float4*>(src + o);
            dst[o] = cvt<T>(v.x);
            dst[o + 1] = cvt<T>(v.y);
            dst[o + 2] = cvt<T>(v.z);
            dst[o + 3] = cvt<T>(v.w);
        } else {
            dst[o] = cvt<T>(src[o]);
        }
    }
}

template <typename T>
__global__ void widen_2d_kernel(const T* __restrict__ src, float* __restrict__ dst, int64_t width, int64_t height,
                                int64_t pitch) {
    const int64_t n = width * height;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t y = i / width, o = y * pitch + (i - y * width);
        dst[o] = widen<T>(src[o]);
    }
}

cudaError_t convert_f32_2d(const float* src, void* dst, int64_t width, int64_t height, int64_t pitch, int elem,
                           cudaStream_t s) {
    if (width <= 0 || height <= 0) return cudaSuccess;
    if (elem == 0)
        return cudaMemcpy2DAsync(dst, pitch * 4, src, pitch * 4, width * 4, height, cudaMemcpyDeviceToDevice, s);
    const bool vec = width % 4 == 0 && pitch % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    const int g = grid_for(width * height);
    switch (elem * 2 + (vec ? 1 : 0)) {
        case 2: convert_2d_kernel<__half, false><<<g, 256, 0, s>>>(src, static_cast<__half*>(dst), width, height, pitch); break;
        case 3: convert_2d_kernel<__half, true><<<g, 256, 0, s>>>(src, static_cast<__half*>(dst), width, height, pitch); break;
        case 4:
            convert_2d_kernel<__nv_bfloat16, false>
                <<<g, 256, 0, s>>>(src, static_cast<__nv_bfloat16*>(dst), width, height, pitch);
            break;
        case 5:
            convert_2d_kernel<__nv_bfloat16, true>
                <<<g, 256, 0, s>>>(src, static_cast<__nv_bfloat16*>(dst), width, height, pitch);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t widen_to_f32_2d(const void* src, float* dst, int64_t width, int64_t height, int64_t pitch, int elem,
                            cudaStream_t s) {
    if (width <= 0 || height <= 0) return cudaSuccess;
    const int g = grid_for(width * height * 4);
    switch (elem) {
        case 0: return cudaMemcpy2DAsync(dst, pitch * 4, src, pitch * 4, width * 4, height, cudaMemcpyDeviceToDevice, s);
        case 1: widen_2d_kernel<__half><<<g, 256, 0, s>>>(static_cast<const __half*>(src), dst, width, height, pitch); break;
        case 2:
            widen_2d_kernel<__nv_bfloat16>
                <<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src), dst, width, height, pitch);
            break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace fireiron::rt
