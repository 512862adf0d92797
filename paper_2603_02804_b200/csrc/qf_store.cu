// Batch-store conversions for StorageMode::MemSave (engine.hpp:30): checkpoint
// slots held as bfloat16 pairs (4 B per complex64 amplitude).
//   narrow: the reference's narrow_to_bf16 bit for bit (statevec.hpp:36-45:
//           round-to-nearest-even, overflow -> inf, NaN quieted)
//   widen:  exact embedding (statevec.hpp:48-53)
// Both are HBM-bound elementwise streams: 16-B loads, one thread per 2 amplitudes.
#include "qf_internal.h"

namespace qfb {
namespace {

__device__ __forceinline__ uint32_t bf16_bits(float v) {
    const uint32_t u = __float_as_uint(v);
    if ((u & 0x7fffffffu) > 0x7f800000u) return (u >> 16) | 0x0040u;
    return (u + 0x7fffu + ((u >> 16) & 1u)) >> 16;
}

__global__ void narrow_kernel(const float4 *__restrict__ src, uint2 *__restrict__ dst, uint64_t n2) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride) {
        const float4 v = src[i]; // two amplitudes (re, im, re, im)
        dst[i] = make_uint2(bf16_bits(v.x) | (bf16_bits(v.y) << 16),
                            bf16_bits(v.z) | (bf16_bits(v.w) << 16));
    }
}

__global__ void widen_kernel(const uint2 *__restrict__ src, float4 *__restrict__ dst, uint64_t n2) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride) {
        const uint2 b = src[i];
        dst[i] = make_float4(__uint_as_float(b.x << 16), __uint_as_float(b.x & 0xffff0000u),
                             __uint_as_float(b.y << 16), __uint_as_float(b.y & 0xffff0000u));
    }
}

int grid_for(uint64_t n2) {
    const uint64_t blocks = (n2 + 255) / 256;
    return int(blocks < 148ull * 16 ? blocks : 148ull * 16);
}

} // namespace

cudaError_t launch_narrow_bf16(cudaStream_t st, const float2 *src, uint32_t *dst, uint64_t amps) {
    const uint64_t n2 = amps / 2; // amps is a multiple of one tile
    if (n2 == 0) return cudaSuccess;
    narrow_kernel<<<grid_for(n2), 256, 0, st>>>(reinterpret_cast<const float4 *>(src),
                                                  reinterpret_cast<uint2 *>(dst), n2);
    return cudaGetLastError();
}

cudaError_t launch_widen_bf16(cudaStream_t st, const uint32_t *src, float2 *dst, uint64_t amps) {
    const uint64_t n2 = amps / 2;
    if (n2 == 0) return cudaSuccess;
    widen_kernel<<<grid_for(n2), 256, 0, st>>>(reinterpret_cast<const uint2 *>(src),
                                                reinterpret_cast<float4 *>(dst), n2);
    return cudaGetLastError();
}

} // namespace qfb
