// Device twin of the seeded input recipe in lift_inputs/__init__.py.
// Holds none of the method's arithmetic; it only fills buffers for tests/bench.
#include <cstdint>
#include <cuda_runtime.h>

namespace {
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t ID_MUL = 0xD1B54A32D192ED03ULL;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
    z += GOLDEN;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

__global__ void fill_kernel(float* __restrict__ out, int64_t n, uint64_t base, int dist,
                            double lo, double span) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        uint64_t r = mix(base + (uint64_t)i);
        float v;
        if (dist == 0) {
            double u = (double)(r >> 40) * 0x1p-24;
            v = (float)__dadd_rn(lo, __dmul_rn(span, u));
        } else {
            v = (float)((int64_t)((r >> 32) % 17u) - 8);
        }
        out[i] = v;
    }
}
}  // namespace

extern "C" int lift_inputs_fill_device(float* out, int64_t n, uint64_t seed, uint64_t tid,
                                       int64_t i0, int dist, double lo, double hi,
                                       cudaStream_t stream) {
    if (n < 0 || (n > 0 && !out) || (dist != 0 && dist != 1)) return 1;
    if (n == 0) return 0;
    const uint64_t base = seed * GOLDEN + tid * ID_MUL + (uint64_t)i0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sms * 16) blocks = (int64_t)sms * 16;
    fill_kernel<<<(unsigned)blocks, 256, 0, stream>>>(out, n, base, dist, lo, hi - lo);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
