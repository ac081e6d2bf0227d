// kernel_gen.cuh -- on-device input generators for giga-pixel workloads
// (SURVEY.md 8(f) row f3).
//
// The reference's generators (image.hpp:77-103 SmoothRandom, noise.hpp:62-89
// inject_sp_noise) draw from one sequential mt19937 stream and a partial
// Fisher-Yates shuffle; the latter divides by zero at 2^32 pixels.  These
// generators keep the same *structure* but are counter-based, so every pixel
// is an independent pure function of (seed, image, row, column):
//   smooth:  field(i) = mix64(seed * K + i) & 0xff, then the reference's
//            clamped 3x3 mean with round-half-up, (sum + cnt/2) / cnt;
//   noise:   pixel i is corrupted iff mix64(seed' + i) < density * 2^64
//            (Bernoulli, expected count density * N, not the reference's
//            exact count), salt (255) iff a second draw < salt_ratio, else
//            pepper (0).
// They are NOT bit-equal to the reference generators; parity is against the
// numpy restatement in oracle/oracle.py (dev_smooth, dev_noise).
#pragma once
#include <cstdint>

namespace phg {

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

constexpr uint64_t kGenMul = 0xD1342543DE82EF95ull;

struct GenArgs {
    uint8_t* img;
    int64_t pitch;
    int64_t image_stride;
    int width, rows, n;    // buffer geometry (rows = rows held)
    int row_base, height;  // global row of buffer row 0, global image height
    uint64_t seed;
    uint64_t thresh;       // noise: corrupted iff draw < thresh (2^64 scale, 0 = none)
    uint64_t salt_thresh;  // noise: salt iff second draw < salt_thresh
    bool all;              // density == 1
    bool salt_all;         // salt_ratio == 1
    unsigned long long* count;
};

// element index of (image, global row, col) in the generator's counter space
__device__ __forceinline__ uint64_t gen_index(const GenArgs& a, int img, int gr, int c) {
    return (static_cast<uint64_t>(img) * a.height + gr) * a.width + c;
}

__global__ void __launch_bounds__(256) gen_smooth_kernel(const GenArgs a) {
    const int img = blockIdx.z;
    const uint64_t base = a.seed * kGenMul;
    for (int r = blockIdx.y; r < a.rows; r += gridDim.y)
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.width; c += gridDim.x * blockDim.x) {
        const int gr = a.row_base + r;
        const int r0 = gr > 0 ? gr - 1 : 0, r1 = gr < a.height - 1 ? gr + 1 : a.height - 1;
        const int c0 = c > 0 ? c - 1 : 0, c1 = c < a.width - 1 ? c + 1 : a.width - 1;
        int sum = 0, cnt = 0;
        for (int i = r0; i <= r1; ++i)
            for (int j = c0; j <= c1; ++j) {
                sum += static_cast<int>(mix64(base + gen_index(a, img, i, j)) & 0xffu);
                ++cnt;
            }
        a.img[img * a.image_stride + static_cast<int64_t>(r) * a.pitch + c] =
            static_cast<uint8_t>((sum + cnt / 2) / cnt);
    }
}

__global__ void __launch_bounds__(256) gen_noise_kernel(const GenArgs a) {
    const int img = blockIdx.z;
    const uint64_t base = a.seed * kGenMul;
    unsigned n = 0;
    for (int r = blockIdx.y; r < a.rows; r += gridDim.y)
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < a.width; c += gridDim.x * blockDim.x) {
        const uint64_t u = mix64(base + gen_index(a, img, a.row_base + r, c));
        if (a.all || u < a.thresh) {
            const bool salt = a.salt_all || mix64(u) < a.salt_thresh;
            a.img[img * a.image_stride + static_cast<int64_t>(r) * a.pitch + c] = salt ? 255 : 0;
            ++n;
        }
    }
    n = __reduce_add_sync(0xffffffffu, n);
    if ((threadIdx.x & 31) == 0 && n && a.count) atomicAdd(a.count, static_cast<unsigned long long>(n));
}

}  // namespace phg
