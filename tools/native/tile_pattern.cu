// tile_pattern.cu — what the fused tile pass's ACCESS PATTERN alone costs: a
// read-modify-write of the whole state in tiles of 2^11 amplitudes whose
// qubit set is {0..lowc-1} + hi qubits (2^lowc-amplitude contiguous segments),
// with no shared memory, no op loop and no barriers. One CTA of 128 threads
// per tile, E amplitudes per thread loaded first, then scaled and stored.
// Prints GB/s per pattern; compare with the same kernel on contiguous tiles.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/native/tile_pattern.cu -o /tmp/tile_pattern && /tmp/tile_pattern [n=30]
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

struct Geom {
    int n, k, lowc, nhi;
    int hiq[16];
};

__device__ __forceinline__ uint64_t ins0(uint64_t x, int p) {
    const uint64_t lo = x & ((1ull << p) - 1);
    return ((x >> p) << (p + 1)) | lo;
}

template <int E, int MINB>
__global__ void __launch_bounds__(128, MINB) k_pattern(double2 *psi, const __grid_constant__ Geom g, int persistent) {
    const uint64_t ntiles = 1ull << (g.n - g.k);
    const uint32_t lowm = (1u << g.lowc) - 1u;
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint64_t base = tile << g.lowc;
        for (int i = 0; i < g.nhi; ++i) base = ins0(base, g.hiq[i]);
        for (int part = 0; part < (1 << g.k) / (128 * E); ++part) {
            double2 v[E];
            uint64_t idx[E];
#pragma unroll
            for (int j = 0; j < E; ++j) {
                const uint32_t l = threadIdx.x + 128u * (uint32_t)(j + part * E);
                uint64_t off = l & lowm;
                const uint32_t h = l >> g.lowc;
                for (int i = 0; i < g.nhi; ++i)
                    if ((h >> i) & 1u) off |= 1ull << g.hiq[i];
                idx[j] = base | off;
            }
#pragma unroll
            for (int j = 0; j < E; ++j) v[j] = psi[idx[j]];
#pragma unroll
            for (int j = 0; j < E; ++j) {
                v[j].x *= 0.999;
                v[j].y *= 1.001;
                psi[idx[j]] = v[j];
            }
        }
        if (!persistent) break;
    }
}

template <int E, int MINB>
float run(double2 *psi, const Geom &g, int persistent, int sms) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pattern<E, MINB>, 128, 0);
    const uint64_t ntiles = 1ull << (g.n - g.k);
    const unsigned grid = persistent ? (unsigned)(per_sm * sms) : (unsigned)ntiles;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e9f;
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        k_pattern<E, MINB><<<grid, 128>>>(psi, g, persistent);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep && ms < best) best = ms;
    }
    return best;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 30;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double2 *psi;
    cudaMalloc(&psi, sizeof(double2) << n);
    cudaMemset(psi, 0, sizeof(double2) << n);
    struct Pat { const char *name; int lowc; std::vector<int> hiq; };
    std::vector<Pat> pats = {
        {"contiguous (lowc 11)", 11, {}},
        {"lowc 8 + 27 28 29", 8, {27, 28, 29}},
        {"lowc 6 + 16..20", 6, {16, 17, 18, 19, 20}},
        {"lowc 5 + 24..29", 5, {24, 25, 26, 27, 28, 29}},
        {"lowc 4 + 12 13 14 26..29", 4, {12, 13, 14, 26, 27, 28, 29}},
        {"lowc 3 + 11..18", 3, {11, 12, 13, 14, 15, 16, 17, 18}},
        {"lowc 3 + 19..26", 3, {19, 20, 21, 22, 23, 24, 25, 26}},
        {"lowc 3 + 6..10 21 22 23", 3, {6, 7, 8, 9, 10, 21, 22, 23}},
        {"lowc 3 + 22..29", 3, {22, 23, 24, 25, 26, 27, 28, 29}},
        {"lowc 2 + 11..19", 2, {11, 12, 13, 14, 15, 16, 17, 18, 19}},
    };
    const double bytes = 2.0 * 16.0 * (double)(1ull << n);
    for (const Pat &p : pats) {
        Geom g{};
        g.n = n; g.k = 11; g.lowc = p.lowc; g.nhi = (int)p.hiq.size();
        for (int i = 0; i < g.nhi; ++i) g.hiq[i] = p.hiq[i];
        for (int i = 0; i < g.nhi; ++i) if (g.hiq[i] >= n) g.hiq[i] -= (30 - n);
        const float a = run<16, 5>(psi, g, 0, sms), b = run<16, 5>(psi, g, 1, sms);
        const float c = run<8, 8>(psi, g, 0, sms), d = run<4, 12>(psi, g, 0, sms);
        printf("{\"pattern\": \"%s\", \"E16_minb5_per_tile_gbs\": %.0f, \"E16_minb5_persistent_gbs\": %.0f, "
               "\"E8_minb8_per_tile_gbs\": %.0f, \"E4_minb12_per_tile_gbs\": %.0f}\n",
               p.name, bytes / a / 1e6, bytes / b / 1e6, bytes / c / 1e6, bytes / d / 1e6);
    }
    return 0;
}
