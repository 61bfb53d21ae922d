// Microbenchmark (diagnostics): cycles of one K1 sweep-phase scan over a
// 64x64 block in shared memory (g > 0 everywhere, h = HINF except a few
// nodes), one CTA of 256 threads alone on the GPU, in variants:
//   0: rolled scan, loads a step ahead (the current K1)
//   1: unroll-2 scan with a `continue` per node (the round-1 K1)
//   2: quad loads (int4 g, uint2 h) fully unrolled ballots
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_scan tools/mb_scan.cu
#include <cstdio>
#include <cstdint>
constexpr int M = 4096, NT = 256, NPT = M / NT;
constexpr uint16_t HINF = 0xFFFF;

__global__ void k(int variant, long long *out, int nact) {
    __shared__ int32_t g[M];
    __shared__ uint16_t h[M];
    __shared__ uint16_t slots[8 * 32];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int v = tid; v < M; v += NT) {
        g[v] = 5;
        h[v] = (v % (M / (nact > 0 ? nact : 1)) == 0 && nact > 0) ? 3 : HINF;
    }
    __syncthreads();
    long long t0 = clock64();
    int acc = 0;
    for (int rep = 0; rep < 10; ++rep) {
        if (variant == 0) {
            int32_t gn = g[tid];
            uint16_t hn = h[tid];
#pragma unroll 1
            for (int i = 0; i < NPT; ++i) {
                const int v = tid + i * NT;
                const int32_t gv = gn;
                const uint16_t hv = hn;
                if (i + 1 < NPT) {
                    gn = g[v + NT];
                    hn = h[v + NT];
                }
                const bool p = gv > 0 && hv != HINF && hv != 0;
                uint32_t word = __ballot_sync(0xFFFFFFFFu, p);
                if (word && lane == 0) acc += __popc(word);
            }
        } else if (variant == 1) {
#pragma unroll 2
            for (int i = 0; i < NPT; ++i) {
                const int v = tid + i * NT;
                const int32_t e = g[v];
                if (e <= 0) continue;
                const uint16_t hv = h[v];
                if (hv == HINF || hv == 0) continue;
                acc += e;
            }
        } else {
#pragma unroll
            for (int j = 0; j < NPT / 4; ++j) {
                const int v0 = 4 * (tid + j * NT);
                const int4 gq = *reinterpret_cast<const int4 *>(g + v0);
                const uint2 hq = *reinterpret_cast<const uint2 *>(h + v0);
                const int gv[4] = {gq.x, gq.y, gq.z, gq.w};
                const uint32_t hv[4] = {hq.x & 0xFFFFu, hq.x >> 16, hq.y & 0xFFFFu, hq.y >> 16};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const bool p = gv[c] > 0 && hv[c] != HINF && hv[c] != 0;
                    uint32_t word = __ballot_sync(0xFFFFFFFFu, p);
                    if (word && lane == 0) acc += __popc(word);
                }
            }
        }
        __syncthreads();
    }
    long long t1 = clock64();
    if (tid == 0) {
        out[0] = (t1 - t0) / 10;
        out[1] = acc;
    }
    (void)slots;
}

int main() {
    long long *d, hbuf[2];
    cudaMalloc(&d, 16);
    for (int nact : {0, 4, 256})
        for (int variant = 0; variant < 3; ++variant) {
            for (int w = 0; w < 3; ++w) k<<<1, NT>>>(variant, d, nact);
            cudaMemcpy(hbuf, d, 16, cudaMemcpyDeviceToHost);
            printf("variant %d active %4d: %lld cycles per scan phase\n", variant, nact, hbuf[0]);
        }
    return 0;
}
