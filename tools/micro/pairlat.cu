// SM-pair handoff latency through L2 tagged words, for the ring kernel's neighbour order: every CTA
// (one per SM) ping-pongs with a partner CTA; prints round-trip cycles with both %smid values, for
// several pairings and mailbox offsets.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pairlat.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// partner of CTA c: mode 0: c ^ 1; mode 1: (c + n/2) % n; mode 2: by smid (smid ^ 1, via a table)
__global__ void pairs(unsigned long long* box, int iters, long long* out, int mode, int off, int* smid_of) {
    extern __shared__ int pad[];
    if (threadIdx.x != 0) return;
    const int c = blockIdx.x, n = gridDim.x;
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    pad[0] = smid;
    int partner = mode == 0 ? (c ^ 1) : (c < n / 2 ? c + n / 2 : c - n / 2);
    if (partner >= n) return;
    const int lo = c < partner ? c : partner;
    unsigned long long* mine = box + (size_t)(lo * 64 + (c == lo ? 0 : 32) + off * 8192) ;
    unsigned long long* other = box + (size_t)(lo * 64 + (c == lo ? 32 : 0) + off * 8192);
    __syncwarp();
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (c == lo) {
            st64(other, (unsigned long long)i);
            while (ld64(mine) != (unsigned long long)i) {
            }
        } else {
            while (ld64(mine) != (unsigned long long)i) {
            }
            st64(other, (unsigned long long)i);
        }
    }
    long long t1 = clock64();
    out[c * 3 + 0] = (t1 - t0) / iters;
    out[c * 3 + 1] = smid;
    out[c * 3 + 2] = partner;
}

// address sweep: only CTAs a and a^1 play; mailbox at byte offset `boff`
__global__ void sweep(unsigned long long* box, int iters, long long* out, int a, long long boff) {
    extern __shared__ int pad[];
    if (threadIdx.x != 0) return;
    const int c = blockIdx.x;
    if ((c | 1) != (a | 1)) return;
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    pad[0] = smid;
    const bool lo = (c & 1) == 0;
    unsigned long long* base = box + boff / 8;
    unsigned long long* mine = base + (lo ? 0 : 8);
    unsigned long long* other = base + (lo ? 8 : 0);
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (lo) {
            st64(other, (unsigned long long)i);
            while (ld64(mine) != (unsigned long long)i) {
            }
        } else {
            while (ld64(mine) != (unsigned long long)i) {
            }
            st64(other, (unsigned long long)i);
        }
    }
    long long t1 = clock64();
    if (lo) {
        out[0] = (t1 - t0) / iters;
        out[1] = smid;
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* box;
    long long* out;
    cudaMalloc(&box, 256 << 20);
    cudaMallocManaged(&out, sizeof(long long) * 3 * nsm);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(pairs, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 2; ++mode) {
        for (int off = 0; off < 3; ++off) {
            cudaMemset(box, 0, 256 << 20);
            int iters = 2000, offv = off * 97;
            int* nul = nullptr;
            void* args[] = {&box, &iters, &out, &mode, &offv, &nul};
            cudaError_t e = cudaLaunchCooperativeKernel((const void*)pairs, dim3(nsm), dim3(32), args, smem, 0);
            if (e != cudaSuccess) { printf("launch: %s\n", cudaGetErrorString(e)); return 1; }
            cudaDeviceSynchronize();
            long long mn = 1 << 30, mx = 0, sum = 0;
            for (int c = 0; c < nsm; ++c) {
                long long v = out[c * 3];
                mn = v < mn ? v : mn;
                mx = v > mx ? v : mx;
                sum += v;
            }
            printf("mode %d (%s) off %d: round trip cycles min %lld mean %lld max %lld\n", mode,
                   mode == 0 ? "c^1" : "c+n/2", off, mn, sum / nsm, mx);
            if (off == 0) {
                printf("  c:smid:partner:cycles");
                for (int c = 0; c < nsm; c += 1) printf(" %d:%lld:%lld:%lld", c, out[c * 3 + 1], out[c * 3 + 2], out[c * 3]);
                printf("\n");
            }
        }
    }
    cudaFuncSetAttribute(sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int a : {0, 8, 16, 100}) {
        printf("sweep pair %d/%d:", a, a + 1);
        for (long long boff = 0; boff < 32768; boff += 128) {
            cudaMemset(box, 0, 1 << 20);
            int iters = 300;
            void* args[] = {&box, &iters, &out, &a, &boff};
            cudaLaunchCooperativeKernel((const void*)sweep, dim3(nsm), dim3(32), args, smem, 0);
            cudaDeviceSynchronize();
            if (boff == 0) printf(" smid %lld |", out[1]);
            printf(" %lld", out[0]);
        }
        printf("\n");
    }
    return 0;
}
