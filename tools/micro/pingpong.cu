// Ping-pong latency between two CTAs through L2 (tagged 64-bit words), for the ring kernel's
// mailbox protocol.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 pingpong.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ unsigned long long ld64(const unsigned long long* p) {
    unsigned long long v;
    if (MODE == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (MODE == 1) asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (MODE == 2) asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
template <int MODE>
__device__ __forceinline__ void st64(unsigned long long* p, unsigned long long v) {
    if (MODE == 0 || MODE == 2) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else if (MODE == 1) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE>
__global__ void pingpong(unsigned long long* box, int iters, long long* out, int stride) {
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x == 0 ? 0 : 1;
    if (blockIdx.x > 1) return;
    unsigned long long* mine = box + me * stride;
    unsigned long long* other = box + (1 - me) * stride;
    long long t0 = clock64();
    for (int i = 1; i <= iters; ++i) {
        if (me == 0) {
            st64<MODE>(other, (unsigned long long)i);
            while (ld64<MODE>(mine) != (unsigned long long)i) {
            }
        } else {
            while (ld64<MODE>(mine) != (unsigned long long)i) {
            }
            st64<MODE>(other, (unsigned long long)i);
        }
    }
    long long t1 = clock64();
    if (me == 0) {
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        out[0] = (t1 - t0) / iters;
        out[1] = smid;
    } else {
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        out[2] = smid;
    }
}

int main() {
    unsigned long long* box;
    long long* out;
    cudaMalloc(&box, 1 << 20);
    cudaMallocManaged(&out, 64);
    const char* names[] = {"relaxed.gpu", "volatile", "cg/relaxed", "acquire/release"};
    for (int stride : {16, 256, 4096}) {
        for (int mode = 0; mode < 4; ++mode) {
            for (int grid : {2, 148}) {
                cudaMemset(box, 0, 1 << 20);
                void (*k)(unsigned long long*, int, long long*, int) =
                    mode == 0 ? pingpong<0> : mode == 1 ? pingpong<1> : mode == 2 ? pingpong<2> : pingpong<3>;
                k<<<grid, 32>>>(box, 2000, out, stride);
                cudaDeviceSynchronize();
                printf("%-16s stride %5d grid %3d: round trip %lld cycles (sm %lld <-> %lld)\n", names[mode], stride,
                       grid, out[0], out[1], out[2]);
            }
        }
    }
    return 0;
}
