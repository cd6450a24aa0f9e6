// Cost of fence.release.cluster (MEMBAR.ALL.GPU) right after remote DSMEM
// stores vs. after they have had time to complete.  Cluster of 2 CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mapa(uint32_t a, unsigned r) {
    uint32_t d; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r)); return d;
}
__global__ void __cluster_dims__(2, 1, 1) k(long long *out, int delay) {
    __shared__ double buf[256];
    unsigned rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank == 0 && threadIdx.x < 32) {
        const uint32_t ra = mapa((uint32_t)__cvta_generic_to_shared(&buf[threadIdx.x]), 1);
        long long acc0 = 0, acc1 = 0, acc2 = 0;
        for (int it = 0; it < 64; ++it) {
            // (a) 7 remote stores then fence immediately
            long long t0 = clock64();
            for (int d = 0; d < 7; ++d) asm volatile("st.shared::cluster.f64 [%0], %1;" :: "r"(ra + 8 * 32 * d), "d"(1.0 * it) : "memory");
            asm volatile("fence.release.cluster;" ::: "memory");
            long long t1 = clock64();
            acc0 += t1 - t0;
            // (b) remote stores, wait `delay` cycles, then fence
            for (int d = 0; d < 7; ++d) asm volatile("st.shared::cluster.f64 [%0], %1;" :: "r"(ra + 8 * 32 * d), "d"(2.0 * it) : "memory");
            long long tw = clock64(); while (clock64() - tw < delay) {}
            long long t2 = clock64();
            asm volatile("fence.release.cluster;" ::: "memory");
            long long t3 = clock64();
            acc1 += t3 - t2;
            // (c) fence with nothing outstanding
            long long t4 = clock64();
            asm volatile("fence.release.cluster;" ::: "memory");
            long long t5 = clock64();
            acc2 += t5 - t4;
        }
        if (threadIdx.x == 0) { out[0] = acc0 / 64; out[1] = acc1 / 64; out[2] = acc2 / 64; }
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
int main() {
    long long *d, h[3];
    cudaMalloc(&d, 3 * sizeof(long long));
    for (int delay : {0, 500, 2000, 5000}) {
        k<<<2, 64>>>(d, delay);
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("delay %5d: stores+fence %lld cyc, fence after delay %lld cyc, idle fence %lld cyc\n", delay, h[0], h[1], h[2]);
    }
    return 0;
}
