// Layout probe: TMEM written with 32x32b (thread t = lane t, value = lane*1000 + col), then read by a
// warp with 16x32bx2.x4 at lane base 0 and 16, half split offset 64: prints (thread -> lane, col).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tmem16x32bx2 tmem16x32bx2.cu
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out) {
    __shared__ uint32_t base;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = base;
    if (warp < 4) {  // every warp writes its quarter: value = lane_global * 1000 + col
        for (int c = 0; c < 128; ++c) {
            uint32_t v = (uint32_t)((warp * 32 + lane) * 1000 + c);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tm + ((uint32_t)(warp * 32) << 16) + c), "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    __syncthreads();
    if (warp == 1) {  // quarter 1: lanes 32..63
        for (int hb = 0; hb < 2; ++hb) {
            uint32_t r[4];
            const uint32_t a = tm + ((uint32_t)(32 + 16 * hb) << 16) + 0;
            asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 64;" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int i = 0; i < 4; ++i) out[(hb * 32 + lane) * 4 + i] = r[i];
        }
    }
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}
int main() {
    uint32_t* d; cudaMalloc(&d, 64 * 4 * 4);
    k<<<1, 128>>>(d);
    uint32_t h[256]; cudaError_t e = cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(e));
    for (int hb = 0; hb < 2; ++hb)
        for (int t = 0; t < 32; t += 5) {
            printf("base+%2d thread %2d:", 16 * hb, t);
            for (int i = 0; i < 4; ++i) { uint32_t v = h[(hb * 32 + t) * 4 + i]; printf(" (lane %u col %u)", v / 1000, v % 1000); }
            printf("\n");
        }
}
