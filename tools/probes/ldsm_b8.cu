// Probe: register layout of ldmatrix.m16n16.x2.trans.shared.b8 on sm_100a.
// smem[r][c] = r * 16 + c (two 16x16 byte matrices, rows addressed by lanes
// 0-15 (matrix 0) and 16-31 (matrix 1)); prints, per lane, the (row, col) of
// every byte it received.
#include <cstdio>
#include <cstdint>
__global__ void k(uint32_t* out) {
    __shared__ __align__(128) uint8_t sm[512];
    for (int i = threadIdx.x; i < 512; i += 32) sm[i] = (uint8_t)(i < 256 ? i : 255 - (i - 256));  // matrix 1 stored complemented
    __syncwarp();
    const int l = threadIdx.x;
    // matrix m = l / 16, row r = l % 16 -> 16 bytes at sm[m * 256 + r * 16]
    uint32_t addr = (uint32_t)__cvta_generic_to_shared(sm + (l / 16) * 256 + (l % 16) * 16);
    uint32_t a, b, c, d;
    asm volatile("ldmatrix.sync.aligned.m16n16.x2.trans.shared.b8 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(addr));
    out[l * 4 + 0] = a; out[l * 4 + 1] = b; out[l * 4 + 2] = c; out[l * 4 + 3] = d;
}
int main() {
    uint32_t* d; cudaMalloc(&d, 512);
    k<<<1, 32>>>(d);
    uint32_t h[128]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
    for (int l = 0; l < 32; ++l) {
        printf("lane %2d:", l);
        for (int r = 0; r < 4; ++r) {
            printf(" |");
            for (int by = 0; by < 4; ++by) {
                int v = (h[l * 4 + r] >> (8 * by)) & 255;
                if (r >= 2) v = 255 - v;  // matrix 1 (if regs 2,3 come from it)
                printf(" %x,%x", v / 16, v % 16);
            }
        }
        printf("\n");
    }
    return 0;
}
