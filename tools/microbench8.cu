// Grid-wide barrier cost on B200: cooperative-groups grid.sync() vs a
// cluster barrier (16 CTAs), 148 / 16 CTAs (experiment tooling).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_grid(int iters, int* out) {
    cg::grid_group g = cg::this_grid();
    int x = 0;
    for (int i = 0; i < iters; ++i) { x += threadIdx.x; g.sync(); }
    if (x == -1) out[0] = x;
}
__global__ void __cluster_dims__(16, 1, 1) k_cluster(int iters, int* out) {
    cg::cluster_group c = cg::this_cluster();
    int x = 0;
    for (int i = 0; i < iters; ++i) { x += threadIdx.x; c.sync(); }
    if (x == -1) out[0] = x;
}
__global__ void __cluster_dims__(8, 1, 1) k_cluster8(int iters, int* out) {
    cg::cluster_group c = cg::this_cluster();
    int x = 0;
    for (int i = 0; i < iters; ++i) { x += threadIdx.x; c.sync(); }
    if (x == -1) out[0] = x;
}
int main() {
    int* o; cudaMalloc(&o, 4);
    int iters = 20000;
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
    for (int G : {148, 74, 16}) {
        void* args[] = {&iters, &o};
        cudaLaunchCooperativeKernel((void*)k_grid, G, 256, args, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_grid, G, 256, args, 0, 0);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        printf("grid.sync  G=%3d: %.3f us/sync (err %d)\n", G, ms * 1e3 / iters, (int)cudaGetLastError());
    }
    cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    k_cluster<<<16, 256>>>(iters, o);
    cudaEventRecord(a); k_cluster<<<16, 256>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster.sync 16: %.3f us/sync (err %d)\n", ms * 1e3 / iters, (int)cudaGetLastError());
    k_cluster8<<<8, 256>>>(iters, o);
    cudaEventRecord(a); k_cluster8<<<8, 256>>>(iters, o); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("cluster.sync 8: %.3f us/sync (err %d)\n", ms * 1e3 / iters, (int)cudaGetLastError());
}
