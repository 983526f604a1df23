// How many clusters of each size can be co-resident for the sweep-pair kernel.
#include "../../paper_1904_06556_b200/csrc/vts_b200.cu"
#include <cstdio>
int main() {
  if (vts::gs_prepare()) return 1;
  for (int cs = 1; cs <= 16; ++cs) {
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(32 * vts::gs::kWarpsPair);
    cfg.dynamicSmemBytes = sizeof(vts::gs::Smem);
    cfg.gridDim = dim3(cs * 16);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (const void*)vts::k_gs_pair<true, true>, &cfg);
    printf("cluster size %2d: max active clusters %3d (%3d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  return 0;
}
