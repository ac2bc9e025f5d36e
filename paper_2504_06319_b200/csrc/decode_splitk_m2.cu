// decode_splitk_m2.cu -- instantiates the cluster-launched (MODE 2) split-K kernels
// (separate translation unit so the three MODE sets compile in parallel).
#include "splitk_impl.cuh"

namespace pda {

cudaError_t launch_splitk_m2(const CUtensorMap& tmK, const CUtensorMap& tmV, const SplitKParams& p, bool bf16,
                             int head_dim, int n_tiles, int stages, dim3 grid, cudaStream_t stream, bool kv8,
                             bool self_issue) {
    return launch_splitk_mode<2>(tmK, tmV, p, bf16, head_dim, n_tiles, stages, grid, stream, kv8, self_issue);
}

}  // namespace pda
