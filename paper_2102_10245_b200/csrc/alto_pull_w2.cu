// Pull-engine instantiations for 128-bit keys (alto_pull_impl.cuh).
#include "alto_pull_impl.cuh"
namespace alto {
int pull_run_w2(const alto_pull_args* a, const PullStage& S, int order, cudaStream_t s) {
  return pull_run<2>(a, S, order, s);
}
}  // namespace alto
