// Instantiations of the specialised streaming MTTKRP: 2-word keys,
// deterministic fixed-point (int64) output.
#include "alto_mstream.cuh"

namespace alto {

int fast_w2_i64(const DevLayout& d, const uint64_t* tab, const StreamParams& P, int vd, int fd, cudaStream_t s) {
  if (vd == ALTO_F32 && fd == ALTO_F32) return try_fast<2, float, long long>(d, tab, P, s);
  if (vd == ALTO_F64 && fd == ALTO_F64) return try_fast<2, double, long long>(d, tab, P, s);
  return ALTO_EUNSUPPORTED;
}

}  // namespace alto
