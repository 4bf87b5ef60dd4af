// Instantiations of the streaming MTTKRP kernel: 1-word keys, f64 output.
#include "alto_stream.cuh"

namespace alto {

int stream_w1_f64(const DevLayout& d, const uint64_t* tab, const StreamParams& P, int vd, int fd,
                   cudaStream_t s) {
  if (vd == ALTO_F32 && fd == ALTO_F32) return by_order<1, float, float, double>(d, tab, P, s);
  if (vd == ALTO_F64 && fd == ALTO_F64) return by_order<1, double, double, double>(d, tab, P, s);
  if (vd == ALTO_F32 && fd == ALTO_F64) return by_order<1, float, double, double>(d, tab, P, s);
  set_error("float64 values with float32 factors: upcast the factors (exact) first");
  return ALTO_EUNSUPPORTED;
}

}  // namespace alto
