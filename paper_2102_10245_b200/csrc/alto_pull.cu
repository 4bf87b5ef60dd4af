// alto_pull.cu — C ABI of the K8/K9 pull engine (alto_pull.cuh).
#include "alto_pull_impl.cuh"

using namespace alto;

extern "C" {

int alto_mttkrp_pull(const alto_pull_args* a, void* stream) {
  ALTO_REQUIRE(a && a->lay, "pull args incomplete");
  ALTO_REQUIRE(a->lay->order >= 1 && a->lay->order <= ALTO_MAX_ORDER, "bad layout order");
  ALTO_REQUIRE(a->mode >= 0 && a->mode < a->lay->order, "mode out of range");
  ALTO_REQUIRE(a->rank >= 1, "rank must be positive");
  ALTO_REQUIRE(a->out != nullptr, "out is NULL");
  ALTO_REQUIRE(a->tile >= 128 && a->tile % 128 == 0, "tile must be a positive multiple of 128");
  ALTO_REQUIRE(a->m >= 0 && a->m < (1ll << 32) - 1, "pull engine supports fewer than 2^32 elements");
  const DevLayout d = make_dev_layout(a->lay);
  for (int n = 0; n < d.order; ++n) ALTO_REQUIRE(d.bits[n] <= 31, "pull engine needs mode extents below 2^31");
  const bool delta = a->mbase != nullptr;
  const MsFields f = delta ? ms_fields_delta(d, a->mode) : ms_fields(d, a->mode);
  if (!f.ok) {
    set_error("pull engine: the mode's field layout does not fit the key width");
    return ALTO_EUNSUPPORTED;
  }
  const long long dim = d.dims[a->mode];
  ALTO_REQUIRE(a->m == 0 || (a->mkeys && a->mvals && a->slice_rows), "mode stream or slice rows missing");
  ALTO_REQUIRE(a->atomic || a->m == 0 || a->slice_rec, "Buffered pull needs slice_rec");
  ALTO_REQUIRE(a->n_seg == 0 || a->seg_row, "shared rows missing");
  ALTO_REQUIRE(a->atomic || a->n_chunks == 0 || (a->rec && a->chunk_off && a->chunk_seg && a->seg_chunk_off &&
                                                   a->part && (a->n_mseg == 0 || a->mseg)),
               "pull plan incomplete");
  cudaStream_t s = as_stream(stream);
  if (a->m == 0) {
    const size_t ob = a->out_dtype == ALTO_F32 ? 4 : 8;
    ALTO_CUDA_TRY(cudaMemsetAsync(a->out, 0, static_cast<size_t>(dim) * a->rank * ob, s));
    return ALTO_OK;
  }
  PullStage S{};
  S.keys = a->mkeys;
  S.vals = a->mvals;
  S.m = a->m;
  S.tile = a->tile;
  S.mode = a->mode;
  S.dim = dim;
  S.f = f;
  for (int n = 0; n < ALTO_MAX_ORDER; ++n) S.factors[n] = n < d.order ? a->factors[n] : nullptr;
  ALTO_REQUIRE(a->n_pairs >= 0 && a->n_pairs <= 2, "at most 2 paired input modes");
  if (a->n_pairs > 0) {
    // gathered inputs: the pairs' product tables, then the unpaired input factors (alto_krp_pair; same
    // rules as alto_mttkrp_args.pair_*)
    ALTO_REQUIRE(a->factor_dtype == ALTO_F32 && a->value_dtype == ALTO_F32 && a->rank == 16 && d.order >= 4,
                 "paired input modes need float32 data, rank 16 and order 4 or 5");
    int nv = 0;
    unsigned used = 1u << a->mode;
    for (int i = 0; i < a->n_pairs; ++i) {
      const int pa = a->pair_a[i], pb = a->pair_b[i];
      ALTO_REQUIRE(pa >= 0 && pb >= 0 && pa < d.order && pb < d.order && pa != pb && !((used >> pa) & 1u) &&
                       !((used >> pb) & 1u) && a->pair_tab[i] &&
                       d.dims[pa] * d.dims[pb] * a->rank * 4ll <= 0xFFFFFFFFll,
                   "bad input-mode pair");
      used |= (1u << pa) | (1u << pb);
      S.vin[nv++] = VIn{a->pair_tab[i], pa, pb, static_cast<unsigned>(d.dims[pb])};
    }
    for (int n = 0; n < d.order; ++n)
      if (!((used >> n) & 1u)) S.vin[nv++] = VIn{a->factors[n], n, -1, 1u};
  }
  S.out = a->out;
  S.rec = a->rec;
  S.slice_rec = reinterpret_cast<const int2*>(a->slice_rec);
  S.slice_rows = reinterpret_cast<const int2*>(a->slice_rows);
  const int st = delta ? pull_run_w1_delta(a, S, d.order, s)
                       : (d.n_words == 1 ? pull_run_w1(a, S, d.order, s) : pull_run_w2(a, S, d.order, s));
  if (st == ALTO_EUNSUPPORTED)
    set_error("pull engine supports orders 3-5, ranks 16/32 (8/64 float32 Buffered) and dtypes "
              "f32/f32/f32, f32/f32/f64, f64/f64/f64, f32/f64/f64");
  return st;
}

int alto_pull_slice_rows(const alto_layout* lay, const uint64_t* mkeys, int64_t m, int32_t mode, int32_t tile,
                         const int32_t* base, int32_t* first_last, void* stream) {
  ALTO_REQUIRE(lay && mode >= 0 && mode < lay->order, "mode out of range");
  ALTO_REQUIRE(tile >= 128 && tile % 128 == 0, "tile must be a positive multiple of 128");
  if (m <= 0) return ALTO_OK;
  const DevLayout d = make_dev_layout(lay);
  const MsFields f = base ? ms_fields_delta(d, mode) : ms_fields(d, mode);
  ALTO_REQUIRE(f.ok, "the mode's field layout does not fit the key width");
  cudaStream_t s = as_stream(stream);
  const long long ns = (m + tile / 8 - 1) / (tile / 8);
  auto* fl = reinterpret_cast<int2*>(first_last);
  const int* b = reinterpret_cast<const int*>(base);
  if (d.n_words == 1 || base)
    pull_slice_rows_kernel<1><<<grid_for(ns, 256), 256, 0, s>>>(mkeys, m, tile, f, mode, b, fl);
  else
    pull_slice_rows_kernel<2><<<grid_for(ns, 256), 256, 0, s>>>(mkeys, m, tile, f, mode, b, fl);
  ALTO_LAUNCH_CHECK("alto_pull_slice_rows");
  return ALTO_OK;
}

}  // extern "C"
