// interp.cu -- C^T for complex grids, plus the plan-level helpers.
// Kernels and launch templates: interp_impl.cuh (one translation unit per value
// type so the template instances compile in parallel).
#include "interp_impl.cuh"

namespace nufft {

template <typename T>
cudaError_t launch_interp(const Geom& g, const PtsView<T>& p, int64_t nbins,
                          const typename Cx<T>::type* grid, typename Cx<T>::type* c, double beta,
                          cudaStream_t s, const void* tmap) {
#define CALL(WW)                                                                            \
    launch_w<T, typename Cx<T>::type, WW>(g, p, nbins, grid, StoreOut<typename Cx<T>::type>{c}, \
                                          beta, s, 0, tmap)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}

template <typename T>
size_t interp_smem_bytes(const Geom& g) {
#define CALL(WW) smem_w<T, typename Cx<T>::type, WW>(g)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return 0;
}

int interp_tile_pitch(int cell_bytes, int T, int W, bool sub) {
    if (sub) return cell_bytes == 16 ? sub_pitch<16>(tile_len<16>(T, W)) : sub_pitch<8>(tile_len<8>(T, W));
    return cell_bytes == 16 ? tile_pitch<16>(T, W) : tile_pitch<8>(T, W);
}


template cudaError_t launch_interp<float>(const Geom&, const PtsView<float>&, int64_t,
                                          const float2*, float2*, double, cudaStream_t,
                                          const void*);
template cudaError_t launch_interp<double>(const Geom&, const PtsView<double>&, int64_t,
                                           const double2*, double2*, double, cudaStream_t,
                                           const void*);
template size_t interp_smem_bytes<float>(const Geom&);
template size_t interp_smem_bytes<double>(const Geom&);

}  // namespace nufft
