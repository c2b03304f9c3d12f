// interp_real.cu -- C^T for real grids (real-valued transforms).
// Kernels and launch templates: interp_impl.cuh (one translation unit per value
// type so the template instances compile in parallel).
#include "interp_impl.cuh"

namespace nufft {

template <typename T>
cudaError_t launch_interp_real(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* grid,
                               T* c, double beta, cudaStream_t s) {
#define CALL(WW) launch_w<T, T, WW>(g, p, nbins, grid, StoreOut<T>{c}, beta, s)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}


template cudaError_t launch_interp_real<float>(const Geom&, const PtsView<float>&, int64_t,
                                               const float*, float*, double, cudaStream_t);
template cudaError_t launch_interp_real<double>(const Geom&, const PtsView<double>&, int64_t,
                                                const double*, double*, double, cudaStream_t);

}  // namespace nufft
