// interp_vec3.cu -- C^T of three real fields at once (the PIF field gather).
// Kernels and launch templates: interp_impl.cuh (one translation unit per value
// type so the template instances compile in parallel).
#include "interp_impl.cuh"

namespace nufft {

// grid = three real grids nf1 nf2 nz (x fastest), gstride reals apart; out = Np
// 3-vectors of reals (caller order)
template <typename T>
cudaError_t launch_interp_vec3(const Geom& g, const PtsView<T>& p, int64_t nbins, const T* grid,
                               int64_t gstride, T* c, double beta, cudaStream_t s) {
#define CALL(WW)                                                                          \
    launch_w<T, Vec3<T>, WW>(g, p, nbins, grid,                                           \
                             StoreOut<Vec3<T>>{reinterpret_cast<Vec3<T>*>(c)}, beta, s, gstride)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}

// the same gather with the PIF kick fused into its output: v_d += s E_d
template <typename T>
cudaError_t launch_interp_vec3_kick(const Geom& g, const PtsView<T>& p, int64_t nbins,
                                    const T* grid, int64_t gstride, T* v0, T* v1, T* v2,
                                    double scale, double beta, cudaStream_t s) {
#define CALL(WW)                                                                          \
    launch_w<T, Vec3<T>, WW>(g, p, nbins, grid, KickOut<T>{v0, v1, v2, (T)scale}, beta, s,   \
                             gstride)
    NUFFT_W_SWITCH(CALL)
#undef CALL
    return cudaErrorInvalidValue;
}


template cudaError_t launch_interp_vec3<float>(const Geom&, const PtsView<float>&, int64_t,
                                               const float*, int64_t, float*, double, cudaStream_t);
template cudaError_t launch_interp_vec3<double>(const Geom&, const PtsView<double>&, int64_t,
                                                const double*, int64_t, double*, double,
                                                cudaStream_t);
template cudaError_t launch_interp_vec3_kick<float>(const Geom&, const PtsView<float>&, int64_t,
                                                    const float*, int64_t, float*, float*, float*,
                                                    double, double, cudaStream_t);
template cudaError_t launch_interp_vec3_kick<double>(const Geom&, const PtsView<double>&, int64_t,
                                                     const double*, int64_t, double*, double*,
                                                     double*, double, double, cudaStream_t);

}  // namespace nufft
