// dist_kernels.cu -- elementwise / packing kernels of the distributed (z-slab)
// NUFFT (§2.4: "both grid values and particles
// are partitioned according to the same spatial decomposition", halos of width
// ceil(w/2), a distributed FFT).  All are one-pass, coalesced on their dense side.
//
//   owner_count   point -> owning rank (z-slab of its fine cell), rank within it
//   pack / unpack move points, strengths and results to / from their owners
//   halo_add      ghost planes received from a neighbour added to owned planes
//   xy_pack       after the 2D (x, y) FFTs of the owned planes: keep the retained
//                 x and y modes (chi is separable) and lay them out by the
//                 destination rank of their y-mode block, ready for the all-to-all
//   z_deconv      after the 1D z FFTs of this rank's y-block: keep the retained
//                 z modes and apply D = p1 p2 p3
//   z_pad         type-2 mirror: D then chi^T along z (zeros elsewhere)
//   xy_unpad      type-2 mirror: received (x, y)-mode blocks -> zero-padded planes
#include "internal.cuh"

namespace nufft {

namespace {

constexpr int kThreads = 256;

inline unsigned grid1d(int64_t n) {
    int64_t b = (n + kThreads - 1) / kThreads;
    const int64_t cap = 148 * 32;
    if (b > cap) b = cap;
    return (unsigned)(b < 1 ? 1 : b);
}

__device__ __forceinline__ double fold_rescale_d(double x, double L, double scale, int64_t nf) {
    double xf = x - L * floor(x / L);
    double s = xf * scale;
    if (s >= (double)nf) s -= (double)nf;
    if (s < 0.0) s += (double)nf;
    return s;
}

template <typename T>
__global__ void owner_count_kernel(int64_t Np, const T* __restrict__ z, double L, double scale,
                                   int64_t nf3, int nzl, uint32_t* __restrict__ owner,
                                   uint32_t* __restrict__ rank_in, unsigned long long* counts) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - lane < Np;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool live = i < Np;
        uint32_t o = 0xffffffffu;
        if (live) {
            const double s = fold_rescale_d((double)z[i], L, scale, nf3);
            int64_t c = (int64_t)s;
            if (c >= nf3) c = nf3 - 1;
            o = (uint32_t)(c / nzl);
        }
        const unsigned active = __ballot_sync(0xffffffffu, live);
        if (live) {
            const unsigned peers = __match_any_sync(active, o);
            const int leader = __ffs(peers) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&counts[o], (unsigned long long)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            owner[i] = o;
            rank_in[i] = (uint32_t)base + (uint32_t)__popc(peers & ((1u << lane) - 1u));
        }
    }
}

template <typename V>
__global__ void pack_kernel(int64_t Np, const V* __restrict__ src, const uint32_t* __restrict__ owner,
                            const uint32_t* __restrict__ rank_in,
                            const unsigned long long* __restrict__ off, V* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Np;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[off[owner[i]] + rank_in[i]] = src[i];
}

template <typename V>
__global__ void unpack_kernel(int64_t Np, const V* __restrict__ src,
                              const uint32_t* __restrict__ owner,
                              const uint32_t* __restrict__ rank_in,
                              const unsigned long long* __restrict__ off, V* __restrict__ dst) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < Np;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[off[owner[i]] + rank_in[i]];
}

template <typename C>
__global__ void halo_add_kernel(int64_t n, C* __restrict__ dst, const C* __restrict__ src) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        C a = dst[i];
        const C b = src[i];
        a.x += b.x;
        a.y += b.y;
        dst[i] = a;
    }
}

__device__ __forceinline__ int64_t mode_of(int64_t i, int64_t N, int modeord) {
    return modeord == 0 ? i - N / 2 : (i < N / 2 ? i : i - N);
}
// signed mode -> storage index
__device__ __forceinline__ int64_t index_of(int64_t n, int64_t N, int modeord) {
    return modeord == 0 ? n + N / 2 : (n >= 0 ? n : n + N);
}

// send[q][z][ys][x] = G[z][m2][m1], x in [0, N1), y storage index i2 = q*NY + ys
template <typename C>
__global__ void xy_pack_kernel(const C* __restrict__ G, int64_t nf1, int64_t nf2, int64_t nzl,
                               int64_t N1, int64_t N2, int P, int modeord, C* __restrict__ send) {
    const int64_t NY = N2 / P;
    const int64_t total = nzl * N2 * N1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i1 = t % N1;
        const int64_t ys = (t / N1) % NY;
        const int64_t z = (t / (N1 * NY)) % nzl;
        const int64_t q = t / (N1 * NY * nzl);
        const int64_t n1 = mode_of(i1, N1, modeord), n2 = mode_of(q * NY + ys, N2, modeord);
        const int64_t m1 = n1 < 0 ? n1 + nf1 : n1, m2 = n2 < 0 ? n2 + nf2 : n2;
        send[t] = G[(z * nf2 + m2) * nf1 + m1];
    }
}

// fk[i3][ys][i1] = Z[m3][ys][i1] p1 p2 p3  (Z: nf3 lines of S = NY N1 values)
template <typename T, typename C>
__global__ void z_deconv_kernel(const C* __restrict__ Z, int64_t nf3, int64_t N1, int64_t NY,
                                int64_t N2, int64_t N3, int64_t y0, const T* __restrict__ p1,
                                const T* __restrict__ p2, const T* __restrict__ p3, int modeord,
                                C* __restrict__ fk) {
    const int64_t total = N3 * NY * N1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i1 = t % N1, ys = (t / N1) % NY, i3 = t / (N1 * NY);
        const int64_t n1 = mode_of(i1, N1, modeord), n2 = mode_of(y0 + ys, N2, modeord),
                      n3 = mode_of(i3, N3, modeord);
        const int64_t m3 = n3 < 0 ? n3 + nf3 : n3;
        const T s = p1[n1 + N1 / 2] * p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
        const C v = Z[(m3 * NY + ys) * N1 + i1];
        fk[t] = C{v.x * s, v.y * s};
    }
}

// Z[m3][ys][i1] = fk[i3][ys][i1] p1 p2 p3 on retained m3, 0 elsewhere
template <typename T, typename C>
__global__ void z_pad_kernel(const C* __restrict__ fk, int64_t nf3, int64_t N1, int64_t NY,
                             int64_t N2, int64_t N3, int64_t y0, const T* __restrict__ p1,
                             const T* __restrict__ p2, const T* __restrict__ p3, int modeord,
                             C* __restrict__ Z) {
    const int64_t total = nf3 * NY * N1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i1 = t % N1, ys = (t / N1) % NY, m3 = t / (N1 * NY);
        C v{0, 0};
        if (m3 < N3 / 2 || m3 >= nf3 - N3 / 2) {
            const int64_t n3 = m3 < N3 / 2 ? m3 : m3 - nf3;
            const int64_t i3 = modeord == 0 ? n3 + N3 / 2 : (n3 >= 0 ? n3 : n3 + N3);
            const int64_t n1 = mode_of(i1, N1, modeord), n2 = mode_of(y0 + ys, N2, modeord);
            const T s = p1[n1 + N1 / 2] * p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
            const C f = fk[(i3 * NY + ys) * N1 + i1];
            v = C{f.x * s, f.y * s};
        }
        Z[t] = v;
    }
}

// G[z][m2][m1] = recv[q][z][ys][i1] on retained (m1, m2), 0 elsewhere
template <typename C>
__global__ void xy_unpad_kernel(const C* __restrict__ recv, int64_t nf1, int64_t nf2,
                                int64_t nzl, int64_t N1, int64_t N2, int P, int modeord,
                                C* __restrict__ G) {
    const int64_t NY = N2 / P;
    const int64_t total = nzl * nf2 * nf1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m1 = t % nf1, m2 = (t / nf1) % nf2, z = t / (nf1 * nf2);
        C v{0, 0};
        const bool k1 = m1 < N1 / 2 || m1 >= nf1 - N1 / 2;
        const bool k2 = m2 < N2 / 2 || m2 >= nf2 - N2 / 2;
        if (k1 && k2) {
            const int64_t n1 = m1 < N1 / 2 ? m1 : m1 - nf1, n2 = m2 < N2 / 2 ? m2 : m2 - nf2;
            const int64_t i1 = modeord == 0 ? n1 + N1 / 2 : (n1 >= 0 ? n1 : n1 + N1);
            const int64_t i2 = modeord == 0 ? n2 + N2 / 2 : (n2 >= 0 ? n2 : n2 + N2);
            const int64_t q = i2 / NY, ys = i2 - q * NY;
            v = recv[((q * nzl + z) * NY + ys) * N1 + i1];
        }
        G[t] = v;
    }
}

// ---------------------------------------------------------------- real transforms (slab)
// Half-spectrum mode layout of a slab plan's real transforms: x index i1 = k1 in
// [0, N1/2] (H1 = N1/2 + 1 values), the rank's y-block, all z.
// xy_pack_half: after the batched 2D R2C of the owned planes (H: nzl x nf2 x hx,
// hx = nf1/2 + 1), keep k1 in [0, N1/2] and the retained y modes, laid out by the
// destination rank of their y-block: send[q][z][ys][x].
template <typename C>
__global__ void xy_pack_half_kernel(const C* __restrict__ H, int64_t nf1, int64_t nf2,
                                    int64_t nzl, int64_t N1, int64_t N2, int P, int modeord,
                                    C* __restrict__ send) {
    const int64_t NY = N2 / P, H1 = N1 / 2 + 1, hx = nf1 / 2 + 1;
    const int64_t total = nzl * N2 * H1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = t % H1;
        const int64_t ys = (t / H1) % NY;
        const int64_t z = (t / (H1 * NY)) % nzl;
        const int64_t q = t / (H1 * NY * nzl);
        const int64_t n2 = mode_of(q * NY + ys, N2, modeord);
        const int64_t m2 = n2 < 0 ? n2 + nf2 : n2;
        send[t] = H[(z * nf2 + m2) * hx + x];
    }
}
// fk[i3][ys][x] = Z[m3][ys][x] p1 p2 p3 (conj first when the type-1 sign is +: a
// real grid's + transform is the conjugate of its - transform)
template <typename T, typename C>
__global__ void z_deconv_half_kernel(const C* __restrict__ Z, int64_t nf3, int64_t N1,
                                     int64_t NY, int64_t N2, int64_t N3, int64_t y0,
                                     const T* __restrict__ p1, const T* __restrict__ p2,
                                     const T* __restrict__ p3, int modeord, int conj,
                                     C* __restrict__ fk) {
    const int64_t H1 = N1 / 2 + 1;
    const int64_t total = N3 * NY * H1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = t % H1, ys = (t / H1) % NY, i3 = t / (H1 * NY);
        const int64_t n2 = mode_of(y0 + ys, N2, modeord), n3 = mode_of(i3, N3, modeord);
        const int64_t m3 = n3 < 0 ? n3 + nf3 : n3;
        // p is even: p1(k1) = p1(-k1), stored for k in [-N1/2, N1/2)
        const T s = p1[N1 / 2 - x] * p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
        const C v = Z[(m3 * NY + ys) * H1 + x];
        fk[t] = C{v.x * s, (conj ? -v.y : v.y) * s};
    }
}
// Z[m3][ys][x] = fk[i3][ys][x] p1 p2 p3 on retained m3, 0 elsewhere (conj first when
// the type-2 sign is -: the C2R path applies +)
template <typename T, typename C>
__global__ void z_pad_half_kernel(const C* __restrict__ fk, int64_t nf3, int64_t N1, int64_t NY,
                                  int64_t N2, int64_t N3, int64_t y0, const T* __restrict__ p1,
                                  const T* __restrict__ p2, const T* __restrict__ p3,
                                  int modeord, int conj, C* __restrict__ Z) {
    const int64_t H1 = N1 / 2 + 1;
    const int64_t total = nf3 * NY * H1;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = t % H1, ys = (t / H1) % NY, m3 = t / (H1 * NY);
        C v{0, 0};
        if (m3 < N3 / 2 || m3 >= nf3 - N3 / 2) {
            const int64_t n3 = m3 < N3 / 2 ? m3 : m3 - nf3;
            const int64_t i3 = modeord == 0 ? n3 + N3 / 2 : (n3 >= 0 ? n3 : n3 + N3);
            const int64_t n2 = mode_of(y0 + ys, N2, modeord);
            const T s = p1[N1 / 2 - x] * p2[n2 + N2 / 2] * p3[n3 + N3 / 2];
            const C f = fk[(i3 * NY + ys) * H1 + x];
            v = C{f.x * s, (conj ? -f.y : f.y) * s};
        }
        Z[t] = v;
    }
}
// H[z][m2][m1] (half planes, hx = nf1/2 + 1) = recv[q][z][ys][x] on retained
// (k1 <= N1/2, k2), 0 elsewhere; on the k1 = 0 line the Hermitian part
// (X(k2) + conj X(-k2)) / 2, which the C2R transform requires
template <typename C>
__global__ void xy_unpad_half_kernel(const C* __restrict__ recv, int64_t nf1, int64_t nf2,
                                     int64_t nzl, int64_t N1, int64_t N2, int P, int modeord,
                                     C* __restrict__ H) {
    const int64_t NY = N2 / P, H1 = N1 / 2 + 1, hx = nf1 / 2 + 1;
    const int64_t total = nzl * nf2 * hx;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t m1 = t % hx, m2 = (t / hx) % nf2, z = t / (hx * nf2);
        const int64_t k2 = m2 < nf2 / 2 ? m2 : m2 - nf2;
        auto X = [&](int64_t kk2) -> C {  // retained value at (m1, kk2) of plane z
            if (m1 >= H1 || kk2 < -N2 / 2 || kk2 >= N2 / 2) return C{0, 0};
            const int64_t i2 = index_of(kk2, N2, modeord), q = i2 / NY, ys = i2 - q * NY;
            return recv[((q * nzl + z) * NY + ys) * H1 + m1];
        };
        C v = X(k2);
        if (m1 == 0) {
            const C b = X(-k2);
            v = C{(v.x + b.x) * 0.5f, (v.y - b.y) * 0.5f};
        }
        H[t] = v;
    }
}

// ---------------------------------------------------------------- PIF particle migration
// A particle's owner is the z-slab of its fine cell (the owner_count rule).
template <typename T>
__device__ __forceinline__ uint32_t slab_owner(T z, double L, double scale, int64_t nf3, int nzl) {
    const double s = fold_rescale_d((double)z, L, scale, nf3);
    int64_t c = (int64_t)s;
    if (c >= nf3) c = nf3 - 1;
    return (uint32_t)(c / nzl);
}

// pass 1: per-destination counts of the particles that left this rank's slab
template <typename T>
__global__ void migrate_count_kernel(int64_t n, const T* __restrict__ z, double L, double scale,
                                     int64_t nf3, int nzl, uint32_t me,
                                     unsigned long long* __restrict__ counts) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - lane < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t o = me;
        if (i < n) o = slab_owner(z[i], L, scale, nf3, nzl);
        const bool leave = o != me;
        const unsigned act = __ballot_sync(0xffffffffu, leave);
        if (leave) {
            const unsigned peers = __match_any_sync(act, o);
            if (lane == __ffs(peers) - 1) atomicAdd(&counts[o], (unsigned long long)__popc(peers));
        }
    }
}

// pass 2: leavers -> send records (6 values: x y z vx vy vz), grouped by
// destination; hole[pos] = the slot they vacate
template <typename T>
__global__ void migrate_pack_kernel(int64_t n, const T* __restrict__ x, const T* __restrict__ y,
                                    const T* __restrict__ z, const T* __restrict__ vx,
                                    const T* __restrict__ vy, const T* __restrict__ vz, double L,
                                    double scale, int64_t nf3, int nzl, uint32_t me,
                                    const unsigned long long* __restrict__ off,
                                    unsigned long long* __restrict__ cursor, T* __restrict__ send,
                                    int64_t* __restrict__ hole) {
    const int lane = threadIdx.x & 31;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i - lane < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t o = me;
        if (i < n) o = slab_owner(z[i], L, scale, nf3, nzl);
        const bool leave = o != me;
        const unsigned act = __ballot_sync(0xffffffffu, leave);
        if (leave) {
            const unsigned peers = __match_any_sync(act, o);
            const int leader = __ffs(peers) - 1;
            unsigned long long base = 0;
            if (lane == leader) base = atomicAdd(&cursor[o], (unsigned long long)__popc(peers));
            base = __shfl_sync(peers, base, leader);
            const int64_t pos = (int64_t)(off[o] + base + __popc(peers & ((1u << lane) - 1u)));
            T* r = send + 6 * pos;
            r[0] = x[i]; r[1] = y[i]; r[2] = z[i]; r[3] = vx[i]; r[4] = vy[i]; r[5] = vz[i];
            hole[pos] = i;
        }
    }
}

// pass 3: the vacated slots below the new count ...
__global__ void migrate_holes_kernel(int64_t nleave, const int64_t* __restrict__ hole,
                                     int64_t new_n, int64_t* __restrict__ lo,
                                     unsigned long long* __restrict__ nlo) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nleave;
         k += (int64_t)gridDim.x * blockDim.x)
        if (hole[k] < new_n) lo[atomicAdd(nlo, 1ull)] = hole[k];
}

// ... and the staying particles at or above it (as many as there are such holes)
template <typename T>
__global__ void migrate_tail_kernel(int64_t n, int64_t new_n, const T* __restrict__ z, double L,
                                    double scale, int64_t nf3, int nzl, uint32_t me,
                                    int64_t* __restrict__ tail,
                                    unsigned long long* __restrict__ ntail) {
    for (int64_t i = new_n + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if (slab_owner(z[i], L, scale, nf3, nzl) == me) tail[atomicAdd(ntail, 1ull)] = i;
}

// pass 4: tail particles fill the holes (state arrays compacted to [0, new_n))
template <typename T>
__global__ void migrate_fill_kernel(const unsigned long long* __restrict__ nholes,
                                    const int64_t* __restrict__ lo,
                                    const int64_t* __restrict__ tail, T* x, T* y, T* z, T* vx,
                                    T* vy, T* vz) {
    const int64_t h = (int64_t)*nholes;  // == number of tail stayers (pass 3)
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < h;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = lo[k], s = tail[k];
        x[d] = x[s]; y[d] = y[s]; z[d] = z[s]; vx[d] = vx[s]; vy[d] = vy[s]; vz[d] = vz[s];
    }
}

// pass 5: received records appended at [new_n, new_n + nrecv)
template <typename T>
__global__ void migrate_unpack_kernel(int64_t nrecv, const T* __restrict__ recv, int64_t at, T* x,
                                      T* y, T* z, T* vx, T* vy, T* vz) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nrecv;
         k += (int64_t)gridDim.x * blockDim.x) {
        const T* r = recv + 6 * k;
        x[at + k] = r[0]; y[at + k] = r[1]; z[at + k] = r[2];
        vx[at + k] = r[3]; vy[at + k] = r[4]; vz[at + k] = r[5];
    }
}

}  // namespace

// ---------------------------------------------------------------- launchers
template <typename T>
cudaError_t launch_owner_count(int64_t Np, const T* z, double L, double scale, int64_t nf3,
                               int nzl, uint32_t* owner, uint32_t* rank_in,
                               unsigned long long* counts, cudaStream_t s) {
    if (Np > 0)
        owner_count_kernel<T><<<grid1d(Np), kThreads, 0, s>>>(Np, z, L, scale, nf3, nzl, owner,
                                                              rank_in, counts);
    return cudaGetLastError();
}

cudaError_t launch_pack_bytes(int64_t Np, int elem_bytes, const void* src, const uint32_t* owner,
                              const uint32_t* rank_in, const unsigned long long* off, void* dst,
                              bool unpack, cudaStream_t s) {
    if (Np <= 0) return cudaSuccess;
    switch (elem_bytes) {
        case 4:
            if (unpack) unpack_kernel<float><<<grid1d(Np), kThreads, 0, s>>>(Np, (const float*)src, owner, rank_in, off, (float*)dst);
            else pack_kernel<float><<<grid1d(Np), kThreads, 0, s>>>(Np, (const float*)src, owner, rank_in, off, (float*)dst);
            break;
        case 8:
            if (unpack) unpack_kernel<double><<<grid1d(Np), kThreads, 0, s>>>(Np, (const double*)src, owner, rank_in, off, (double*)dst);
            else pack_kernel<double><<<grid1d(Np), kThreads, 0, s>>>(Np, (const double*)src, owner, rank_in, off, (double*)dst);
            break;
        case 16:
            if (unpack) unpack_kernel<double2><<<grid1d(Np), kThreads, 0, s>>>(Np, (const double2*)src, owner, rank_in, off, (double2*)dst);
            else pack_kernel<double2><<<grid1d(Np), kThreads, 0, s>>>(Np, (const double2*)src, owner, rank_in, off, (double2*)dst);
            break;
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_halo_add(int64_t n, typename Cx<T>::type* dst, const typename Cx<T>::type* src,
                            cudaStream_t s) {
    if (n > 0) halo_add_kernel<typename Cx<T>::type><<<grid1d(n), kThreads, 0, s>>>(n, dst, src);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_xy_pack(const typename Cx<T>::type* G, const int64_t nf[3], int64_t nzl,
                           const int64_t N[3], int P, int modeord, typename Cx<T>::type* send,
                           cudaStream_t s) {
    xy_pack_kernel<typename Cx<T>::type><<<grid1d(nzl * N[1] * N[0]), kThreads, 0, s>>>(
        G, nf[0], nf[1], nzl, N[0], N[1], P, modeord, send);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_z_deconv(const typename Cx<T>::type* Z, const int64_t nf[3], const int64_t N[3],
                            int64_t NY, int64_t y0, const T* p1, const T* p2, const T* p3,
                            int modeord, typename Cx<T>::type* fk, cudaStream_t s) {
    z_deconv_kernel<T, typename Cx<T>::type><<<grid1d(N[2] * NY * N[0]), kThreads, 0, s>>>(
        Z, nf[2], N[0], NY, N[1], N[2], y0, p1, p2, p3, modeord, fk);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_z_pad(const typename Cx<T>::type* fk, const int64_t nf[3], const int64_t N[3],
                         int64_t NY, int64_t y0, const T* p1, const T* p2, const T* p3,
                         int modeord, typename Cx<T>::type* Z, cudaStream_t s) {
    z_pad_kernel<T, typename Cx<T>::type><<<grid1d(nf[2] * NY * N[0]), kThreads, 0, s>>>(
        fk, nf[2], N[0], NY, N[1], N[2], y0, p1, p2, p3, modeord, Z);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_xy_unpad(const typename Cx<T>::type* recv, const int64_t nf[3], int64_t nzl,
                            const int64_t N[3], int P, int modeord, typename Cx<T>::type* G,
                            cudaStream_t s) {
    xy_unpad_kernel<typename Cx<T>::type><<<grid1d(nzl * nf[1] * nf[0]), kThreads, 0, s>>>(
        recv, nf[0], nf[1], nzl, N[0], N[1], P, modeord, G);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_migrate_count(int64_t n, const T* z, double L, double scale, int64_t nf3,
                                 int nzl, int me, unsigned long long* counts, cudaStream_t s) {
    if (n > 0)
        migrate_count_kernel<T><<<grid1d(n), kThreads, 0, s>>>(n, z, L, scale, nf3, nzl,
                                                               (uint32_t)me, counts);
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_migrate_move(int64_t n, int64_t nleave, int64_t nrecv, T* const st[6],
                                double L, double scale, int64_t nf3, int nzl, int me,
                                const unsigned long long* off, unsigned long long* cursor,
                                T* send, const T* recv, int64_t* hole, int64_t* lo,
                                int64_t* tail, unsigned long long* nlo_ntail, int phase,
                                cudaStream_t s) {
    const int64_t new_n = n - nleave;
    if (phase == 0) {  // pack leavers, list holes and tail stayers, fill the holes
        if (nleave > 0) {
            migrate_pack_kernel<T><<<grid1d(n), kThreads, 0, s>>>(
                n, st[0], st[1], st[2], st[3], st[4], st[5], L, scale, nf3, nzl, (uint32_t)me,
                off, cursor, send, hole);
            migrate_holes_kernel<<<grid1d(nleave), kThreads, 0, s>>>(nleave, hole, new_n, lo,
                                                                     nlo_ntail);
            migrate_tail_kernel<T><<<grid1d(nleave), kThreads, 0, s>>>(
                n, new_n, st[2], L, scale, nf3, nzl, (uint32_t)me, tail, nlo_ntail + 1);
            // holes below new_n == stayers at or above it (both counted on the device;
            // nleave bounds them)
            migrate_fill_kernel<T><<<grid1d(nleave), kThreads, 0, s>>>(
                nlo_ntail, lo, tail, st[0], st[1], st[2], st[3], st[4], st[5]);
        }
    } else if (nrecv > 0) {
        migrate_unpack_kernel<T><<<grid1d(nrecv), kThreads, 0, s>>>(
            nrecv, recv, new_n, st[0], st[1], st[2], st[3], st[4], st[5]);
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_xy_pack_half(const typename Cx<T>::type* H, const int64_t nf[3], int64_t nzl,
                                const int64_t N[3], int P, int modeord,
                                typename Cx<T>::type* send, cudaStream_t s) {
    xy_pack_half_kernel<typename Cx<T>::type><<<grid1d(nzl * N[1] * (N[0] / 2 + 1)), kThreads, 0,
                                                s>>>(H, nf[0], nf[1], nzl, N[0], N[1], P, modeord,
                                                     send);
    return cudaGetLastError();
}
template <typename T>
cudaError_t launch_z_deconv_half(const typename Cx<T>::type* Z, const int64_t nf[3],
                                 const int64_t N[3], int64_t NY, int64_t y0, const T* p1,
                                 const T* p2, const T* p3, int modeord, int conj,
                                 typename Cx<T>::type* fk, cudaStream_t s) {
    z_deconv_half_kernel<T, typename Cx<T>::type><<<grid1d(N[2] * NY * (N[0] / 2 + 1)), kThreads,
                                                    0, s>>>(Z, nf[2], N[0], NY, N[1], N[2], y0, p1,
                                                            p2, p3, modeord, conj, fk);
    return cudaGetLastError();
}
template <typename T>
cudaError_t launch_z_pad_half(const typename Cx<T>::type* fk, const int64_t nf[3],
                              const int64_t N[3], int64_t NY, int64_t y0, const T* p1, const T* p2,
                              const T* p3, int modeord, int conj, typename Cx<T>::type* Z,
                              cudaStream_t s) {
    z_pad_half_kernel<T, typename Cx<T>::type><<<grid1d(nf[2] * NY * (N[0] / 2 + 1)), kThreads, 0,
                                                 s>>>(fk, nf[2], N[0], NY, N[1], N[2], y0, p1, p2,
                                                      p3, modeord, conj, Z);
    return cudaGetLastError();
}
template <typename T>
cudaError_t launch_xy_unpad_half(const typename Cx<T>::type* recv, const int64_t nf[3],
                                 int64_t nzl, const int64_t N[3], int P, int modeord,
                                 typename Cx<T>::type* H, cudaStream_t s) {
    xy_unpad_half_kernel<typename Cx<T>::type><<<grid1d(nzl * nf[1] * (nf[0] / 2 + 1)), kThreads,
                                                 0, s>>>(recv, nf[0], nf[1], nzl, N[0], N[1], P,
                                                         modeord, H);
    return cudaGetLastError();
}

#define NUFFT_DIST_INST(T)                                                                         \
    template cudaError_t launch_owner_count<T>(int64_t, const T*, double, double, int64_t, int,      \
                                               uint32_t*, uint32_t*, unsigned long long*,            \
                                               cudaStream_t);                                        \
    template cudaError_t launch_halo_add<T>(int64_t, Cx<T>::type*, const Cx<T>::type*,               \
                                            cudaStream_t);                                           \
    template cudaError_t launch_xy_pack<T>(const Cx<T>::type*, const int64_t*, int64_t,              \
                                           const int64_t*, int, int, Cx<T>::type*, cudaStream_t);    \
    template cudaError_t launch_z_deconv<T>(const Cx<T>::type*, const int64_t*, const int64_t*,      \
                                            int64_t, int64_t, const T*, const T*, const T*, int,     \
                                            Cx<T>::type*, cudaStream_t);                             \
    template cudaError_t launch_z_pad<T>(const Cx<T>::type*, const int64_t*, const int64_t*,         \
                                         int64_t, int64_t, const T*, const T*, const T*, int,        \
                                         Cx<T>::type*, cudaStream_t);                                \
    template cudaError_t launch_xy_unpad<T>(const Cx<T>::type*, const int64_t*, int64_t,             \
                                            const int64_t*, int, int, Cx<T>::type*, cudaStream_t);
NUFFT_DIST_INST(float)
NUFFT_DIST_INST(double)
#define NUFFT_DIST_HALF_INST(T)                                                                   \
    template cudaError_t launch_xy_pack_half<T>(const Cx<T>::type*, const int64_t*, int64_t,      \
                                                const int64_t*, int, int, Cx<T>::type*,          \
                                                cudaStream_t);                                     \
    template cudaError_t launch_z_deconv_half<T>(const Cx<T>::type*, const int64_t*,              \
                                                 const int64_t*, int64_t, int64_t, const T*,      \
                                                 const T*, const T*, int, int, Cx<T>::type*,      \
                                                 cudaStream_t);                                    \
    template cudaError_t launch_z_pad_half<T>(const Cx<T>::type*, const int64_t*, const int64_t*, \
                                              int64_t, int64_t, const T*, const T*, const T*, int, \
                                              int, Cx<T>::type*, cudaStream_t);                   \
    template cudaError_t launch_xy_unpad_half<T>(const Cx<T>::type*, const int64_t*, int64_t,     \
                                                 const int64_t*, int, int, Cx<T>::type*,          \
                                                 cudaStream_t);
NUFFT_DIST_HALF_INST(float)
NUFFT_DIST_HALF_INST(double)
#undef NUFFT_DIST_HALF_INST
template cudaError_t launch_migrate_count<float>(int64_t, const float*, double, double, int64_t,
                                                 int, int, unsigned long long*, cudaStream_t);
template cudaError_t launch_migrate_count<double>(int64_t, const double*, double, double, int64_t,
                                                  int, int, unsigned long long*, cudaStream_t);
template cudaError_t launch_migrate_move<float>(int64_t, int64_t, int64_t, float* const*, double,
                                                double, int64_t, int, int,
                                                const unsigned long long*, unsigned long long*,
                                                float*, const float*, int64_t*, int64_t*,
                                                int64_t*, unsigned long long*, int, cudaStream_t);
template cudaError_t launch_migrate_move<double>(int64_t, int64_t, int64_t, double* const*, double,
                                                 double, int64_t, int, int,
                                                 const unsigned long long*, unsigned long long*,
                                                 double*, const double*, int64_t*, int64_t*,
                                                 int64_t*, unsigned long long*, int, cudaStream_t);
#undef NUFFT_DIST_INST

}  // namespace nufft
