// FP32 screen of the k-means assignment with exact FP64 fallback
// (kmeans_screen.cu): internal launchers used by the Lloyd plan (kmeans.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace csc {

// the screen handles this (d, k) (shared-memory tile fits)
bool screen_supported(int64_t d, int64_t k);
size_t screen_smem(int64_t d, int64_t k);
// centroid columns of the transposed fp32 tile (k rounded up to 64)
int64_t screen_kpad(int64_t k);
// F32 = (float)F with ld32 (multiple of 4, zero padding), fn32 = |F32 row|^2
int screen_convert_features(const double *f, int64_t n, int64_t d, int64_t ld, float *f32,
                            int64_t ld32, float *fn32, cudaStream_t st);
// c32t [d][kpad] transposed fp32 centroids, cn32 [kpad] (+inf past k),
// cmax[0] = max_j |c_j| from the fp64 cnorm
int screen_convert_centroids(const double *c, int64_t k, int64_t d, int64_t ldc,
                             const double *cnorm, float *c32t, float *cn32, double *cmax,
                             cudaStream_t st);
// rows (or all n when rows == nullptr; count in nrows_dev when given): decided
// rows get labels / widened Hamerly bounds (and a counts histogram when
// counts != nullptr); the others are appended to amb (count namb, which the
// caller zeroes) for the FP64 assignment.
int screen_assign(const float *f32, int64_t ld32, const float *fn32, const double *fn64,
                  int64_t n, int64_t d, const float *c32t, const float *cn32, int64_t k,
                  const double *cmax, const int32_t *rows, const int32_t *nrows_dev,
                  int32_t *labels, double *ub, double *lb, int32_t *counts, int32_t *amb,
                  int32_t *namb, cudaStream_t st);

// Tensor-core variant (kmeans_screen_tc.cu, tcgen05 kind::tf32, 3xTF32 split):
// same contract as screen_assign with centroids in hi / lo K-major tiles
// (tc_convert_centroids); raw_out (tests) receives E instead of decisions.
bool tc_screen_supported(int64_t d, int64_t k);
// centroid tile shape of the tensor-core screen: k rounded to 16 (UMMA N),
// d rounded to 32 (one ring unit); tile element (j, t) of hi / lo at
// (t / 4) * npad * 4 + j * 4 + t % 4
inline int tc_npad_of(int64_t k) { return (int)((k + 15) / 16 * 16); }
inline int tc_kp_of(int64_t d) { return (int)((d + 31) / 32 * 32); }
int64_t tc_centroid_floats(int64_t d, int64_t k);
int tc_convert_centroids(const double *c, int64_t k, int64_t d, int64_t ldc, const double *cnorm,
                         float *chi, float *clo, float *cn32, double *cmax, cudaStream_t st);
int tc_screen_assign(const float *f32, int64_t ld32, const float *fn32, int64_t n, int64_t d,
                     const float *chi, const float *clo, const float *cn32, int64_t k,
                     const double *cmax, const int32_t *rows, const int32_t *nrows_dev,
                     int32_t *labels, double *ub, double *lb, int32_t *counts, int32_t *amb,
                     int32_t *namb, float *raw_out, cudaStream_t st);

}  // namespace csc
