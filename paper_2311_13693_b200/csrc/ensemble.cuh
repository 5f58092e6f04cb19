#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/xtsg.h"

namespace xtsg {

// One mode's P replica matrices (rows x cols), generated row by row
// (gen_mode_matrices, compression.cpp:51-72). Element (p, r, c) of the
// output lives at p*stride_p + r*stride_r + c*stride_c.
struct RowJob {
  int64_t rows, cols, shared_rows;
  int32_t kind;  // XTSG_KIND_GAUSSIAN / XTSG_KIND_SPARSE (anchors always Gaussian)
  double s;
  uint64_t shared_seed;  // derive(seed, 101 + mode)
  uint64_t seed;         // ensemble seed (replica streams derive(seed, 1000+8p+tag))
  uint64_t mode_tag;     // 0, 1, 2
  int64_t p_offset;      // first replica index of this launch
  int64_t stride_p, stride_r, stride_c;
};

struct EnsembleShape {
  int64_t inner[3];  // two-stage inner rows per mode (== dims for one-stage)
};

template <class T>
void launch_mode_rows(const RowJob& job, int64_t count, T* out, cudaStream_t st);
void launch_stream_normals(uint64_t seed, int64_t n, double* out, cudaStream_t st);
void launch_stream_sparse(uint64_t seed, int64_t n, double s, double* out, cudaStream_t st);

void check_sparse_spec(double s, int64_t cols);
EnsembleShape validate_ensemble(const int64_t dims[3], const int64_t reduced[3], int64_t count,
                                int64_t shared_rows, const xtsg_ensemble_spec& spec);

}  // namespace xtsg
