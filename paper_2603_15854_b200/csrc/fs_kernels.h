// fs_kernels.h -- internal launch interface between the C ABI (fs_api.cu) and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/flashsample.h"

namespace fs {

struct State;

// Parameters of one stage-1 launch (one chunk of <= 256 batch rows).
struct StageOneParams {
  const void* h;              // [B, D] (SIMT kernel reads it directly; the TC kernel via TMA)
  const void* W;              // [V, D]
  const float* bias;          // [V] (shard-local) or nullptr
  const float* temperature;   // [B] for this chunk or nullptr
  const uint32_t* mask;       // [B][mask_words] for this chunk (global ids) or nullptr
  int64_t mask_words;
  int64_t vocab_offset;       // global id of local row 0
  uint64_t seed, step;
  int B, D, V;                // V = local rows
  int row_offset;             // global batch index of this chunk's row 0
  int group_size;             // local rows per group (multiple of 128); >= V for one group
  int max_seg;                // candidate slots per CTA
  int stages;                 // TMA ring depth (TC kernel)
  State* part;                // [grid * max_seg][B] candidate states
  int* part_group;            // [grid * max_seg] group id of each slot, -1 = unused
};

struct TcMaps {
  CUtensorMap w128, w16, h;
};

int tc_block_n(int B);
int tc_stages(int BN);
cudaError_t launch_fused_tc(const TcMaps& maps, const StageOneParams& p, int BN, bool lse, int grid,
                            cudaStream_t stream);
// CUDA-core stage 1: grid = ceil(V/128) aligned tiles, one slot per tile.
cudaError_t launch_fused_simt(const StageOneParams& p, fs_dtype dtype, bool lse, cudaStream_t stream);

// Stage 2: reduce the candidate slots of every row into groups and the final sample.
cudaError_t launch_reduce(const State* part, const int* part_group, int n_slots, int B, int n_groups,
                          int32_t* idx_out, float* score_out, float* logZ_out, fs_summary* groups_out,
                          cudaStream_t stream, bool pdl);
cudaError_t launch_combine(const fs_summary* gathered, int n, int B, int32_t* idx_out, float* score_out,
                           float* logZ_out, cudaStream_t stream);
cudaError_t launch_merge(const fs_summary* a, const fs_summary* b, fs_summary* out, int count,
                         cudaStream_t stream);
cudaError_t launch_random_bits(uint64_t seed, uint64_t step, uint32_t tag, const int32_t* b, const int64_t* v,
                               uint32_t* r, int64_t n, cudaStream_t stream);
cudaError_t launch_gumbel(const uint32_t* r, float* g, int64_t n, cudaStream_t stream);

}  // namespace fs
