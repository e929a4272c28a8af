// fs_api.cu -- the C ABI declared in include/flashsample.h: argument validation, workspace,
// TMA descriptors, kernel selection and the stage-1 / stage-2 launch sequence.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/flashsample.h"
#include "fs_device.cuh"
#include "fs_kernels.h"

#define FS_VERSION_STRING "flashsample-b200 0.1.0 (sm_100a)"

namespace {

thread_local std::string g_last_error;

fs_status fail(fs_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}
fs_status cuda_fail(cudaError_t e, const char* where) {
  return fail(FS_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace

struct fs_ctx {
  int device = 0;
  int num_sms = 0;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  int force_simt = 0;
  int max_ctas = 0;
  int pdl = 1;
  int stages_override = 0;
  PFN_encodeTiled encode = nullptr;
};

namespace {

fs_status ensure_ws(fs_ctx* ctx, size_t bytes) {
  if (bytes <= ctx->ws_bytes) return FS_OK;
  if (ctx->ws) cudaFree(ctx->ws);
  ctx->ws = nullptr;
  ctx->ws_bytes = 0;
  size_t want = std::max(bytes, (size_t)1 << 20);
  cudaError_t e = cudaMalloc(&ctx->ws, want);
  if (e != cudaSuccess) return fail(FS_ERR_OOM, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
  ctx->ws_bytes = want;
  return FS_OK;
}

fs_status make_map(fs_ctx* ctx, CUtensorMap* m, const void* base, int64_t inner, int64_t rows, int box_rows) {
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
  const cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1u, 1u};
  CUresult r = ctx->encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(FS_ERR_INVALID, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) + ")");
  return FS_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct PathArgs {
  fs_dtype dtype;
  const void* h;
  const void* W;
  const float* bias;
  const float* temperature;
  const uint32_t* mask;
  int64_t mask_words;
  uint64_t seed, step;
  int B, D, V;
  int64_t vocab_offset;
  int group_size;     // local rows per group; >= V means one group
  bool lse;
  int32_t* idx_out;
  float* score_out;
  float* logZ_out;
  fs_summary* groups_out;
  int n_groups;
};

fs_status run_path(fs_ctx* ctx, const PathArgs& a, cudaStream_t stream) {
  cudaError_t e = cudaSetDevice(ctx->device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  const bool tc = !ctx->force_simt && a.dtype == FS_BF16 && (a.D % 8 == 0) && aligned16(a.h) && aligned16(a.W);
  const size_t esz = a.dtype == FS_BF16 ? 2 : 4;
  const int U = (a.V + 15) / 16;
  int G = std::min(ctx->max_ctas > 0 ? ctx->max_ctas : ctx->num_sms, U);
  int max_seg = 1, n_slots;
  if (tc) {
    const int64_t rows_max = 16LL * ((U + G - 1) / G);
    max_seg = (a.group_size >= a.V) ? 1 : (int)((rows_max + a.group_size - 1) / a.group_size + 1);
    n_slots = G * max_seg;
  } else {
    n_slots = (a.V + 127) / 128;
  }
  const int chunk = 256;
  const int Bc_max = std::min(a.B, chunk);
  const size_t part_bytes = (size_t)n_slots * Bc_max * sizeof(fs::State);
  const size_t grp_off = (part_bytes + 255) & ~size_t(255);
  fs_status st = ensure_ws(ctx, grp_off + (size_t)n_slots * sizeof(int));
  if (st != FS_OK) return st;
  fs::State* part = static_cast<fs::State*>(ctx->ws);
  int* part_group = reinterpret_cast<int*>(static_cast<char*>(ctx->ws) + grp_off);

  for (int r0 = 0; r0 < a.B; r0 += chunk) {
    const int Bc = std::min(chunk, a.B - r0);
    fs::StageOneParams p{};
    p.h = static_cast<const char*>(a.h) + (size_t)r0 * a.D * esz;
    p.W = a.W;
    p.bias = a.bias;
    p.temperature = a.temperature ? a.temperature + r0 : nullptr;
    p.mask = a.mask ? a.mask + (size_t)r0 * a.mask_words : nullptr;
    p.mask_words = a.mask_words;
    p.vocab_offset = a.vocab_offset;
    p.seed = a.seed;
    p.step = a.step;
    p.B = Bc;
    p.D = a.D;
    p.V = a.V;
    p.row_offset = r0;
    p.group_size = a.group_size;
    p.max_seg = max_seg;
    p.part = part;
    p.part_group = part_group;
    if (tc) {
      const int BN = fs::tc_block_n(Bc);
      p.stages = ctx->stages_override > 0 ? ctx->stages_override : fs::tc_stages(BN);
      fs::TcMaps maps;
      if ((st = make_map(ctx, &maps.w128, a.W, a.D, a.V, 128)) != FS_OK) return st;
      if ((st = make_map(ctx, &maps.w16, a.W, a.D, a.V, 16)) != FS_OK) return st;
      if ((st = make_map(ctx, &maps.h, p.h, a.D, Bc, BN)) != FS_OK) return st;
      e = fs::launch_fused_tc(maps, p, BN, a.lse, G, stream);
      if (e != cudaSuccess) return cuda_fail(e, "stage-1 tcgen05 kernel launch");
    } else {
      e = fs::launch_fused_simt(p, a.dtype, a.lse, stream);
      if (e != cudaSuccess) return cuda_fail(e, "stage-1 CUDA-core kernel launch");
    }
    e = fs::launch_reduce(part, part_group, n_slots, Bc, a.n_groups, a.idx_out ? a.idx_out + r0 : nullptr,
                          a.score_out ? a.score_out + r0 : nullptr, a.logZ_out ? a.logZ_out + r0 : nullptr,
                          a.groups_out ? a.groups_out + (size_t)r0 * a.n_groups : nullptr, stream, ctx->pdl != 0);
    if (e != cudaSuccess) return cuda_fail(e, "stage-2 reduce launch");
  }
  return FS_OK;
}

fs_status check_common(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, int B, int D, int V) {
  if (!ctx) return fail(FS_ERR_INVALID, "ctx is NULL");
  if (dtype != FS_BF16 && dtype != FS_F32) return fail(FS_ERR_INVALID, "unknown dtype");
  if (!h || !W) return fail(FS_ERR_INVALID, "h and W are required");
  if (B < 1 || D < 1 || V < 1) return fail(FS_ERR_INVALID, "B, D and V must be >= 1");
  const size_t esz = dtype == FS_BF16 ? 2 : 4;
  if ((reinterpret_cast<uintptr_t>(h) | reinterpret_cast<uintptr_t>(W)) % esz)
    return fail(FS_ERR_INVALID, "h and W must be aligned to their element size");
  return FS_OK;
}

}  // namespace

extern "C" {

const char* fs_version(void) { return FS_VERSION_STRING; }

const char* fs_status_str(fs_status s) {
  switch (s) {
    case FS_OK: return "FS_OK";
    case FS_ERR_INVALID: return "FS_ERR_INVALID";
    case FS_ERR_UNSUPPORTED: return "FS_ERR_UNSUPPORTED";
    case FS_ERR_CUDA: return "FS_ERR_CUDA";
    case FS_ERR_OOM: return "FS_ERR_OOM";
  }
  return "FS_ERR_UNKNOWN";
}

const char* fs_last_error(void) { return g_last_error.c_str(); }

fs_status fs_ctx_create(int device, fs_ctx** out) {
  if (!out) return fail(FS_ERR_INVALID, "out is NULL");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) return fail(FS_ERR_UNSUPPORTED, "no CUDA device available");
  if (device < 0 || device >= n) return fail(FS_ERR_INVALID, "device ordinal out of range");
  int major = 0, minor = 0, sms = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  if (major != 10 || minor != 0)
    return fail(FS_ERR_UNSUPPORTED, "this build targets sm_100a (B200); device is sm_" + std::to_string(major) +
                                        std::to_string(minor));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) return fail(FS_ERR_CUDA, "cuTensorMapEncodeTiled entry point not found");
  fs_ctx* c = new fs_ctx();
  c->device = device;
  c->num_sms = sms;
  c->encode = reinterpret_cast<PFN_encodeTiled>(fn);
  *out = c;
  return FS_OK;
}

void fs_ctx_destroy(fs_ctx* ctx) {
  if (!ctx) return;
  if (ctx->ws) cudaFree(ctx->ws);
  delete ctx;
}

fs_status fs_ctx_set_option(fs_ctx* ctx, const char* name, int64_t value) {
  if (!ctx || !name) return fail(FS_ERR_INVALID, "ctx and name are required");
  if (!strcmp(name, "force_simt")) ctx->force_simt = (int)value;
  else if (!strcmp(name, "max_ctas")) ctx->max_ctas = (int)value;
  else if (!strcmp(name, "pdl")) ctx->pdl = (int)value;
  else if (!strcmp(name, "stages")) ctx->stages_override = (int)value;
  else return fail(FS_ERR_INVALID, std::string("unknown option ") + name);
  return FS_OK;
}

fs_status fs_sample(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, const float* bias,
                    const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int D, int V,
                    int32_t* idx_out, float* score_out, void* stream) {
  fs_status s = check_common(ctx, dtype, h, W, B, D, V);
  if (s != FS_OK) return s;
  if (!idx_out) return fail(FS_ERR_INVALID, "idx_out is required");
  PathArgs a{dtype, h, W, bias, temperature, mask, ((int64_t)V + 31) / 32, seed, step, B, D, V, 0,
             ((V + 127) / 128) * 128, false, idx_out, score_out, nullptr, nullptr, 1};
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

fs_status fs_sample_grouped(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W, const float* bias,
                            const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B,
                            int D, int V, int group_size, int32_t* idx_out, float* score_out, float* logZ_out,
                            fs_summary* groups_out, void* stream) {
  fs_status s = check_common(ctx, dtype, h, W, B, D, V);
  if (s != FS_OK) return s;
  if (!idx_out) return fail(FS_ERR_INVALID, "idx_out is required");
  if (group_size < 128 || group_size % 128 != 0) return fail(FS_ERR_INVALID, "group_size must be a positive multiple of 128");
  const int n_groups = (V + group_size - 1) / group_size;
  PathArgs a{dtype, h, W, bias, temperature, mask, ((int64_t)V + 31) / 32, seed, step, B, D, V, 0,
             group_size, true, idx_out, score_out, logZ_out, groups_out, n_groups};
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

fs_status fs_sample_shard(fs_ctx* ctx, fs_dtype dtype, const void* h, const void* W_shard, const float* bias_shard,
                          const float* temperature, const uint32_t* mask, uint64_t seed, uint64_t step, int B, int D,
                          int V_local, int64_t vocab_offset, int64_t V_total, fs_summary* summary_out, void* stream) {
  fs_status s = check_common(ctx, dtype, h, W_shard, B, D, V_local);
  if (s != FS_OK) return s;
  if (!summary_out) return fail(FS_ERR_INVALID, "summary_out is required");
  if (vocab_offset < 0 || V_total < vocab_offset + V_local || V_total >= (1LL << 31))
    return fail(FS_ERR_INVALID, "need 0 <= vocab_offset, vocab_offset + V_local <= V_total < 2^31");
  PathArgs a{dtype, h, W_shard, bias_shard, temperature, mask, (V_total + 31) / 32, seed, step, B, D, V_local,
             vocab_offset, ((V_local + 127) / 128) * 128, true, nullptr, nullptr, nullptr, summary_out, 1};
  return run_path(ctx, a, static_cast<cudaStream_t>(stream));
}

fs_status fs_combine_summaries(const fs_summary* gathered, int n, int B, int32_t* idx_out, float* score_out,
                               float* logZ_out, void* stream) {
  if (!gathered || !idx_out || n < 1 || B < 1) return fail(FS_ERR_INVALID, "gathered, idx_out, n >= 1, B >= 1 required");
  cudaError_t e = fs::launch_combine(gathered, n, B, idx_out, score_out, logZ_out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "combine launch");
}

fs_status fs_merge_summaries(const fs_summary* a, const fs_summary* b, fs_summary* out, int count, void* stream) {
  if (!a || !b || !out || count < 0) return fail(FS_ERR_INVALID, "a, b, out required");
  if (count == 0) return FS_OK;
  cudaError_t e = fs::launch_merge(a, b, out, count, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "merge launch");
}

fs_status fs_random_bits(uint64_t seed, uint64_t step, uint32_t tag, const int32_t* b, const int64_t* v,
                         uint32_t* r_out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!b || !v || !r_out))) return fail(FS_ERR_INVALID, "b, v, r_out required");
  cudaError_t e = fs::launch_random_bits(seed, step, tag, b, v, r_out, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "random_bits launch");
}

fs_status fs_gumbel_from_bits(const uint32_t* r, float* g_out, int64_t n, void* stream) {
  if (n < 0 || (n > 0 && (!r || !g_out))) return fail(FS_ERR_INVALID, "r, g_out required");
  cudaError_t e = fs::launch_gumbel(r, g_out, n, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? FS_OK : cuda_fail(e, "gumbel launch");
}

}  // extern "C"
