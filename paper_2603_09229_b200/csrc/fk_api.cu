// fk_api.cu -- the extern "C" boundary declared in include/flashkmeans.h.
// Validation happens here, before any launch (the reference validates before
// any kernel call: flash_assign.py:152-157, sort_inverse.py:120-122,
// baseline.py:134-137); kernels never see malformed shapes.
#include <climits>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/flashkmeans.h"
#include "fk_common.cuh"
#include "fk_kernels.h"

namespace {

thread_local std::string g_last_cuda_error;

fk_status cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FK_OK;
  g_last_cuda_error = cudaGetErrorString(e);
  return FK_ECUDA;
}

struct DevInfo {
  int sms = 0;
  int major = 0, minor = 0;
};

DevInfo dev_info() {
  static std::mutex mu;
  static DevInfo cache[64];
  static bool have[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  std::lock_guard<std::mutex> lk(mu);
  if (!have[dev]) {
    DevInfo d;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&d.minor, cudaDevAttrComputeCapabilityMinor, dev);
    cache[dev] = d;
    have[dev] = true;
  }
  return cache[dev];
}

bool valid_dt(int dt) { return dt >= FK_F32 && dt <= FK_F64; }
size_t elem_size(int dt) { return dt == FK_F32 ? 4 : dt == FK_F64 ? 8 : 2; }
bool is_lowp(int dt) { return dt == FK_BF16 || dt == FK_F16; }
size_t al256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr int64_t kMaxPoints = (int64_t(1) << 31) - 1;

bool shape_ok(int64_t B, int64_t N, int64_t K, int64_t d) {
  if (B < 1 || N < 1 || K < 1 || d < 1) return false;
  if (B * N > kMaxPoints) return false;  // flattened point index is int32
  if (B * K > (int64_t(1) << 30)) return false;
  if (K > (int64_t(1) << 30) || d > (int64_t(1) << 20)) return false;
  return true;
}

bool tc_path(int dt, int64_t d, const void* X, const void* C) {
  return is_lowp(dt) && fk::assign_tc_supported(d) && dev_info().major == 10 &&
         (reinterpret_cast<uintptr_t>(X) % 16 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
}

}  // namespace

extern "C" {

const char* fk_version(void) { return "flashkmeans-b200 0.1.0 (sm_100a)"; }

const char* fk_status_string(fk_status s) {
  switch (s) {
    case FK_OK: return "ok";
    case FK_EINVAL: return "invalid argument";
    case FK_EUNSUPPORTED: return "unsupported shape or device";
    case FK_ECUDA: return "CUDA error";
    case FK_EWORKSPACE: return "workspace too small";
  }
  return "unknown status";
}

const char* fk_last_cuda_error(void) { return g_last_cuda_error.c_str(); }

int fk_device_supported(int device) {
  int major = 0;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess)
    return 0;
  return major == 10 ? 1 : 0;
}

// Load every kernel of every translation unit on the current device now
// (cuModuleEnumerateFunctions + cuFuncLoad, CUDA >= 12.4), so the first call
// on a new shape -- a new head shape in the batched config
// -- pays no lazy module-loading time.  Idempotent per device.
fk_status fk_preload(void) {
  typedef CUresult (*GetModFn)(CUmodule*, CUfunction);
  typedef CUresult (*CountFn)(unsigned int*, CUmodule);
  typedef CUresult (*EnumFn)(CUfunction*, unsigned int, CUmodule);
  typedef CUresult (*LoadFn)(CUfunction);
  static std::mutex mu;
  static unsigned long long done_mask = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return FK_EUNSUPPORTED;
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 64 && (done_mask >> dev) & 1ull) return FK_OK;
  auto sym = [](const char* name) -> void* {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return f;
  };
  auto get_mod = (GetModFn)sym("cuFuncGetModule");
  auto count = (CountFn)sym("cuModuleGetFunctionCount");
  auto enumerate = (EnumFn)sym("cuModuleEnumerateFunctions");
  auto load = (LoadFn)sym("cuFuncLoad");
  if (!get_mod || !count || !enumerate || !load) return FK_EUNSUPPORTED;
  const void* anchors[] = {fk::module_anchor_assign_exact(), fk::module_anchor_assign_split(),
                           fk::module_anchor_assign_tc(),
                           fk::module_anchor_kmeanspp(), fk::module_anchor_select(),
                           fk::module_anchor_update()};
  for (const void* a : anchors) {
    cudaFunction_t f = nullptr;
    cudaError_t e = cudaGetFuncBySymbol(&f, a);
    if (e != cudaSuccess) return cuda_status(e);
    CUmodule mod = nullptr;
    unsigned int n = 0;
    if (get_mod(&mod, (CUfunction)f) != CUDA_SUCCESS || count(&n, mod) != CUDA_SUCCESS)
      return FK_ECUDA;
    std::vector<CUfunction> fs(n);
    if (n && enumerate(fs.data(), n, mod) != CUDA_SUCCESS) return FK_ECUDA;
    for (CUfunction fn : fs)
      if (load(fn) != CUDA_SUCCESS) return FK_ECUDA;
  }
  if (dev < 64) done_mask |= 1ull << dev;
  return FK_OK;
}

// ------------------------------------------------------------------ assign
namespace {
// f32/f64: the certified tensor-core path (fk_assign_split.cu) unless the
// problem is too small to pay for its ~7 launches (the exact CUDA-core mirror
// is then faster) or FK_ASSIGN_F32=mirror|split forces one.
int f32_path_env() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("FK_ASSIGN_F32");
    v = !e ? -1 : (e[0] == 'm' ? 0 : e[0] == 's' ? 1 : -1);
  }
  return v;
}
bool split_auto(int64_t B, int64_t N, int64_t K, int64_t d) {
  if (!fk::assign_split_supported(d) || dev_info().major != 10) return false;
  const int e = f32_path_env();
  if (e >= 0) return e == 1;
  return (double)B * N * K * d >= 6.7e7;  // ~20 us of the exact mirror
}
// X's split operand (B, N, 32 ns) bf16, then the reference's exact ||x||^2
// (B, N) in the data type: both fixed while X is.
size_t xsplit_x2_bytes(int64_t B, int64_t N, int64_t d) {
  return al256((size_t)B * N * 32 * fk::split_steps(d) * 2);
}
size_t xsplit_bytes(int dt, int64_t B, int64_t N, int64_t d) {
  return xsplit_x2_bytes(B, N, d) + al256((size_t)B * N * elem_size(dt));
}
fk_status build_xsplit(int dt, const void* X, int64_t B, int64_t N, int64_t d, uint8_t* xs,
                       int sms, cudaStream_t s) {
  fk_status st = cuda_status(fk::launch_split_rows(dt, X, B * N, d, xs, sms, s));
  if (st != FK_OK) return st;
  return cuda_status(fk::launch_row_norms_exact(dt, X, B * N, d, xs + xsplit_x2_bytes(B, N, d), s));
}
struct SplitWs {
  void *c2, *ext, *cn_ref, *xn_ref, *ct;
  unsigned int* cmax;
  int32_t *cnt, *list, *rec, *rec_cnt;
  int8_t* stat;
  float *est, *second;
  int rec_cap;
  size_t bytes;
};
SplitWs split_ws_layout(uint8_t* base, int dt, int64_t B, int64_t N, int64_t K, int64_t d) {
  const size_t es = elem_size(dt);
  const int kpad = fk::assign_tc_kpad(K);
  SplitWs w;
  size_t o = 0;
  auto take = [&](size_t n) { void* p = base ? base + o : nullptr; o += al256(n); return p; };
  w.c2 = take((size_t)B * K * 32 * fk::split_steps(d) * 2);
  w.ext = take((size_t)B * kpad * 32);
  w.cn_ref = take((size_t)B * K * es);
  w.ct = take((size_t)B * K * d * es);  // (B, d, K) transposed C: coalesced candidate columns
  w.cmax = (unsigned int*)take((size_t)B * 8 + 16);  // cmax (B), cnt (B), rec_cnt: one memset
  w.cnt = base ? (int32_t*)(w.cmax + B) : nullptr;
  w.rec_cnt = base ? (int32_t*)(w.cmax + 2 * B) : nullptr;
  const int64_t cap = B * N / 8 + 1024;  // beyond: full fallback
  w.rec_cap = (int)(cap < INT32_MAX ? cap : INT32_MAX);
  w.rec = (int32_t*)take((size_t)w.rec_cap * fk::kSplitRecInts * 4);
  w.stat = (int8_t*)take((size_t)B * N);
  w.est = (float*)take((size_t)B * N * 4);
  w.second = (float*)take((size_t)B * N * 4);
  w.list = (int32_t*)take((size_t)B * N * 4);
  w.bytes = o;
  return w;
}
size_t exact_ws_bytes(int dt, int64_t B, int64_t N, int64_t K) {
  const size_t es = elem_size(dt);
  return al256((size_t)B * N * es) + al256((size_t)B * K * es);
}

fk_status run_split(int dt, const void* X, const void* xsplit, const void* C, int64_t B, int64_t N,
                    int64_t K, int64_t d, int fast, int32_t* idx_out, void* mind_out,
                    const int32_t* idx_prev, int32_t* changed, uint8_t* ws, cudaStream_t s) {
  SplitWs w = split_ws_layout(ws, dt, B, N, K, d);
  w.xn_ref = const_cast<uint8_t*>(reinterpret_cast<const uint8_t*>(xsplit)) + xsplit_x2_bytes(B, N, d);
  const int kpad = fk::assign_tc_kpad(K);
  const DevInfo di = dev_info();
  fk_status st = cuda_status(cudaMemsetAsync(w.cmax, 0, (size_t)B * 8 + 16, s));
  if (st != FK_OK) return st;
  st = cuda_status(fk::launch_split_centroids(dt, C, B, K, d, kpad, w.c2, w.ext, w.cmax, w.ct, s));
  if (st != FK_OK) return st;
  st = cuda_status(fk::launch_row_norms_exact(dt, C, B * K, d, w.cn_ref, s));
  if (st != FK_OK) return st;
  st = cuda_status(fk::launch_assign_tc_split(xsplit, w.c2, w.ext, B, N, K, fk::split_steps(d),
                                              idx_out, w.est, w.second, w.cmax, w.stat, w.rec,
                                              w.rec_cnt, w.rec_cap, di.sms, s));
  if (st != FK_OK) return st;
  st = cuda_status(fk::launch_certify(dt, X, C, w.cn_ref, w.cmax, B, N, K, d, idx_out, w.est,
                                      w.second, w.stat, w.xn_ref, mind_out, idx_prev, changed,
                                      w.list, w.cnt, fast, s));
  if (st != FK_OK) return st;
  st = cuda_status(fk::launch_candidates(dt, X, w.ct, w.cn_ref, w.xn_ref, w.cmax, N, K, d, w.rec, w.rec_cnt,
                                         w.rec_cap, idx_out, mind_out, idx_prev, changed, di.sms, s));
  if (st != FK_OK) return st;
  return cuda_status(fk::launch_fallback_rows(dt, X, C, w.ct, w.cn_ref, w.xn_ref, w.cmax, B, N, K,
                                              d, w.list, w.cnt, idx_out, mind_out, idx_prev, changed,
                                              di.sms, s));
}
}  // namespace

size_t fk_assign_workspace(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d) {
  if (!valid_dt(dt) || B < 1 || N < 1 || K < 1) return 0;
  if (is_lowp(dt))  // ||c||^2 (fp32) + the bias-in-GEMM operand (16 x 16-bit per centroid)
    return al256((size_t)B * fk::assign_tc_kpad(K) * 4) + al256((size_t)B * fk::assign_tc_kpad(K) * 32);
  const size_t ex = exact_ws_bytes(dt, B, N, K);
  if (!split_auto(B, N, K, d)) return ex;
  const size_t sp = xsplit_bytes(dt, B, N, d) + split_ws_layout(nullptr, dt, B, N, K, d).bytes;
  return sp > ex ? sp : ex;
}

size_t fk_assign_xsplit_bytes(fk_dtype dt, int64_t B, int64_t N, int64_t d) {
  if ((dt != FK_F32 && dt != FK_F64) || B < 1 || N < 1 || !fk::assign_split_supported(d)) return 0;
  return xsplit_bytes(dt, B, N, d);
}

fk_status fk_assign_xsplit(fk_dtype dt, const void* X, int64_t B, int64_t N, int64_t d,
                           void* xsplit, void* stream) {
  if ((dt != FK_F32 && dt != FK_F64) || !X || !xsplit || !shape_ok(B, N, 1, d)) return FK_EINVAL;
  if (!fk::assign_split_supported(d)) return FK_EUNSUPPORTED;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return build_xsplit(dt, X, B, N, d, reinterpret_cast<uint8_t*>(xsplit), dev_info().sms,
                      reinterpret_cast<cudaStream_t>(stream));
}

fk_status fk_assign_split_fallback_rows(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d,
                                         const void* ws, int32_t* counts_host, void* stream) {
  if ((dt != FK_F32 && dt != FK_F64) || !ws || !counts_host || !shape_ok(B, N, K, d)) return FK_EINVAL;
  const SplitWs w = split_ws_layout(reinterpret_cast<uint8_t*>(const_cast<void*>(ws)), dt, B, N, K, d);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  fk_status st = cuda_status(cudaMemcpyAsync(counts_host, w.cnt, (size_t)B * 4, cudaMemcpyDeviceToHost, s));
  if (st != FK_OK) return st;
  return cuda_status(cudaStreamSynchronize(s));
}

size_t fk_assign_split_workspace(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d) {
  if ((dt != FK_F32 && dt != FK_F64) || B < 1 || N < 1 || K < 1 || d < 1) return 0;
  const size_t ex = exact_ws_bytes(dt, B, N, K);
  const size_t sp = split_ws_layout(nullptr, dt, B, N, K, d).bytes;
  return sp > ex ? sp : ex;
}

fk_status fk_assign_split(fk_dtype dt, const void* X, const void* xsplit, const void* C, int64_t B,
                          int64_t N, int64_t K, int64_t d, int32_t dot_mode, int32_t* idx_out,
                          void* mind_out, const int32_t* idx_prev, int32_t* changed_flag, void* ws,
                          size_t ws_bytes, void* stream) {
  if ((dt != FK_F32 && dt != FK_F64) || !shape_ok(B, N, K, d)) return FK_EINVAL;
  if (!X || !C || !idx_out || !mind_out || dot_mode < 0 || dot_mode > 2) return FK_EINVAL;
  if (idx_prev && !changed_flag) return FK_EINVAL;
  if (!ws || ws_bytes < fk_assign_split_workspace(dt, B, N, K, d)) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  if (dot_mode == FK_DOT_MIRROR || !fk::assign_split_supported(d)) {
    void* xn = w;
    void* cn = w + al256((size_t)B * N * elem_size(dt));
    fk_status st = cuda_status(fk::launch_row_norms_exact(dt, X, B * N, d, xn, s));
    if (st != FK_OK) return st;
    st = cuda_status(fk::launch_row_norms_exact(dt, C, B * K, d, cn, s));
    if (st != FK_OK) return st;
    return cuda_status(fk::launch_assign_exact(dt, X, C, xn, cn, B, N, K, d, idx_out, mind_out,
                                               idx_prev, changed_flag, s));
  }
  if (!xsplit) return FK_EINVAL;
  // FK_DOT_FAST: the certified path is already tensor-core speed, and a
  // tensor-core argmin left uncertified can differ from the reference where
  // two centroids sit closer than the estimate's error (same blob), which the
  // reference's fast mode (f64 reassociation only) never does: serve it exactly.
  static int nofb = -1;  // FK_SPLIT_NOFALLBACK=1: keep every estimate (measures the fallback's cost)
  if (nofb < 0) {
    const char* e = getenv("FK_SPLIT_NOFALLBACK");
    nofb = (e && e[0] == '1') ? 1 : 0;
  }
  return run_split(dt, X, xsplit, C, B, N, K, d, nofb, idx_out, mind_out, idx_prev, changed_flag,
                   w, s);
}

int64_t fk_assign_bias_rows(int64_t K) { return K < 1 ? 0 : fk::assign_tc_kpad(K); }

fk_status fk_assign_bias(fk_dtype dt, const void* C, int64_t B, int64_t K, int64_t d, void* bias_out,
                         void* stream) {
  if (!is_lowp(dt) || !C || !bias_out || B < 1 || K < 1 || d < 1) return FK_EINVAL;
  return cuda_status(fk::launch_cn_ext(dt, C, B, K, d, fk::assign_tc_kpad(K), bias_out,
                                       reinterpret_cast<cudaStream_t>(stream)));
}

static fk_status assign_impl(fk_dtype dt, const void* X, const void* C, const void* bias, int64_t B,
                             int64_t N, int64_t K, int64_t d, int32_t* idx_out, void* mind_out,
                             const int32_t* idx_prev, int32_t* changed_flag, void* ws, size_t ws_bytes,
                             void* stream, int32_t* hist_table, int32_t* hist_inval, int64_t hist_bpb,
                             int64_t hist_per, const float* xnorm = nullptr);

fk_status fk_assign(fk_dtype dt, const void* X, const void* C, const void* bias, int64_t B, int64_t N,
                    int64_t K, int64_t d, int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                    int32_t* changed_flag, void* ws, size_t ws_bytes, void* stream) {
  return assign_impl(dt, X, C, bias, B, N, K, d, idx_out, mind_out, idx_prev, changed_flag, ws, ws_bytes,
                     stream, nullptr, nullptr, 1, 1);
}

fk_status fk_assign_hist(fk_dtype dt, const void* X, const void* C, const void* bias, int64_t B,
                         int64_t N, int64_t K, int64_t d, int32_t* idx_out, void* mind_out,
                         const int32_t* idx_prev, int32_t* changed_flag, void* ws, size_t ws_bytes,
                         int32_t* hist_table, int32_t* hist_inval, int64_t hist_bpb, int64_t hist_per,
                         const float* xnorm, void* stream) {
  if (!hist_table || !hist_inval || hist_bpb < 1 || hist_per < 1 || hist_bpb * hist_per < N)
    return FK_EINVAL;
  if (!is_lowp(dt) || !tc_path(dt, d, X, C)) return FK_EUNSUPPORTED;
  return assign_impl(dt, X, C, bias, B, N, K, d, idx_out, mind_out, idx_prev, changed_flag, ws, ws_bytes,
                     stream, hist_table, hist_inval, hist_bpb, hist_per, xnorm);
}

fk_status fk_assign_row_norms(fk_dtype dt, const void* X, int64_t B, int64_t N, int64_t K, int64_t d,
                              float* out, void* stream) {
  if (!valid_dt(dt) || !shape_ok(B, N, K, d) || !X || !out) return FK_EINVAL;
  if (!is_lowp(dt) || !tc_path(dt, d, X, X)) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_row_norms_tc(dt == FK_BF16 ? 1 : 0, X, B, N, K, d, out,
                                             reinterpret_cast<cudaStream_t>(stream)));
}

static fk_status assign_impl(fk_dtype dt, const void* X, const void* C, const void* bias, int64_t B,
                             int64_t N, int64_t K, int64_t d, int32_t* idx_out, void* mind_out,
                             const int32_t* idx_prev, int32_t* changed_flag, void* ws, size_t ws_bytes,
                             void* stream, int32_t* hist_table, int32_t* hist_inval, int64_t hist_bpb,
                             int64_t hist_per, const float* xnorm) {
  if (!valid_dt(dt) || !shape_ok(B, N, K, d)) return FK_EINVAL;
  if (!X || !C || !idx_out || !mind_out) return FK_EINVAL;
  if (idx_prev && !changed_flag) return FK_EINVAL;
  const size_t need = fk_assign_workspace(dt, B, N, K, d);
  if (need > 0 && (!ws || ws_bytes < need)) return FK_EWORKSPACE;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const DevInfo di = dev_info();
  if (di.major != 10) return FK_EUNSUPPORTED;
  if (is_lowp(dt)) {
    float* cn = reinterpret_cast<float*>(ws);
    if (tc_path(dt, d, X, C)) {
      const int kpad = fk::assign_tc_kpad(K);
      const int fmt = dt == FK_BF16 ? 1 : 0;
      void* ext = nullptr;
      fk_status st;
      if (fk::assign_tc_uses_ext(fmt) && bias) {
        ext = const_cast<void*>(bias);  // precomputed by fk_normalize / fk_assign_bias
        st = FK_OK;
      } else if (fk::assign_tc_uses_ext(fmt)) {
        ext = reinterpret_cast<uint8_t*>(ws) + al256((size_t)B * kpad * 4);
        st = cuda_status(fk::launch_cn_ext(dt, C, B, K, d, kpad, ext, s));
      } else {
        st = cuda_status(fk::launch_cn_pad(dt, C, B, K, d, kpad, cn, s,
                                           fk::assign_tc_bias_mode(fmt) == 2 ? 0.5f : 1.0f));
      }
      if (st != FK_OK) return st;
      return cuda_status(fk::launch_assign_tc(fmt, X, C, cn, ext, B, N, K, d, idx_out,
                                              reinterpret_cast<float*>(mind_out), idx_prev,
                                              changed_flag, di.sms, s, hist_table, hist_inval, hist_bpb,
                                              hist_per, xnorm));
    }
    fk_status st = cuda_status(fk::launch_cn_pad(dt, C, B, K, d, (int)K, cn, s));
    if (st != FK_OK) return st;
    return cuda_status(fk::launch_assign_cuda_core_lowp(dt, X, C, cn, B, N, K, d, idx_out,
                                                        reinterpret_cast<float*>(mind_out),
                                                        idx_prev, changed_flag, s));
  }
  const size_t es = elem_size(dt);
  uint8_t* w = reinterpret_cast<uint8_t*>(ws);
  if (split_auto(B, N, K, d)) {  // X's split operand in the workspace, then the certified path
    fk_status st = build_xsplit(dt, X, B, N, d, w, di.sms, s);
    if (st != FK_OK) return st;
    return run_split(dt, X, w, C, B, N, K, d, 0, idx_out, mind_out, idx_prev, changed_flag,
                     w + xsplit_bytes(dt, B, N, d), s);
  }
  void* xn = w;
  void* cn = w + al256((size_t)B * N * es);
  fk_status st = cuda_status(fk::launch_row_norms_exact(dt, X, B * N, d, xn, s));
  if (st != FK_OK) return st;
  st = cuda_status(fk::launch_row_norms_exact(dt, C, B * K, d, cn, s));
  if (st != FK_OK) return st;
  return cuda_status(fk::launch_assign_exact(dt, X, C, xn, cn, B, N, K, d, idx_out, mind_out,
                                             idx_prev, changed_flag, s));
}

// ------------------------------------------------------------------ update
size_t fk_update_workspace(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d) {
  if (!valid_dt(dt) || B < 1 || N < 1 || K < 1 || d < 1) return 0;
  return fk::update_workspace_bytes(dt, B, N, K, d);
}

fk_status fk_update(fk_dtype dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                    int64_t K, int64_t d, int64_t update_chunk, int32_t accumulate, double* sums,
                    int64_t* counts, int64_t* merges_out, void* ws, size_t ws_bytes,
                    void* stream) {
  if (!valid_dt(dt) || !shape_ok(B, N, K, d)) return FK_EINVAL;
  if (!X || !ids || !sums || !counts || update_chunk < 1) return FK_EINVAL;
  const size_t need = fk_update_workspace(dt, B, N, K, d);
  if (!ws || ws_bytes < need) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_update(dt, X, ids, B, N, K, d, update_chunk, accumulate, sums,
                                       counts, merges_out, ws, dev_info().sms,
                                       reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_update_hist_slots(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d, void* ws,
                               int32_t** hist_table, int32_t** hist_inval, int64_t* hist_bpb,
                               int64_t* hist_per, int64_t* clear_words) {
  if (!valid_dt(dt) || !shape_ok(B, N, K, d) || !ws || !hist_table || !hist_inval || !hist_bpb ||
      !hist_per || !clear_words)
    return FK_EINVAL;
  if (!is_lowp(dt) || !fk::assign_tc_supported(d)) return FK_EUNSUPPORTED;  // no tensor-core assign to fold into
  return fk::update_hist_slots(dt, B, N, K, d, dev_info().sms, ws, hist_table, hist_inval, hist_bpb,
                               hist_per, clear_words)
             ? FK_OK
             : FK_EUNSUPPORTED;
}

fk_status fk_update_prehist(fk_dtype dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                            int64_t K, int64_t d, int64_t update_chunk, int32_t accumulate, double* sums,
                            int64_t* counts, int64_t* merges_out, void* ws, size_t ws_bytes,
                            void* stream) {
  if (!valid_dt(dt) || !shape_ok(B, N, K, d)) return FK_EINVAL;
  if (!X || !ids || !sums || !counts || update_chunk < 1) return FK_EINVAL;
  if (!is_lowp(dt)) return FK_EUNSUPPORTED;
  const size_t need = fk_update_workspace(dt, B, N, K, d);
  if (!ws || ws_bytes < need) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_update(dt, X, ids, B, N, K, d, update_chunk, accumulate, sums, counts,
                                       merges_out, ws, dev_info().sms,
                                       reinterpret_cast<cudaStream_t>(stream), 1));
}

fk_status fk_argsort(const int32_t* ids, int64_t B, int64_t N, int64_t K, int32_t* order_out,
                     int64_t* offsets_out, void* ws, size_t ws_bytes, void* stream) {
  if (!shape_ok(B, N, K, 1) || !ids || !order_out || !offsets_out) return FK_EINVAL;
  if (!ws || ws_bytes < fk_update_workspace(FK_F32, B, N, K, 1)) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_argsort(ids, B, N, K, order_out, offsets_out, ws, dev_info().sms,
                                        reinterpret_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------------ normalize
fk_status fk_normalize(fk_dtype master_dt, const double* sums, const int64_t* counts,
                       const void* prev, void* out, fk_dtype operand_dt, void* operand_out,
                       uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K, int64_t d,
                       void* bias_out, void* stream) {
  if (master_dt != FK_F32 && master_dt != FK_F64) return FK_EINVAL;
  if (operand_out && !valid_dt(operand_dt)) return FK_EINVAL;
  if (!sums || !counts || !prev || !out || B < 1 || K < 1 || d < 1) return FK_EINVAL;
  if (bias_out && !(operand_out && is_lowp(operand_dt))) return FK_EINVAL;
  return cuda_status(fk::launch_normalize(master_dt, sums, counts, prev, out, operand_dt,
                                          operand_out, empty_mask, max_shift2, B, K, d, bias_out,
                                          fk::assign_tc_kpad(K),
                                          reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_normalize_loop_tail(fk_dtype master_dt, const double* sums, const int64_t* counts,
                                 const void* prev, void* out, fk_dtype operand_dt, void* operand_out,
                                 uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K,
                                 int64_t d, void* bias_out, fk_dtype mind_dt, const void* mind,
                                 int64_t N, double* partials, double* objective, double* history,
                                 int64_t* history_row, int32_t* changed_flag, int64_t* merges,
                                 double* flags, uint32_t* counter, void* stream) {
  if (master_dt != FK_F32 && master_dt != FK_F64) return FK_EINVAL;
  if (operand_out && !valid_dt(operand_dt)) return FK_EINVAL;
  if (!sums || !counts || !prev || !out || !empty_mask || !max_shift2 || B < 1 || K < 1 || d < 1)
    return FK_EINVAL;
  if (bias_out && !(operand_out && is_lowp(operand_dt))) return FK_EINVAL;
  if (!valid_dt(mind_dt) || !mind || N < 1 || !partials || !objective || !changed_flag || !merges ||
      !flags || !counter || (history && !history_row))
    return FK_EINVAL;
  return cuda_status(fk::launch_normalize_tail(
      master_dt, sums, counts, prev, out, operand_dt, operand_out, empty_mask, max_shift2, B, K, d,
      bias_out, fk::assign_tc_kpad(K), mind_dt == FK_F64 ? 1 : 0, mind, N, partials, objective,
      history, history_row, changed_flag, merges, flags, counter, dev_info().sms,
      reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_objective_partials(fk_dtype mind_dt, const void* mind, int64_t B, int64_t N,
                                double* partials, void* stream) {
  if (!valid_dt(mind_dt) || !mind || !partials || B < 1 || N < 1) return FK_EINVAL;
  return cuda_status(fk::launch_objective_partials(mind_dt == FK_F64 ? 1 : 0, mind, B, N, partials,
                                                   reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_loop_tail(const double* partials, int64_t B, int64_t N, double* objective,
                       double* history, int64_t* history_row, int32_t* changed, double* max_shift2,
                       int64_t* merges, double* flags_out, void* stream) {
  if (!partials || !objective || !changed || !max_shift2 || !merges || !flags_out || B < 1 || N < 1)
    return FK_EINVAL;
  if (history && !history_row) return FK_EINVAL;
  return cuda_status(fk::launch_loop_tail(partials, B, N, objective, history, history_row, changed,
                                          max_shift2, merges, flags_out,
                                          reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_row_norms(fk_dtype dt, const void* M, int64_t rows, int64_t d, void* out,
                       void* stream) {
  if ((dt != FK_F32 && dt != FK_F64) || !M || !out || rows < 0 || d < 1) return FK_EINVAL;
  return cuda_status(
      fk::launch_row_norms_exact(dt, M, rows, d, out, reinterpret_cast<cudaStream_t>(stream)));
}

size_t fk_objective_workspace(int64_t B, int64_t N) {
  if (B < 1 || N < 1) return 0;
  return fk::objective_workspace_bytes(B, N);
}

fk_status fk_objective(fk_dtype mind_dt, const void* mind, int64_t B, int64_t N, double* out,
                       void* ws, size_t ws_bytes, void* stream) {
  if (!valid_dt(mind_dt) || !mind || !out || B < 1 || N < 1) return FK_EINVAL;
  if (!ws || ws_bytes < fk_objective_workspace(B, N)) return FK_EWORKSPACE;
  return cuda_status(fk::launch_objective(mind_dt == FK_F64 ? 1 : 0, mind, B, N, out, ws,
                                          reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_scatter(fk_dtype dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                     int64_t K, int64_t d, double* sums, int64_t* counts, void* stream) {
  if (!valid_dt(dt) || !shape_ok(B, N, K, d) || !X || !ids || !sums || !counts) return FK_EINVAL;
  return cuda_status(fk::launch_scatter(dt, X, ids, B, N, K, d, sums, counts,
                                        reinterpret_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------ multi-GPU exchange
fk_status fk_stats_pack(int32_t unpack, int64_t* counts, double* objective, int32_t* changed,
                        double* red, int64_t BK, int64_t B, void* stream) {
  if (!counts || !objective || !changed || !red || BK < 1 || B < 1) return FK_EINVAL;
  return cuda_status(fk::launch_stats_pack(unpack ? 1 : 0, counts, objective, changed, red, BK, B,
                                           reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_merges_from_counts(const int64_t* counts, int64_t B, int64_t K, int64_t update_chunk,
                                int64_t* merges, int32_t accumulate, void* stream) {
  if (!counts || !merges || B < 1 || K < 1 || update_chunk < 1) return FK_EINVAL;
  return cuda_status(fk::launch_merges_counts(counts, B, K, update_chunk, merges, accumulate ? 1 : 0,
                                              reinterpret_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------- reseed
size_t fk_farthest_workspace(int64_t B, int64_t E) {
  if (B < 1 || E < 1) return 0;
  return fk::farthest_workspace_bytes(B, E);
}

fk_status fk_farthest(fk_dtype mind_dt, const void* mind, int64_t B, int64_t N, int64_t E,
                      int64_t* idx_out, void* ws, size_t ws_bytes, void* stream) {
  if ((mind_dt != FK_F32 && mind_dt != FK_F64) || !mind || !idx_out || B < 1 || N < 1 || E < 1 ||
      E > N || N >= ((int64_t)1 << 32))
    return FK_EINVAL;
  if (E > 8192) return FK_EUNSUPPORTED;
  if (!ws || ws_bytes < fk_farthest_workspace(B, E)) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_farthest(mind_dt == FK_F64 ? 1 : 0, mind, B, N, E, idx_out, ws,
                                         dev_info().sms, reinterpret_cast<cudaStream_t>(stream)));
}

// ------------------------------------------------------------- k-means++
size_t fk_kmeanspp_workspace(int64_t B, int64_t N, int64_t K, int64_t d) {
  if (B < 1 || N < 1 || B * N > kMaxPoints || K < 0 || d < 0) return 0;
  return fk::kmeanspp_workspace_bytes(B, N, K, d);
}

fk_status fk_kmeanspp_init(int32_t* halted, int64_t B, int64_t N, int64_t K, void* ws,
                           size_t ws_bytes, void* stream) {
  if (!halted || B < 1 || N < 1 || K < 1 || K > N || B * N > kMaxPoints) return FK_EINVAL;
  if (!ws || ws_bytes < fk_kmeanspp_workspace(B, N, 0, 0)) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(
      fk::launch_kmeanspp_init(halted, ws, B, N, K, reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_kmeanspp_sweep(fk_dtype dt, const void* X, int64_t B, int64_t rows, int64_t d,
                            int64_t x_batch_stride, const void* centers, int64_t c_batch_stride,
                            double* min_d2, int64_t m_batch_stride, int32_t first,
                            const int32_t* halted, int64_t j, void* stream) {
  if (!valid_dt(dt) || !X || !centers || !min_d2 || B < 1 || rows < 0 || d < 1 ||
      d > (1 << 20) || (int64_t)d * 8 > 200 * 1024)
    return FK_EINVAL;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_kmeanspp_sweep(dt, X, B, rows, d, x_batch_stride, centers,
                                               c_batch_stride, nullptr, 0, 0, min_d2,
                                               m_batch_stride, first ? 1 : 0, halted, j,
                                               reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_kmeanspp_select(const double* min_d2, int64_t B, int64_t N, const double* u,
                             int64_t K, int64_t j, int64_t* idx, int32_t* halted, void* ws,
                             size_t ws_bytes, void* stream) {
  if (!min_d2 || !u || !idx || !halted || B < 1 || N < 1 || K < 2 || K > N || j < 1 || j >= K ||
      B * N > kMaxPoints)
    return FK_EINVAL;
  if (!ws || ws_bytes < fk_kmeanspp_workspace(B, N, 0, 0)) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_kmeanspp_select(min_d2, B, N, u, K, j, idx, halted, ws,
                                                reinterpret_cast<cudaStream_t>(stream)));
}

fk_status fk_kmeanspp(fk_dtype dt, const void* X, int64_t B, int64_t N, int64_t d, int64_t K,
                      const double* u, int64_t* idx, int32_t* halted, double* min_d2, void* ws,
                      size_t ws_bytes, void* stream) {
  if (!valid_dt(dt) || !X || !idx || !halted || !min_d2 || B < 1 || N < 1 || d < 1 || K < 1 ||
      K > N || B * N > kMaxPoints || d > (1 << 20) || (int64_t)d * 8 > 200 * 1024)
    return FK_EINVAL;
  if (K > 1 && !u) return FK_EINVAL;
  if (!ws || ws_bytes < fk_kmeanspp_workspace(B, N, K, d)) return FK_EWORKSPACE;
  if (dev_info().major != 10) return FK_EUNSUPPORTED;
  return cuda_status(fk::launch_kmeanspp(dt, X, B, N, d, K, u, idx, halted, min_d2, ws,
                                         reinterpret_cast<cudaStream_t>(stream)));
}

}  // extern "C"
