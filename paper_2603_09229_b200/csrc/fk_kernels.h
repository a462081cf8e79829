// fk_kernels.h -- internal launcher declarations shared by the .cu files.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace fk {

enum Dt { DT_F32 = 0, DT_BF16 = 1, DT_F16 = 2, DT_F64 = 3 };

// fk_assign_tc.cu
bool assign_tc_supported(int64_t d);
int assign_tc_kpad(int64_t K);
bool assign_tc_uses_ext(int fmt);
int assign_tc_bias_mode(int fmt);  // 0 epilogue, 1 bias-in-GEMM, 2 TMEM seed
cudaError_t launch_assign_tc(int fmt, const void* X, const void* C, const float* cn_pad,
                             const void* cn_ext, int64_t B, int64_t N, int64_t K, int64_t d,
                             int32_t* idx_out, float* mind_out, const int32_t* idx_prev,
                             int32_t* changed, int num_sms, cudaStream_t stream,
                             int32_t* hist_tab = nullptr, int32_t* hist_inval = nullptr,
                             int64_t hist_bpb = 1, int64_t hist_per = 1,
                             const float* xn_in = nullptr);
cudaError_t launch_row_norms_tc(int fmt, const void* X, int64_t B, int64_t N, int64_t K, int64_t d,
                                float* out, cudaStream_t stream);

constexpr int kSplitRecInts = 10;  // fk_assign_tc.cu FK_SPLIT_REC: [row, n, up to 8 chunk bases]
cudaError_t launch_assign_tc_split(const void* X2, const void* C2, const void* ext, int64_t B,
                                   int64_t N, int64_t K, int ns, int32_t* idx_out, float* est_out,
                                   float* second_out, const unsigned int* cmax, int8_t* stat_out,
                                   int32_t* cand_rec, int32_t* cand_cnt, int cand_cap, int num_sms,
                                   cudaStream_t stream);

// fk_assign_exact.cu
cudaError_t launch_cn_pad(int dt, const void* C, int64_t B, int64_t K, int64_t d, int kpad,
                          float* cn_pad, cudaStream_t stream, float scale = 1.0f);
// (B, kpad, 16) operand [hi, mid, lo, 0...] of ||c||^2 / 2 (+inf beyond K)
cudaError_t launch_cn_ext(int dt, const void* C, int64_t B, int64_t K, int64_t d, int kpad,
                          void* out, cudaStream_t stream);
cudaError_t launch_row_norms_exact(int dt, const void* M, int64_t rows, int64_t d, void* out,
                                   cudaStream_t stream);
cudaError_t launch_assign_exact(int dt, const void* X, const void* C, const void* xn,
                                const void* cn, int64_t B, int64_t N, int64_t K, int64_t d,
                                int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                                int32_t* changed, cudaStream_t stream);
cudaError_t launch_assign_exact_rows(int dt, const void* X, const void* C, const void* xn,
                                     const void* cn, int64_t B, int64_t N, int64_t K, int64_t d,
                                     const int32_t* list, const int32_t* list_cnt,
                                     int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                                     int32_t* changed, cudaStream_t stream);

// fk_assign_split.cu
bool assign_split_supported(int64_t d);
int split_steps(int64_t d);
cudaError_t launch_split_rows(int dt, const void* M, int64_t rows, int64_t d, void* out,
                              int num_sms, cudaStream_t s);
cudaError_t launch_split_centroids(int dt, const void* C, int64_t B, int64_t K, int64_t d,
                                   int kpad, void* c2, void* ext, unsigned int* cmax, void* ct,
                                   cudaStream_t s);
cudaError_t launch_fallback_rows(int dt, const void* X, const void* C, const void* ct,
                                 const void* cn, const void* xn_ref, const unsigned int* cmax,
                                 int64_t B, int64_t N, int64_t K, int64_t d, const int32_t* list,
                                 const int32_t* list_cnt, int32_t* idx_out, void* mind_out,
                                 const int32_t* idx_prev, int32_t* changed, int num_sms,
                                 cudaStream_t s);
cudaError_t launch_certify(int dt, const void* X, const void* C, const void* cn_ref,
                           const unsigned int* cmax, int64_t B, int64_t N, int64_t K, int64_t d,
                           const int32_t* ids, const float* est, const float* second,
                           const int8_t* stat, const void* xn_in, void* mind_out,
                           const int32_t* idx_prev, int32_t* changed, int32_t* list,
                           int32_t* list_cnt, int fast, cudaStream_t s);
cudaError_t launch_candidates(int dt, const void* X, const void* ct, const void* cn_ref,
                              const void* xn_ref, const unsigned int* cmax, int64_t N, int64_t K,
                              int64_t d,
                              const int32_t* rec, const int32_t* rec_cnt, int rec_cap,
                              int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                              int32_t* changed, int num_sms, cudaStream_t s);
cudaError_t launch_assign_cuda_core_lowp(int dt, const void* X, const void* C, const float* cn,
                                         int64_t B, int64_t N, int64_t K, int64_t d,
                                         int32_t* idx_out, float* mind_out,
                                         const int32_t* idx_prev, int32_t* changed,
                                         cudaStream_t stream);

// fk_update.cu
size_t update_workspace_bytes(int dt, int64_t B, int64_t N, int64_t K, int64_t d);
cudaError_t launch_update(int dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                          int64_t K, int64_t d, int64_t chunk, int accumulate, double* sums,
                          int64_t* counts, int64_t* merges, void* ws, int num_sms,
                          cudaStream_t stream, int prehist = 0);
bool update_hist_slots(int dt, int64_t B, int64_t N, int64_t K, int64_t d, int num_sms, void* ws,
                       int32_t** table, int32_t** inval, int64_t* bpb, int64_t* per, int64_t* words);
cudaError_t launch_argsort(const int32_t* ids, int64_t B, int64_t N, int64_t K, int32_t* order_out,
                           int64_t* off_out, void* ws, int num_sms, cudaStream_t stream);
cudaError_t launch_normalize(int master_dt, const double* sums, const int64_t* counts,
                             const void* prev, void* out, int operand_dt, void* operand_out,
                             uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K,
                             int64_t d, void* bias_out, int64_t bias_kpad, cudaStream_t stream);
cudaError_t launch_normalize_tail(int master_dt, const double* sums, const int64_t* counts,
                                  const void* prev, void* out, int operand_dt, void* operand_out,
                                  uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K,
                                  int64_t d, void* bias_out, int64_t bias_kpad, int mind_f64,
                                  const void* mind, int64_t N, double* part, double* obj,
                                  double* hist, int64_t* hist_it, int32_t* changed,
                                  int64_t* merges, double* flags, unsigned int* counter,
                                  int num_sms, cudaStream_t s);
cudaError_t launch_objective_partials(int mind_is_f64, const void* mind, int64_t B, int64_t N,
                                      double* part, cudaStream_t s);
cudaError_t launch_loop_tail(const double* part, int64_t B, int64_t N, double* obj, double* hist,
                             int64_t* hist_it, int32_t* changed, double* shift2, int64_t* merges,
                             double* flags, cudaStream_t s);
size_t objective_workspace_bytes(int64_t B, int64_t N);
cudaError_t launch_objective(int mind_is_f64, const void* mind, int64_t B, int64_t N, double* out,
                             void* ws, cudaStream_t stream);
cudaError_t launch_scatter(int dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                           int64_t K, int64_t d, double* sums, int64_t* counts,
                           cudaStream_t stream);

cudaError_t launch_stats_pack(int unpack, int64_t* counts, double* obj, int32_t* changed,
                              double* red, int64_t BK, int64_t B, cudaStream_t s);
cudaError_t launch_merges_counts(const int64_t* counts, int64_t B, int64_t K, int64_t chunk,
                                 int64_t* merges, int accumulate, cudaStream_t s);

// fk_select.cu
size_t farthest_workspace_bytes(int64_t B, int64_t E);
cudaError_t launch_farthest(int mind_is_f64, const void* mind, int64_t B, int64_t N, int64_t E,
                            int64_t* idx_out, void* ws, int num_sms, cudaStream_t s);

// fk_kmeanspp.cu
size_t pairwise_total_workspace(int64_t B, int64_t N);
cudaError_t launch_pairwise_total(const double* m, int64_t B, int64_t N, double* out, void* ws,
                                  cudaStream_t s);
size_t kmeanspp_workspace_bytes(int64_t B, int64_t N, int64_t K, int64_t d);
cudaError_t launch_kmeanspp_init(int32_t* halted, void* ws, int64_t B, int64_t N, int64_t K,
                                 cudaStream_t s);
cudaError_t launch_kmeanspp_sweep(int dt, const void* X, int64_t B, int64_t rows, int64_t d,
                                  int64_t x_sb, const void* cen, int64_t cen_sb,
                                  const int64_t* idx, int64_t K, int64_t col, double* m,
                                  int64_t m_sb, int first, const int32_t* halted, int64_t j,
                                  cudaStream_t s);
cudaError_t launch_kmeanspp_select(const double* m, int64_t B, int64_t N, const double* u,
                                   int64_t K, int64_t j, int64_t* idx, int32_t* halted, void* ws,
                                   cudaStream_t s);
cudaError_t launch_kmeanspp(int dt, const void* X, int64_t B, int64_t N, int64_t d, int64_t K,
                            const double* u, int64_t* idx, int32_t* halted, double* m, void* ws,
                            cudaStream_t s);

// FK_MODULE_ANCHOR of each translation unit (fk_preload)
const void* module_anchor_assign_exact();
const void* module_anchor_assign_split();
const void* module_anchor_assign_tc();
const void* module_anchor_kmeanspp();
const void* module_anchor_select();
const void* module_anchor_update();

}  // namespace fk
