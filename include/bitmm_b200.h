/*
 * bitmm_b200 — C ABI of the B200 (sm_100a) bitwise-GEMM hot path.
 *
 * Drop-in boundary for the reference's kernel layer (namespace bitmm in
 * /root/reference/proj/include/bitmm/kernels.hpp and apb.hpp). Every entry point
 * takes plain pointers and sizes in the reference's own packed layouts:
 *
 *   BitMatrix (tensor.hpp:59-112): rows x wpr uint64 words, row-major; element i
 *     of a row is bit (i % 64) of word (i / 64); bit 1 decodes to +1, bit 0 to -1;
 *     wpr >= ceil(cols / 64) and every padding bit is zero.
 *   ThmPlanes (tensor.hpp:134-145): three BitMatrix payloads t, h, m of equal shape
 *     plus scale and optional gamma (has_gamma = 0 means std::nullopt).
 *   DenseMatrix (tensor.hpp:123-154): rows x cols float, row-major.
 *   CsrMatrix (tensor.hpp:115-128): row_ptr[rows+1], col_idx[nnz] (uint64), vals[nnz].
 *
 * "b_packed" / "a_packed" operands are packed along K per OUTPUT COLUMN, exactly as
 * the reference (kernels.hpp:44-46): row c of the packed operand is column c of the
 * logical K x N operand. Outputs are row-major with leading dimension ldc.
 *
 * Two flavours per routine:
 *   *_dev  : device pointers, stream-ordered on `stream` (a cudaStream_t, may be 0);
 *            operand-encoding errors detected on the device are latched and reported
 *            by bitmm_device_status().
 *   *_host : host pointers; copies in, computes, copies out and synchronises. This is
 *            the flavour a reference DenseMatrix-returning wrapper calls.
 *
 * Error codes mirror the reference's exception types:
 *   BITMM_ERR_INVALID_ARGUMENT  <-> std::invalid_argument (kernels.cpp:52, 70-73, 115-118,
 *                                    165-166, 187-188, 226-227, 301, 335-338; tensor.cpp:74)
 *   BITMM_ERR_INVALID_ENCODING  <-> bitmm::InvalidEncoding (tensor.cpp:133-153)
 * bitmm_last_error() returns the message of the most recent failure on this thread.
 *
 * There is no CPU fallback: without a CUDA device every compute entry point
 * returns BITMM_ERR_NO_DEVICE.
 */
#ifndef BITMM_B200_H
#define BITMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  BITMM_OK = 0,
  BITMM_ERR_INVALID_ARGUMENT = 1,
  BITMM_ERR_INVALID_ENCODING = 2,
  BITMM_ERR_CUDA = 3,
  BITMM_ERR_NO_DEVICE = 4,
  BITMM_ERR_IO = 5 /* ≙ bitmm::IoError (errors.hpp:14): container format / file errors */
};

/* Shared-dimension cap (tensor.hpp:21, kMaxSharedDim = 2^20). */
#define BITMM_MAX_SHARED_DIM (INT64_C(1) << 20)

int bitmm_abi_version(void);
const char* bitmm_last_error(void);
/* Number of SMs of the current device, or 0 if no device. */
int bitmm_device_sm_count(void);
/* Synchronises `stream`, returns and clears the latched device-side encoding status. */
int bitmm_device_status(void* stream);
/* Pre-grows the internal device workspace so no allocation happens inside timed loops. */
int bitmm_reserve_workspace(size_t bytes);
/* Workspace bytes a routine needs for the given shape (routine: 0=1x1, 1=1x2, 2=2x2, 3=1x32/APB,
 * 4=APB with 2-bit activations; m = rows, n = tokens, k = cols). */
size_t bitmm_workspace_bytes(int routine, int64_t m, int64_t n, int64_t k);
/* Number of kernels launched by the most recent compute call on this thread. */
int bitmm_last_launch_count(void);
/* Device -> host bytes copied by the most recent *_host GEMM call on this thread. The
 * 1/1, 1/2 and 2/2 host calls with >= 32 MB of output move it as one 16-bit word per cell (the integer
 * units narrowed on the device, widened and scaled on the host into the caller's int32 /
 * fp32 buffers, bit-identical) whenever K allows: 1/1 K <= 65535, 1/2 K <= 10922,
 * 2/2 K <= 7281. BITMM_HOST_WIRE=32 in the environment forces the 4-byte copies. */
uint64_t bitmm_last_d2h_bytes(void);

/* Stream-ordered kernel timing (used by bench.py for the roofline): while enabled, every
 * kernel the library launches is bracketed by CUDA events on its launching stream.
 * bitmm_profile_collect() synchronises those events and folds them into per-kernel totals
 * readable by index; bitmm_profile_reset() clears them. */
int bitmm_profile_enable(int on);
int bitmm_profile_collect(void);
int bitmm_profile_reset(void);
int bitmm_profile_kernel_count(void);
const char* bitmm_profile_kernel_name(int i);
int bitmm_profile_kernel_launches(int i);
double bitmm_profile_kernel_ms(int i);

/* ---- Multi-GPU N-shard gather over NVLink ----
 * CUDA IPC export / import of a device allocation, so every rank's GEMM epilogue stores its
 * output column block straight into the root rank's M x N matrix (peer memory over NVLink):
 * the gather IS the epilogue, overlapped with the MMAs tile by tile, and no collective runs
 * after the compute. get_handle writes a 64-byte handle plus the byte offset of dev_ptr inside
 * its allocation; open maps a peer's handle and returns the allocation's base (add the
 * offset); close unmaps it. A GEMM output that lives on another device is written by the
 * epilogue's st.global path (TMA stores stay for local outputs). */
int bitmm_ipc_get_handle(const void* dev_ptr, void* handle, uint64_t* offset);
int bitmm_ipc_open(const void* handle, void** dev_ptr);
int bitmm_ipc_close(void* dev_ptr);

/* ---- Single-process multi-GPU 1/1 (N sharded over the GPUs) ----
 * A plan owns, on each of `ndev` devices (devs[0] is the root), the replicated A operand (m x wpr
 * words), the device's block of b_packed rows (output columns split into ndev blocks of whole
 * 32-column groups) and its output space, plus the root's m x n int32 matrix. upload copies the
 * host operands (A to every device, each device its b_packed rows); run computes every block
 * on its own device and brings it to the root:
 *   BITMM_GATHER_NONE : blocks stay on their devices (kernel-only timing);
 *   BITMM_GATHER_PEER : every device's GEMM epilogue stores its block straight into the root's
 *                       matrix through peer memory (NVLink): the gather is the epilogue;
 *   BITMM_GATHER_NCCL : blocks computed locally, then NCCL send/recv to the root (one group),
 *                       which lays them out at their columns (libnccl.so.2 loaded at run time;
 *                       needs distinct devices).
 * *ms_out = the device-timed run (max over devices; the root's time includes the gather).
 * download copies rows [row0, row0 + rows) of the root's matrix (units, K - 2 popcount) to host
 * memory. A device may be
 * listed more than once (blocks run one after another on it; no NCCL then). A plan is used by
 * one host thread at a time; different plans are independent. */
enum { BITMM_GATHER_NONE = 0, BITMM_GATHER_PEER = 1, BITMM_GATHER_NCCL = 2 };
int bitmm_shard_plan_create(const int* devs, int ndev, int64_t m, int64_t n, int64_t k, int64_t wpr,
                            void** plan);
int bitmm_shard_plan_upload(void* plan, const uint64_t* a, const uint64_t* b_packed);
int bitmm_shard_run(void* plan, int gather, double* ms_out);
int bitmm_shard_download(void* plan, int64_t row0, int64_t rows, int32_t* c, int64_t ldc);
int bitmm_shard_plan_destroy(void* plan);

/* ---- 1/1: replaces gemm_1x1 (kernels.hpp:47-48, kernels.cpp:163-183) ----
 * C[r][c] = (gamma_a * gamma_b) * float(K - 2*popcount(a_r xor b_c)).
 * Writes int32 units to c_units and/or scaled floats to c (either may be NULL). */
int bitmm_gemm_1x1_dev(const uint64_t* a, int64_t m, const uint64_t* b_packed, int64_t n, int64_t k,
                       int64_t wpr, float gamma_a, float gamma_b, int32_t* c_units, float* c,
                       int64_t ldc, void* stream);
int bitmm_gemm_1x1_host(const uint64_t* a, int64_t m, const uint64_t* b_packed, int64_t n,
                        int64_t k, int64_t wpr, float gamma_a, float gamma_b, int32_t* c_units,
                        float* c, int64_t ldc);
/* Same contract, evaluated by the CUDA-core LOP3+POPC kernel (measured alternative). */
int bitmm_gemm_1x1_popc_dev(const uint64_t* a, int64_t m, const uint64_t* b_packed, int64_t n,
                            int64_t k, int64_t wpr, float gamma_a, float gamma_b,
                            int32_t* c_units, float* c, int64_t ldc, void* stream);

/* ---- 1/2: replaces gemm_1x2 (kernels.hpp:55, kernels.cpp:185-221) ----
 * w: m x wpr binary rows; planes t/h/mm: n x wpr, packed along K per output column.
 * units = 2 * sum_k sign(w[r][k]) * p[c][k]; scale = 0.5f*gamma*a_scale*(a_gamma or 1)
 * (kernels.cpp:193). Optional per-row (row_scale[m]) and per-column (col_scale[n])
 * multipliers extend the scalar: C = ((scale*row_scale[r])*col_scale[c]) * float(units). */
int bitmm_gemm_1x2_dev(const uint64_t* w, int64_t m, float gamma, const uint64_t* t,
                       const uint64_t* h, const uint64_t* mm, int64_t n, int64_t k, int64_t wpr,
                       float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                       const float* col_scale, int32_t* c_units, float* c, int64_t ldc,
                       void* stream);
int bitmm_gemm_1x2_host(const uint64_t* w, int64_t m, float gamma, const uint64_t* t,
                        const uint64_t* h, const uint64_t* mm, int64_t n, int64_t k, int64_t wpr,
                        float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                        const float* col_scale, int32_t* c_units, float* c, int64_t ldc);

/* ---- 2/2: replaces gemm_2x2 (kernels.hpp:62, kernels.cpp:223-275) ----
 * units = 4 * sum_k p_w[r][k] * p_a[c][k];
 * scale = 0.25f*w_scale*a_scale*(w_gamma or 1)*(a_gamma or 1) (kernels.cpp:232-233). */
int bitmm_gemm_2x2_dev(const uint64_t* wt, const uint64_t* wh, const uint64_t* wm, int64_t m,
                       float w_scale, int has_w_gamma, float w_gamma, const uint64_t* at,
                       const uint64_t* ah, const uint64_t* am, int64_t n, int64_t k, int64_t wpr,
                       float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                       const float* col_scale, int32_t* c_units, float* c, int64_t ldc,
                       void* stream);
int bitmm_gemm_2x2_host(const uint64_t* wt, const uint64_t* wh, const uint64_t* wm, int64_t m,
                        float w_scale, int has_w_gamma, float w_gamma, const uint64_t* at,
                        const uint64_t* ah, const uint64_t* am, int64_t n, int64_t k, int64_t wpr,
                        float a_scale, int has_a_gamma, float a_gamma, const float* row_scale,
                        const float* col_scale, int32_t* c_units, float* c, int64_t ldc);

/* ---- 1/32 binary x fp32: replaces gemm_1x32_ref (kernels.hpp:73, kernels.cpp:300-332) ----
 * C[r][c] = gamma_r * sum_k sign(w[r][k]) * b[k][c], gamma_r = row_gamma ? row_gamma[r] : gamma.
 * b is K x n fp32 row-major with leading dimension ldb. */
int bitmm_gemm_1x32_dev(const uint64_t* w, int64_t m, int64_t k, int64_t wpr, float gamma,
                        const float* row_gamma, const float* b, int64_t n, int64_t ldb, float* c,
                        int64_t ldc, void* stream);
int bitmm_gemm_1x32_host(const uint64_t* w, int64_t m, int64_t k, int64_t wpr, float gamma,
                         const float* row_gamma, const float* b, int64_t n, int64_t ldb, float* c,
                         int64_t ldc);

/* ---- sparse x dense: replaces spmm_csr (kernels.hpp:76, kernels.cpp:334-352) ---- */
int bitmm_spmm_csr_dev(int64_t rows, int64_t cols, const uint64_t* row_ptr, const uint64_t* col_idx,
                       const float* vals, const float* b, int64_t n, int64_t ldb, float* c,
                       int64_t ldc, void* stream);
int bitmm_spmm_csr_host(int64_t rows, int64_t cols, const uint64_t* row_ptr,
                        const uint64_t* col_idx, const float* vals, int64_t nnz, const float* b,
                        int64_t n, int64_t ldb, float* c, int64_t ldc);

/* ---- APB layer forward: replaces layer_forward (apb.hpp:65, apb.cpp:158-164) ----
 * C = alpha_r * (sign(bin) . b) + residual . b, fused in one GEMM epilogue.
 * alpha_r = row_alpha ? row_alpha[r] : alpha (the reference ApbLayer holds a scalar alpha,
 * apb.hpp:48). bin: rows x wpr; residual CSR over rows x cols; b: cols x n fp32. */
int bitmm_layer_forward_dev(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                            const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                            const uint64_t* col_idx, const float* vals, const float* b, int64_t n,
                            int64_t ldb, float* c, int64_t ldc, void* stream);
int bitmm_layer_forward_host(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                             const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                             const uint64_t* col_idx, const float* vals, int64_t nnz,
                             const float* b, int64_t n, int64_t ldb, float* c, int64_t ldc);

/* ---- GEMM group: several routines in one launch pair ----
 * Runs up to 4 GEMM problems (an item that asks for both c_units and c counts as two) as ONE
 * operand-expansion launch plus ONE persistent tensor-core launch over the concatenated tiles,
 * so a batch of independent GEMMs pays one ramp-up and one tail instead of one per GEMM. Each
 * item has exactly the semantics (scales, errors, outputs) of the matching bitmm_gemm_*_dev
 * call; results are bit-identical to issuing those calls one by one. Stream-ordered. */
enum { BITMM_ROUTINE_1X1 = 0, BITMM_ROUTINE_1X2 = 1, BITMM_ROUTINE_2X2 = 2 };
typedef struct bitmm_gemm_item {
  int routine;                /* BITMM_ROUTINE_* */
  const uint64_t* a0;         /* 1x1: a; 1x2: w (binary weights); 2x2: weight plane t */
  const uint64_t* a1;         /* 2x2: weight plane h */
  const uint64_t* a2;         /* 2x2: weight plane m */
  const uint64_t* b0;         /* 1x1: b_packed; 1x2 / 2x2: activation plane t */
  const uint64_t* b1;         /* 1x2 / 2x2: activation plane h */
  const uint64_t* b2;         /* 1x2 / 2x2: activation plane m */
  int64_t m, n, k, wpr;
  float a_scale;              /* 1x1: gamma_a; 1x2: gamma; 2x2: weight plane scale */
  int has_a_gamma;            /* 2x2: weight plane gamma present */
  float a_gamma;
  float b_scale;              /* 1x1: gamma_b; 1x2 / 2x2: activation plane scale */
  int has_b_gamma;            /* 1x2 / 2x2: activation plane gamma present */
  float b_gamma;
  const float* row_scale;     /* optional [m] (1x2, 2x2), as in the _dev calls */
  const float* col_scale;     /* optional [n] (1x2, 2x2) */
  int32_t* c_units;           /* optional [m][ldc] */
  float* c;                   /* optional [m][ldc] */
  int64_t ldc;
} bitmm_gemm_item;
int bitmm_gemm_batch_dev(const bitmm_gemm_item* items, int count, void* stream);

/* ---- GEMM group, host flavour ----
 * The *_host calls of up to 4 items (host pointers in a0..b2, the optional row / column scales,
 * host outputs c_units / c with leading dimension ldc), with the same results. When every output
 * crosses PCIe on the 16-bit wire (>= 32 MB and K within the wire's bounds), the items' pipelines
 * run as one: every item's input copies first, then the slices of all items back to back, so the
 * device -> host link stays busy across items (one ramp-up and one tail instead of one per call).
 * Otherwise the items run one after the other. An error stops the batch; outputs of items not
 * yet completed are then unspecified. BITMM_HOST_BATCH=0 always runs them one after the other. */
int bitmm_gemm_batch_host(const bitmm_gemm_item* items, int count);

/* ---- Late-output host call: the drop-in's per-call latency (gemm_1x1 / 1x2 / 2x2 returning a
 * fresh DenseMatrix, kernels.cpp:163-275) ----
 * The *_host call of one item (host pointers in a0..b2 and the optional row / column scales;
 * its c_units, c and ldc are ignored) whose output buffers are supplied AFTER the call's copies
 * and kernels are enqueued: the library calls out_fn(user, &out) once, while the device works,
 * and writes the result into out.c_units and / or out.c (row-major, out.ldc >= n; preset to n)
 * as `want` asks. A reference wrapper constructs its zero-filled DenseMatrix inside out_fn, so
 * the allocation overlaps the GEMM instead of preceding it. out_fn is not called when the call
 * fails before anything is enqueued; a non-zero return from it fails the call with
 * BITMM_ERR_INVALID_ARGUMENT. A device-detected error (encoding, padding) is reported before
 * any output byte is written. Results are identical to the matching *_host call. */
enum { BITMM_WANT_UNITS = 1, BITMM_WANT_C = 2 };
typedef struct bitmm_host_out {
  int32_t* c_units;
  float* c;
  int64_t ldc;
} bitmm_host_out;
typedef int (*bitmm_out_fn)(void* user, bitmm_host_out* out);
int bitmm_gemm_host_late(const bitmm_gemm_item* item, int want, bitmm_out_fn out_fn, void* user);

/* ---- Row ops, batched (kernels.hpp:29-38, kernels.cpp:120-140) ----
 * count independent row pairs of `words` u64 each, rows contiguous:
 *   dot_binary: out[r] = n - 2*popc(u_r ^ v_r)   (n: logical length, words_for(n) <= words)
 *   mbm:        out[r] = popc(z_r) - 2*popc((x_r ^ y_r) & z_r)
 * Stream-ordered; the per-row reference calls stay on the host (one launch per row would cost
 * more than the popcounts). */
int bitmm_dot_binary_dev(const uint64_t* u, const uint64_t* v, int64_t count, int64_t words,
                         int64_t n, int64_t* out, void* stream);
int bitmm_mbm_dev(const uint64_t* x, const uint64_t* y, const uint64_t* z, int64_t count,
                  int64_t words, int64_t* out, void* stream);
/* Host flavour of the same (host rows in, host results out, synchronous): what a drop-in
 * dot_binary / mbm binding calls with count = 1 (integration/reference_dropin, built with
 * BITMM_DROPIN_ROWOPS_GPU). */
int bitmm_dot_binary_host(const uint64_t* u, const uint64_t* v, int64_t count, int64_t words,
                          int64_t n, int64_t* out);
int bitmm_mbm_host(const uint64_t* x, const uint64_t* y, const uint64_t* z, int64_t count,
                   int64_t words, int64_t* out);

/* ---- ThmPlanes::validate on device (tensor.cpp:133-153) ----
 * Checks scale > 0, zero padding and legal {t,h,m} states of plane words already on the
 * device; returns BITMM_ERR_INVALID_ENCODING with the reference's message (same precedence:
 * scale, padding, then the first illegal word in row-major order). Synchronous. */
int bitmm_validate_planes_dev(const uint64_t* t, const uint64_t* h, const uint64_t* m,
                              int64_t rows, int64_t cols, int64_t wpr, float scale, void* stream);

/* ---- BTSR container -> device (tensor_io.hpp:14-37, tensor_io.cpp:139-215) ----
 * BTSR v1: magic "BTSR" | version u32 | kind u8 (0 dense, 1 bit, 2 csr) | rows u64 | cols u64 |
 * payload (dense: f32[rows*cols]; bit: wpr u64, u64[rows*wpr]; csr: nnz u64,
 * row_ptr u64[rows+1], col_idx u64[nnz], vals f32[nnz]), little-endian.
 * bitmm_btsr_read_header validates the header and the file size (no GPU needed).
 * bitmm_btsr_load_dev streams the payload into caller-allocated device buffers through pinned
 * chunks on `stream` and applies the reference's object checks on the way (BitMatrix padding,
 * CsrMatrix::validate, finite dense values). expected_kind -1 accepts any kind, else a
 * mismatch fails like load_dense/load_bit/load_csr ("expected bit tensor: <path>").
 * dense -> payload f32[rows*cols]; bit -> payload u64[rows*wpr]; csr -> row_ptr / col_idx /
 * vals. Failures return BITMM_ERR_IO with the reference's IoError text. */
typedef struct bitmm_btsr_header {
  int kind;
  int64_t rows, cols;
  int64_t words_per_row; /* bit */
  int64_t nnz;           /* csr */
} bitmm_btsr_header;
int bitmm_btsr_read_header(const char* path, bitmm_btsr_header* out);
int bitmm_btsr_load_dev(const char* path, int expected_kind, void* payload, uint64_t* row_ptr,
                        uint64_t* col_idx, float* vals, void* stream);

/* ---- APB layer with 2-bit activations (paper-faithful inference) ----
 * No single reference entry point: it is the composition of reference calls
 *   C = gemm_1x2(bin, alpha_r, planes)            (kernels.hpp:55, kernels.cpp:185-221)
 *     + spmm_csr(residual, D)                      (kernels.hpp:76, kernels.cpp:334-352)
 * added like layer_forward (apb.cpp:161-162), where planes {t,h,m} are tokens x wpr (K-packed
 * per token, gemm_1x2's a_packed) and D[k][c] = float(p[c][k]) * (a_scale * gamma_a) is the
 * dequantized level. Per-row alpha uses gemm_1x2's scale order ((0.5*alpha_r)*s)*gamma_a.
 * C: rows x tokens. Bit-identical to that composition. */
int bitmm_layer_forward_2bit_dev(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                                 const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                                 const uint64_t* col_idx, const float* vals, const uint64_t* t,
                                 const uint64_t* h, const uint64_t* m, int64_t tokens,
                                 float a_scale, int has_a_gamma, float a_gamma, float* c,
                                 int64_t ldc, void* stream);
int bitmm_layer_forward_2bit_host(int64_t rows, int64_t cols, float alpha, const float* row_alpha,
                                  const uint64_t* bin, int64_t wpr, const uint64_t* row_ptr,
                                  const uint64_t* col_idx, const float* vals, int64_t nnz,
                                  const uint64_t* t, const uint64_t* h, const uint64_t* m,
                                  int64_t tokens, float a_scale, int has_a_gamma, float a_gamma,
                                  float* c, int64_t ldc);

/* ---- GPU packers (dense fp32 -> reference packed layouts) ----
 * pack_signs: replaces pack_signs (tensor.hpp:248, tensor.cpp:155-164): bit i of row r is
 *   (a[r][i] >= 0) (sign(0) = +1), rows of `wpr` u64 words with zero padding (wpr >= ceil(cols/64);
 *   the reference's default 512-bit lanes give wpr = ceil(cols/512)*8).
 * quantize_thm: replaces quantize_uniform_2bit + decompose_thm (transform.hpp:29,47;
 *   transform.cpp:21-36, 47-75): level = clamp(lround(a/s), 0, 3) -> {t,h,m} planes. */
int bitmm_pack_signs_dev(const float* a, int64_t rows, int64_t cols, int64_t lda, uint64_t* words,
                         int64_t wpr, void* stream);
int bitmm_pack_signs_host(const float* a, int64_t rows, int64_t cols, int64_t lda, uint64_t* words,
                          int64_t wpr);
int bitmm_quantize_thm_dev(const float* a, int64_t rows, int64_t cols, int64_t lda, float s,
                           uint64_t* t, uint64_t* h, uint64_t* m, int64_t wpr, void* stream);
int bitmm_quantize_thm_host(const float* a, int64_t rows, int64_t cols, int64_t lda, float s,
                            uint64_t* t, uint64_t* h, uint64_t* m, int64_t wpr);

/* decompose_thm: replaces decompose_thm (transform.hpp:47, transform.cpp:47-75) on 2-bit levels
 *   (TwoBitMatrix::levels: one byte per element, row-major rows x cols) -> {t,h,m} planes of `wpr`
 *   words. A level above 3 is BITMM_ERR_INVALID_ARGUMENT ("2-bit level out of range"); the _dev
 *   flavour latches it for bitmm_device_status(). */
int bitmm_decompose_thm_dev(const uint8_t* levels, int64_t rows, int64_t cols, uint64_t* t,
                            uint64_t* h, uint64_t* m, int64_t wpr, void* stream);
int bitmm_decompose_thm_host(const uint8_t* levels, int64_t rows, int64_t cols, uint64_t* t,
                             uint64_t* h, uint64_t* m, int64_t wpr);

/* decompose_apb: replaces decompose_apb (apb.hpp:58, apb.cpp:119-142). bin = pack_signs(a) into
 *   `wpr`-word rows; the residual is a CSR of every entry with |a| != alpha, in column order, value
 *   a - alpha*sign(a) computed in double and rounded to float with ties away from zero
 *   (apb.cpp:35-46). row_alpha (optional, `rows` entries) gives each row its own alpha (the
 *   per-row alpha of BASELINE config 4); every alpha must be positive ("alpha must be positive",
 *   BITMM_ERR_INVALID_ARGUMENT). Two calls: the first writes bin and row_ptr[rows+1] and returns
 *   the residual size in *nnz (col_idx / vals may be NULL); when col_idx and vals hold at least
 *   `capacity` >= *nnz entries they are filled too. Synchronous (the size comes back to the host). */
int bitmm_decompose_apb_dev(const float* a, int64_t rows, int64_t cols, int64_t lda, float alpha,
                            const float* row_alpha, uint64_t* bin, int64_t wpr, uint64_t* row_ptr,
                            uint64_t* col_idx, float* vals, int64_t capacity, int64_t* nnz,
                            void* stream);
int bitmm_decompose_apb_host(const float* a, int64_t rows, int64_t cols, int64_t lda, float alpha,
                             const float* row_alpha, uint64_t* bin, int64_t wpr, uint64_t* row_ptr,
                             uint64_t* col_idx, float* vals, int64_t capacity, int64_t* nnz);

#ifdef __cplusplus
}
#endif

#endif /* BITMM_B200_H */
