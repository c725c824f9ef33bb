/*
 * omni.h -- C-ABI of libomni.so, the sm_100a (B200) kernels behind the
 * omnisim-compatible Python API in paper_1606_04487_b200/.
 *
 * The reference (omnisim 0.1.0, /root/reference/pkg/src/omnisim) is pure
 * Python/NumPy and has no FFI; each entry point below replaces one NumPy op
 * site on the data-parallel CNN training hot path and cites it.  The binding
 * a maintainer adds on the reference side is ctypes.
 *
 * ABI rules
 *   - every entry point returns 0 on success, a negative OMNI_E* status
 *     otherwise; omni_last_error() returns a message for the calling thread;
 *   - all launches are asynchronous on the caller's stream (a cudaStream_t
 *     passed as void*; NULL = legacy default stream);
 *   - the library never allocates persistent device memory: callers pass
 *     every buffer, including GEMM split-K workspace (omni_gemm_plan sizes it);
 *   - plain pointers and sizes only; row strides ("ld") are in ELEMENTS.
 */
#ifndef OMNI_H_
#define OMNI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OMNI_OK 0
#define OMNI_EINVAL -1       /* bad argument: maps to ValueError           */
#define OMNI_ECUDA -2        /* CUDA runtime / driver failure: RuntimeError */
#define OMNI_EUNSUPPORTED -3 /* shape/layout outside what a kernel handles  */
#define OMNI_ETIMEOUT -4     /* a wait gave up (a peer process stalled or died) */

const char* omni_last_error(void);
int omni_version(void);
int omni_device_sm_count(int device);
/* Kernels launched by this library so far (process-wide; for launch accounting). */
long long omni_launch_count(void);
/* SMs the persistent GEMM grids leave free for concurrent communication
 * kernels (data parallel; default 0 or $OMNI_SM_RESERVE).  Plans (and so
 * split-K workspace sizes) depend on it: set it before sizing workspaces.   */
int omni_set_sm_reserve(int sms);
int omni_get_sm_reserve(void);

/* ---------------------------------------------------------------- K1 --
 * Batched lowering (type-1 im2col over b_p images starting at `start`).
 * Replaces tensors.lower (tensors.py:164-181).  Row = img*m^2 + x*m + y,
 * column = (c*k + kx)*k + ky (tensors.py:167-168); zero padding; pure copy,
 * hence bit-exact in both element types.  Dhat is (b_p*m^2) x ld, ld >= c*k*k;
 * columns [c*k*k, ld) are written with zeros.                              */
int omni_lower_nchw_f32(const float* D, int b, int c, int n, int k, int stride, int pad,
                        int start, int b_p, float* Dhat, long long ld, void* stream);
int omni_lower_nchw_f64(const double* D, int b, int c, int n, int k, int stride, int pad,
                        int start, int b_p, double* Dhat, long long ld, void* stream);
/* Training-path lowering from NHWC activations (pixel stride cs >= c) with the
 * tap-major column order (kx*k + ky)*c + ch.  Same values as the reference's
 * lowered matrix up to that fixed column permutation.  ones_col != 0 writes
 * 1.0 into column c*k*k (the bias column: with the bias staged in the same
 * column of the weights, the GEMM adds the bias and the weight-gradient GEMM
 * produces the bias gradient).                                             */
int omni_lower_nhwc_f32(const float* X, int b, int n, int c, int cs, int k, int stride,
                        int pad, int ones_col, float* Dhat, long long ld, void* stream);

/* Lifting: Rhat (b*m^2) x ld -> NCHW (b, d_out, m, m).  Replaces tensors.lift
 * (tensors.py:213-219); index remap only, bit-exact.                        */
int omni_lift_nchw_f32(const float* Rhat, long long ld, int b, int m, int d_out, float* R,
                       void* stream);
int omni_lift_nchw_f64(const double* Rhat, long long ld, int b, int m, int d_out, double* R,
                       void* stream);

/* col2im (adjoint of omni_lower_nhwc_f32), deterministic gather form: dX (NHWC,
 * pixel stride cs) is OVERWRITTEN with the sum over every lowered entry that
 * copied from it.  Not in the reference (its only conv is layer 1, so
 * problems.py:263-269 never needs dX); pinned by the adjoint identity.
 * relu_mask_x (NHWC like dX, may be NULL) fuses the ReLU backward mask of the
 * layer that produced X: dX = col2im(dDhat) * (X > 0) (problems.py:261).    */
int omni_col2im_nhwc_f32(const float* dDhat, long long ld, int b, int n, int c, int cs, int k,
                         int stride, int pad, const float* relu_mask_x, float* dX, void* stream);

/* ---------------------------------------------------------------- K2 --
 * C[i,j] (op)= sum_r A(i,r) * B(j,r),  i < M, j < N, r < K, where
 *   A(i,r) = a_mn_major ? A[r*lda + i] : A[i*lda + r]
 *   B(j,r) = b_mn_major ? B[r*ldb + j] : B[j*ldb + r]
 * Replaces tensors.gemm (tensors.py:193-210) and every product in
 * problems.py:218,250-251,263-267.  tcgen05.mma kind::tf32 with TMA-fed
 * 128B-swizzled shared-memory stages and TMEM accumulators.
 * Requirements: lda, ldb multiples of 4 and A, B 16-byte aligned (TMA).     */
#define OMNI_PREC_TF32 0      /* one tf32 pass (fast path)                        */
#define OMNI_PREC_3XTF32 1    /* hi/lo split in shared memory, 3 tf32 passes       */
#define OMNI_PREC_FP32_SIMT 2 /* CUDA-core fp32 (test reference only; not hot path) */

#define OMNI_EPI_STORE 0       /* C = acc                                  */
#define OMNI_EPI_BIAS 1        /* C = acc + bias[j]                        */
#define OMNI_EPI_BIAS_RELU 2   /* C = max(acc + bias[j], 0)                */
#define OMNI_EPI_ACCUM 3       /* C = C + acc                              */
#define OMNI_EPI_MASK_AUX 4    /* C = acc * (aux[i*ld_aux + j] > 0)  (ReLU bwd) */
#define OMNI_EPI_RELU 5        /* C = max(acc, 0)                          */

/* Plan query: returns the split-K workspace (bytes) omni_gemm_f32 will need for
 * these arguments; *splits / *bn report the chosen schedule (may be NULL).   */
long long omni_gemm_plan(int precision, int M, int N, int K, int a_mn_major, int b_mn_major,
                         int* splits, int* bn);
int omni_gemm_f32(int precision, int M, int N, int K, const float* A, long long lda,
                  int a_mn_major, const float* B, long long ldb, int b_mn_major, float* C,
                  long long ldc, int epilogue, const float* bias, const float* aux,
                  long long ld_aux, float* workspace, long long ws_bytes, void* stream);

/* Implicit-GEMM convolution on tcgen05 -- replaces tensors.conv_lowered
 * (tensors.py:222-256: lower + gemm + lift) for the training path, and the
 * weight-gradient einsum of problems.py:263-267 -- with the operands gathered
 * by TMA im2col from the NHWC activation X (b, n, n, cs): no lowered matrix in
 * HBM.  The GEMM
 * K index is (tap, channel) tap-major, i.e. the column order of
 * omni_lower_nhwc_f32, with cp = round_up(c, 32) channels per tap (channels
 * c..cp-1 of a partial 32-channel block read as zeros).
 *   OMNI_CONV_FPROP: Y[pix, o] (op)= sum_{tap,ch} X(pix, tap, ch) G[o*ldg + tap*cp + ch]
 *                    (G = tap-major weights d_out x ldg; Y = b*m*m rows, ld ldy)
 *   OMNI_CONV_WGRAD: Y[o*ldy + tap*cp + ch] = sum_pix G[pix*ldg + o] X(pix, tap, ch)
 *                    (G = output gradient dY, b*m*m rows, ld ldg)
 * The data gradient of a stride-1 conv is OMNI_CONV_FPROP on dY with pad
 * k-1-pad and the spatially flipped, transposed weights.                     */
/*   OMNI_CONV_WGRAD_BIAS: as OMNI_CONV_WGRAD, plus the bias gradient
 *                    Y[o*ldy + k*k*cp] = sum_pix G[pix*ldg + o] as one more GEMM row
 *                    (a ones operand chunk; needs ldy > k*k*cp).  The workspace
 *                    (size from omni_conv_implicit_plan) reserves room for that
 *                    ones tile; the library reads its own constant copy.  */
#define OMNI_CONV_FPROP 0
#define OMNI_CONV_WGRAD 1
#define OMNI_CONV_WGRAD_BIAS 2
long long omni_conv_implicit_plan(int precision, int op, int b, int n, int c, int k, int stride,
                                  int pad, int d_out);
int omni_conv_implicit_f32(int precision, int op, const float* X, int b, int n, int c, int cs,
                           int k, int stride, int pad, int d_out, const float* G, long long ldg,
                           float* Y, long long ldy, int epilogue, const float* bias,
                           const float* aux, long long ld_aux, float* workspace,
                           long long ws_bytes, void* stream);

/* ---------------------------------------------------------------- K3 --
 * Pooling over NHWC (pixel strides cs_in / cs_out).  mode 0 = max (first max in
 * (dy,dx) window order, argmax = input pixel index iy*w + ix, as
 * problems.py:213-216), mode 1 = average (Caffe semantics: divisor is the
 * window clipped to the padded extent).  ceil_mode selects Caffe's output size
 * rule.  Backward is a deterministic gather; if relu_mask_x == 1 the input
 * gradient is also multiplied by (X > 0) (fused ReLU mask, problems.py:261).
 * relu_mask_x == 2 (max pool only): X is the pooled OUTPUT (b, oh, ow, cs_out)
 * and each window's gradient is masked by (Y > 0) -- the same result, since
 * gradient reaches only the argmax element and Y equals it, at 1/k^2-ish of
 * the bytes.  Forward mode 2 = max with that mask folded into the indices:
 * windows whose maximum is not > 0 get the argmax sign bit set (argmax &
 * 0x7fffffff is mode 0's), so backward mode 0 with relu_mask_x = 0 routes
 * exactly what relu_mask_x = 2 does without reading Y.                      */
int omni_pool_out_size(int n, int k, int stride, int pad, int ceil_mode);
int omni_pool_fwd_nhwc_f32(int mode, const float* X, int b, int h, int w, int c, int cs_in,
                           int k, int stride, int pad, int ceil_mode, float* Y, int cs_out,
                           int32_t* argmax, void* stream);
int omni_pool_bwd_nhwc_f32(int mode, const float* dY, int b, int h, int w, int c, int cs_in,
                           int k, int stride, int pad, int ceil_mode, int cs_out,
                           const int32_t* argmax, const float* X, int relu_mask_x, float* dX,
                           void* stream);

/* ---------------------------------------------------------------- K4 --
 * Softmax cross-entropy over rows of logits (b x C, row stride ld):
 * loss[0] = mean_i(lse_i - z_{i,y_i}) (problems.py:230-233); dlogits =
 * (softmax - onehot) * scale (problems.py:246-248 with scale = 1/b).  One
 * launch; deterministic.  dlogits may be NULL (loss only).                   */
int omni_softmax_xent_f32(const float* logits, long long ld, const int32_t* labels, int b,
                          int C, float* loss, float* dlogits, long long ldd, float scale,
                          void* stream);

/* ---------------------------------------------------------------- misc --
 * ReLU forward/backward on a dense buffer (problems.py:211, :261; strict >). */
int omni_relu_fwd_f32(const float* X, float* Y, long long n, void* stream);
int omni_relu_bwd_f32(const float* dY, const float* Y, float* dX, long long n, void* stream);
/* Bias gradient: db[j] = sum_i dY[i*ld + j], i < M (deterministic 2-pass).
 * ws must hold omni_bias_grad_ws_elems(M, N) floats.                         */
long long omni_bias_grad_ws_elems(int M, int N);
int omni_bias_grad_f32(const float* dY, long long ld, int M, int N, float* db, float* ws,
                       void* stream);
/* Window implicit GEMM of a space-to-depth first layer (conv_window.cu):
 * Xs is the (b, n2, n2, 48) space-to-depth image (omni_space_to_depth_f32,
 * cp = 48), the conv is k2 x k2, stride 1, no padding, m = n2 - k2 + 1.
 *   OMNI_CONV_FPROP:      Y[pix*ldy + o] = epi(sum_{tap,ch} Xs(pix, tap, ch) G[o*ldg + tap*48 + ch])
 *                         (G = omni_conv_weight_s2d_f32 rows; d_out in {32, 64, 96, 128};
 *                          epilogue STORE / BIAS / BIAS_RELU / RELU)
 *   OMNI_CONV_WGRAD_BIAS: Y[o*ldy + tap*48 + ch] = sum_pix G[pix*ldg + o] Xs(pix, tap, ch),
 *                         Y[o*ldy + k2*k2*48] = sum_pix G[pix*ldg + o]  (ldy >= k2*k2*48 + 16;
 *                          d_out <= 128; workspace per omni_conv_window_plan)
 * TF32 only (the 3xTF32 path keeps the generic implicit GEMM with cp = 64).
 * omni_conv_window_plan returns the workspace bytes, or -1 when the window
 * kernels do not cover the geometry (window rows > 256, k2 > 3, ...).         */
long long omni_conv_window_plan(int op, int b, int n2, int cp, int k2, int d_out);
int omni_conv_window_f32(int op, const float* Xs, int b, int n2, int cp, int k2, int d_out, const float* G,
                         long long ldg, float* Y, long long ldy, int epilogue, const float* bias,
                         float* workspace, long long ws_bytes, void* stream);
/* Mailbox of the free-running compute groups (async_groups.py, mailbox.cu):
 * a POSIX shared-memory page of lock-free atomics through which the update
 * server (co-located on rank 0) and the group leaders hand over gradients and
 * snapshots; the payloads move GPU to GPU by DMA (omni_copy_async on
 * IPC-mapped buffers).  post: a leader whose gradient has landed takes a
 * ticket; next: the server takes the next ticket's group (FIFO by arrival,
 * simulator.py:3-7); snap_post / snap_wait: per-group snapshot sequence
 * (-1 = stop).  Waits return OMNI_ETIMEOUT after timeout_ms.                */
long long omni_mailbox_bytes(void);
int omni_mailbox_create(const char* name, int ngroups, void** box);
int omni_mailbox_open(const char* name, void** box, int timeout_ms);
int omni_mailbox_close(void* box, const char* unlink_name);
int omni_mailbox_post(void* box, int group, long long* ticket);
int omni_mailbox_next(void* box, int* group, int timeout_ms);
int omni_mailbox_snap_post(void* box, int group, long long seq);
int omni_mailbox_snap_wait(void* box, int group, long long last, long long* seq, int timeout_ms);

/* K8 fused momentum SGD (sgd.py:92-101): V = mu*V - eta*(g + lam*w_read);
 * W = W + V.  w_read may alias W (synchronous step).                         */
int omni_sgd_momentum_f32(float* W, float* V, const float* g, const float* w_read, float eta,
                          float mu, float lam, long long n, void* stream);
/* The g ordered updates of one compute-group round on a shard (groups.py,
 * simulator.py:123-213 deterministic schedule): rows is nrows x n (pitch ld),
 * row m = rank m's gradient shard; for i = 0..g-1 in order, group i's gradient
 * is the sum of rows members[i*k .. i*k+k) in that order, the K8 update
 * V = mu*V - eta*(G_i + lam*snaps[i]); W += V is applied, and snaps[i] = W
 * (group i's next snapshot).  members / snaps are host arrays (g*k <= 64).   */
int omni_group_updates_f32(const float* rows, int nrows, long long ld, const int* members, int g,
                           int k, float* W, float* V, float* const* snaps, long long n, float eta,
                           float mu, float lam, void* stream);
/* K8 in float64 for the drop-in host API (SGDState keeps float64, sgd.py:72-101):
 * same update, the reference's evaluation order, no FMA contraction, so it
 * is bit-identical to the NumPy expression.                                  */
int omni_sgd_momentum_f64(double* W, double* V, const double* g, const double* w_read, double eta,
                          double mu, double lam, long long n, void* stream);
/* K9 batch gather (problems.py:197-199): dst[i,:] = src[idx[i],:].            */
int omni_gather_rows_f32(const float* src, long long row_elems, const int64_t* idx, int nidx,
                         float* dst, void* stream);
int omni_gather_i32(const int32_t* src, const int64_t* idx, int nidx, int32_t* dst,
                    void* stream);
/* Weight layout staging (the device counterpart of tensors.lower_kernel,
 * tensors.py:184-190, in tap-major column order):
 * OIHW (o,c,k,k) <-> tap-major (o, (kx*k+ky)*c + ch)
 * rows of stride ld (pad columns zeroed).  inverse=0 reads W and writes Wt;
 * inverse=1 reads Wt and writes W.  bias (may be NULL) travels in column
 * c*k*k of Wt in the same direction.                                       */
int omni_conv_weight_to_tap_f32(float* W, int o, int c, int k, float* Wt, long long ld,
                                int inverse, float* bias, void* stream);
/* Data-gradient weights of a stride-1 conv: Wf (c rows, ld >= o*k*k) with
 * Wf[ch*ld + (kx*k + ky)*o + oo] = W[oo, ch, k-1-kx, k-1-ky] (W is OIHW).     */
int omni_conv_weight_flip_f32(const float* W, int o, int c, int k, float* Wf, long long ld,
                              void* stream);
/* Space-to-depth with channel padding (first-layer implicit GEMM; part of
 * conv_lowered, tensors.py:222-256, for strided narrow layers): X (b, n, n,
 * pixel stride cs, c channels) -> Y (b, n2, n2, cp),
 * Y[img, X, Y, (dx*s + dy)*c + ch] = X[img, s*X + dx, s*Y + dy, ch], zero outside
 * the image and in channels >= s*s*c.  A stride-s k x k conv of X equals a
 * stride-1 ceil(k/s) x ceil(k/s) conv of Y with the weights below.            */
int omni_space_to_depth_f32(const float* X, int b, int n, int c, int cs, int s, float* Y, int n2,
                            int cp, void* stream);
/* Same, fused with the batch gather: image i of Y is image idx[i] of the
 * dataset X (the device-resident sample, problems.py:197-199).               */
int omni_space_to_depth_gather_f32(const float* X, const int64_t* idx, int b, int n, int c, int cs,
                                   int s, float* Y, int n2, int cp, void* stream);
/* Weights of that conv, tap-major rows Wt (o x ld, ld >= ceil(k/s)^2 * cp):
 * Wt[o*ld + (kx2*k2 + ky2)*cp + (dx*s + dy)*c + ch] = W[o, ch, s*kx2+dx, s*ky2+dy]
 * (0 past the kernel).  inverse=1 maps a gradient in that layout back to OIHW
 * and, when bias != NULL, copies column ceil(k/s)^2 * cp (the
 * OMNI_CONV_WGRAD_BIAS row) to bias[o].                                        */
int omni_conv_weight_s2d_f32(float* W, int o, int c, int k, int s, int cp, float* Wt, long long ld,
                             int inverse, float* bias, void* stream);
/* Batched 2-D transpose: dst[bi][j*ldd + i] = src[bi][i*lds + j], i < rows,
 * j < cols; batch strides in elements.  Used for NHWC <-> flattened CHW and
 * for FC weight staging.                                                     */
int omni_transpose_f32(const float* src, long long lds, long long src_bstride, int rows,
                       int cols, float* dst, long long ldd, long long dst_bstride, int batch,
                       void* stream);
/* Fill / scale helpers. */
int omni_fill_f32(float* X, float value, long long n, void* stream);

/* ------------------------------------------------------------ comm --
 * Communicators for the multi-GPU path: the gradient
 * allreduce inside a compute group (replaces the reference's logical
 * data-parallel mean, simulator.py:3-7 / sgd.py:210-256 with N GPUs) and the
 * server <-> group-leader transfers of the asynchronous runtime (the
 * reference's FIFO model server, simulator.py:123-213).  NCCL is loaded at
 * run time (dlopen "libnccl.so.2"); without it every entry point returns
 * OMNI_EUNSUPPORTED.  Communicators are opaque pointers (ncclComm_t).
 * NCCL calls must come from the thread that owns the communicator's device. */
#define OMNI_COMM_ID_BYTES 128
#define OMNI_COMM_SPLIT_NOCOLOR (-1)
int omni_comm_nccl_version(int* version);
/* One process per GPU: rank 0 makes the id, the host ships it to every rank. */
int omni_comm_unique_id(void* id /* OMNI_COMM_ID_BYTES */);
int omni_comm_init_rank(void** comm, int nranks, const void* id, int rank, int device);
/* One process driving ndev GPUs: comms[i] on devs[i] (devs NULL = 0..ndev-1). */
int omni_comm_init_all(int ndev, const int* devs, void** comms);
/* Compute groups: ranks with the same color form one communicator, ordered by
 * key; OMNI_COMM_SPLIT_NOCOLOR opts out (newcomm = NULL).  Collective.  Inside
 * a group_start/end bracket *newcomm is written at group end, so the slot
 * must outlive the bracket.                                                */
int omni_comm_split(void* comm, int color, int key, void** newcomm);
int omni_comm_destroy(void* comm);
int omni_comm_size_rank(void* comm, int* size, int* rank);
/* In-place sum over the communicator (a group's gradient), on the stream. */
int omni_allreduce_sum_f32(void* comm, float* buf, size_t n, void* stream);
/* Point to point (snapshot / gradient exchange with the update server).   */
/* In-place broadcast of buf from communicator rank `root` (a compute group's
 * new snapshot from its leader to the other members).                        */
int omni_broadcast_f32(void* comm, float* buf, size_t n, int root, void* stream);
int omni_send_f32(void* comm, const float* buf, size_t n, int peer, void* stream);
int omni_recv_f32(void* comm, float* buf, size_t n, int peer, void* stream);
/* recv[r*n .. (r+1)*n) = rank r's send (n floats), every rank (the sharded
 * group runtime's master-model assembly).                                    */
int omni_allgather_f32(void* comm, const float* send, float* recv, size_t n, void* stream);
/* Personalised all-to-all: parts[m] (a host array of nranks device pointers,
 * n floats each) goes to rank m; rank m's part for this rank lands at
 * recv + m*n.  The sharded group round's gradient-shard and snapshot-shard
 * exchanges (groups.py), without staging the parts contiguously.            */
int omni_all_to_all_f32(void* comm, const float* const* parts, float* recv, size_t n,
                        void* stream);
/* Bracket several send/recv calls so NCCL fuses them (no deadlock on
 * simultaneous exchanges).                                                 */
int omni_comm_group_start(void);
int omni_comm_group_end(void);

/* ------------------------------------------------------------- p2p --
 * Peer-memory data-parallel update (one process per GPU, one NVSwitch node):
 * the gradient allreduce and the momentum update of a layer slice [lo, hi)
 * fused into one kernel that reads the N ranks' gradients straight out of
 * their HBM (CUDA IPC mappings), sums them in rank order 0..N-1, applies
 * V = mu V - eta (G_sum + lam w_read); W += V (sgd.py:92-101; the caller
 * folds the mean's 1/N into eta and lam) to this rank's part of the slice --
 * elements [lo + r*c, lo + (r+1)*c) with c = 4*ceil((hi-lo)/(4N)), clipped to
 * hi; the caller passes that sub-range -- and stores the new W into every
 * rank's W.  V stays valid on the owning rank only.  grads[p] / weights[p] are
 * rank p's buffers as mapped in this process (weights[rank] is local), all
 * with the same 16-byte alignment; weights[p] = NULL (p != rank) skips that
 * store (the copy-engine variant: gradients pushed into local lanes with
 * omni_copy_async, W sent the same way).  N <= 8.
 *
 * Cross-GPU ordering: flag blocks of int64 [2 kinds][N src][max_slots], one
 * per rank; omni_p2p_step increments this rank's device step counter *step;
 * omni_p2p_signal stores *step into slot [kind][rank][slot] of every rank's
 * block (system-scope release, after the stream's previous work);
 * omni_p2p_wait blocks the stream until this rank's block holds >= *step in
 * [kind][*][slot_lo, slot_hi) (acquire; traps after 30 s instead of hanging
 * if a peer died).  All values live on the device, so a CUDA graph of a whole
 * step replays correctly.                                                   */
#define OMNI_P2P_GRAD_READY 0 /* src's gradient of the slot is final, W no longer read */
#define OMNI_P2P_W_DONE 1     /* src wrote its part of the slot's W into every rank */
#define OMNI_IPC_HANDLE_BYTES 64
int omni_p2p_step(long long* step, void* stream);
int omni_p2p_signal(long long* const* flags, int nranks, int rank, int kind, int slot,
                    int max_slots, const long long* step, void* stream);
int omni_p2p_wait(const long long* flags, int nranks, int rank, int kind, int slot_lo, int slot_hi,
                  int max_slots, const long long* step, void* stream);
int omni_p2p_reduce_sgd_f32(const float* const* grads, float* const* weights, int nranks, int rank,
                            long long lo, long long hi, float* V, const float* w_read, float eta,
                            float mu, float lam, void* stream);
/* Asynchronous copy on the stream by the copy engines (peer-mapped pointers
 * allowed: an NVLink DMA that occupies no SM).                              */
int omni_copy_async(void* dst, const void* src, long long bytes, void* stream);
/* IPC: the handle of the allocation holding ptr and ptr's byte offset in it;
 * open maps a peer's allocation (base pointer; add the offset), close unmaps. */
int omni_ipc_handle(const void* ptr, void* handle, long long* offset);
int omni_ipc_open(const void* handle, void** base);
int omni_ipc_close(void* base);

#ifdef __cplusplus
}
#endif
#endif /* OMNI_H_ */
