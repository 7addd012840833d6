/*
 * softmax_b200.h -- C ABI of the B200-native row-softmax hot path.
 *
 * This is the drop-in boundary for the reference's softmax entry point
 * (/root/reference/pkg/src/softmax_kit/kernels.py:350-362,
 *   softmax(m: Matrix2D, variant: KernelVariant, cfg: LaneConfig) -> Matrix2D)
 * and its inner plugin point (kernels.py:283-339, variant_pipeline ->
 * PhasePipeline(maxsub, exp, sumscale)).  The reference is Python + numba;
 * its "FFI" for this path is the Python call, so the binding a maintainer adds
 * is a ctypes stub.  Plain pointers and sizes only: no torch
 * types cross this boundary.
 *
 * Conventions
 *  - float32 row-major [rows, cols] with row pitch ld (elements, >= cols).
 *  - Device entry points (sk_softmax_f32, sk_row_stats_f32, sk_normalize_f32,
 *    sk_rescale_sumexp) are asynchronous on `stream` (a cudaStream_t, passed
 *    as void* so the header does not need cuda_runtime.h); no host sync.
 *  - Status codes map onto the reference error taxonomy (errors.py:4-21):
 *      SK_ERR_ARGUMENT  -> ArgumentError      (tensor.py:43-57, kernels.py:304-305)
 *      SK_ERR_NONFINITE -> NumericDomainError (kernels.py:342-347)
 *      SK_ERR_RESOURCE  -> ResourceError      (tensor.py:98-101)
 *      SK_ERR_CUDA      -> SoftmaxKitError    (no reference analogue)
 *  - Thread-safe across streams: kernels have no global state; the optional
 *    library-managed workspace is keyed by (device, stream).
 */
#ifndef SOFTMAX_B200_H_
#define SOFTMAX_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SK_ABI_VERSION 1

enum sk_status {
  SK_OK = 0,
  SK_ERR_ARGUMENT = 1,
  SK_ERR_NONFINITE = 2,
  SK_ERR_CUDA = 3,
  SK_ERR_RESOURCE = 4,
};

/* Arithmetic mode = the variant ladder (kernels.py:76-96) collapsed to what
 * changes the numbers on a GPU:
 *   SK_MODE_CLIPPED   ReferenceClipped (ValueClip at -64, kernels.py:99, :147)
 *   SK_MODE_EXACT     ReferenceInference, MklStyleScalar, VectorizedSum,
 *                     FullVectorized (no clip, accurate exp)
 *   SK_MODE_APPROX    FullVectorizedApproxExp (no clip, ex2.approx exp;
 *                     tolerance 1e-5, bench.py:52)                           */
enum sk_mode { SK_MODE_CLIPPED = 0, SK_MODE_EXACT = 1, SK_MODE_APPROX = 2 };

/* Sentinel stored in *bad_row when no non-finite input was seen. */
#define SK_NO_BAD_ROW 0xFFFFFFFFFFFFFFFFull
/* written into *bad_row when a cross-CTA / cross-GPU row-statistics exchange
 * timed out (a peer never arrived); the output is then undefined. */
#define SK_EXCHANGE_ABORTED 0xFFFFFFFFFFFFFFFEull

/* The library's per-device non-finite flag (a device uint64, SK_NO_BAD_ROW
 * when clear): what the torch ops (torch_ops/sk_torch_ops.cpp) and the Python
 * wrappers pass as bad_row, so an asynchronous call's bad row is seen by
 * whoever checks the flag next (kernels.check_device_flag()).
 * sk_flag_read copies *flag to the host on `stream` (waiting for the stream)
 * and, with reset, clears it again. */
int sk_device_flag(int device, unsigned long long** flag);
int sk_flag_read(unsigned long long* flag, void* stream, int reset, unsigned long long* value);

int sk_abi_version(void);
const char* sk_status_string(int status);
/* Last CUDA error text seen by this thread (empty if none). */
const char* sk_last_error(void);

/*
 * Fused row softmax on device buffers.  Replaces the three numba phase loops
 * _maxsub_rows_scalar / _exp_rows_scalar / _sumscale_rows_scalar
 * (kernels.py:136-189) with one pass over HBM where the shape allows.
 *
 *  x, y       device pointers, must not alias; y receives [rows, cols].
 *  ldx, ldy   row pitches in elements (>= cols).
 *  bad_row    device uint64; the kernels atomicMin() the index of any row
 *             holding NaN/+-Inf into it.  Initialise it to SK_NO_BAD_ROW once;
 *             it is only written on bad input.  May be NULL (then a
 *             library-owned flag is used and not reported).
 *  workspace  device scratch of sk_softmax_workspace_bytes() bytes (no
 *             initialisation needed; launches on one stream may share it), or
 *             NULL for a library-managed per-(device, stream) workspace.
 * rows == 0 is a no-op.  Returns SK_OK or an error status.
 */
int sk_softmax_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                   int64_t ldy, int mode, unsigned long long* bad_row, void* workspace,
                   size_t workspace_bytes, void* stream);

size_t sk_softmax_workspace_bytes(int64_t rows, int64_t cols);

/*
 * Host-buffer softmax: the compat path behind softmax(Matrix2D, ...).
 * x_host is copied to the device in row chunks, each chunk is computed and
 * copied back, pipelined over H2D / compute / D2H streams and a ring of device
 * buffers (or, with the "host_zero_copy" tuning, one kernel reads and writes
 * pinned host memory directly).  Pinned (page-locked) host buffers give full
 * PCIe bandwidth; pageable ones work, slower.  Returns after y_host is complete.
 * On non-finite input returns SK_ERR_NONFINITE and stores the first bad row
 * in *bad_row_out (y_host contents then unspecified).
 */
int sk_softmax_f32_host(const float* x_host, float* y_host, int64_t rows, int64_t cols,
                        int mode, int device, int64_t* bad_row_out);

/*
 * Column-shard building blocks (sharding.py): local per-row statistics of
 * the [rows, cols] block x, merged across ranks with all-reduce(MAX) on
 * row_max then all-reduce(SUM) on row_sum.  RowStats, kernels.py:108-112.
 *   sk_row_stats_f32:  row_max[r] = max_c x[r,c];
 *                      row_sum[r] = sum_c exp(clip(x[r,c] - row_max[r]))  (f64)
 *   sk_rescale_sumexp: row_sum[r] *= exp(local_max[r] - global_max[r])
 *   sk_normalize_f32:  y[r,c] = exp(clip(x[r,c] - row_max[r])) * (1/(float)row_sum[r])
 */
int sk_row_stats_f32(const float* x, int64_t rows, int64_t cols, int64_t ldx, int mode,
                     float* row_max, double* row_sum, unsigned long long* bad_row,
                     void* workspace, size_t workspace_bytes, void* stream);
size_t sk_row_stats_workspace_bytes(int64_t rows, int64_t cols);
int sk_rescale_sumexp(const float* local_max, const float* global_max, double* row_sum,
                      int64_t rows, void* stream);
int sk_normalize_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                     int64_t ldy, int mode, const float* row_max, const double* row_sum,
                     void* stream);

/*
 * Fused column shard (north_star's column-sharded very-wide-row mode; replaces
 * the row_stats -> all-reduce(MAX) -> rescale -> all-reduce(SUM) -> normalize
 * chain above, RowStats kernels.py:108-112 / 272-276, with ONE kernel per rank).
 * Every rank holds a [rows, cols] column shard (same rows, same cols on every
 * rank; cols % 4 == 0, 16-B aligned rows) and one exchange block of
 * sk_xchg_block_bytes() from sk_xchg_alloc (zeroed, IPC-exportable).  The
 * kernel keeps each row slice resident in shared memory, stores its CTAs'
 * (max, sum) pairs straight into every rank's block over NVLink, polls its own
 * block and writes y -- the cross-GPU all-reduce of the row statistics runs
 * inside the kernel, overlapped with streaming.  Results are identical on all
 * ranks and equal to the single-GPU softmax of the full rows (within the fp32
 * tolerance).  Calls must be issued in the same order on every rank.
 *   sk_ipc_handle / sk_ipc_open / sk_ipc_close: cudaIpc{Get,Open,Close}MemHandle
 *       on an exchange block (handle = SK_IPC_HANDLE_BYTES opaque bytes, sent to
 *       the peers with any host collective).
 *   sk_colshard_softmax_f32: blocks[r] = rank r's block as mapped in THIS
 *       process (blocks[rank] = the local one); bad_row: device flag as in
 *       sk_softmax_f32 (row index within the shard); SK_EXCHANGE_ABORTED if a
 *       peer never arrived.
 *   sk_colshard_emulate_f32: all `world` ranks of a [rows, cols] matrix
 *       (cols % world == 0, shard r = columns [r*cols/world, (r+1)*cols/world))
 *       as ONE cooperative kernel on this GPU with `world` local blocks -- the
 *       same kernel and exchange code, for testing with fewer GPUs than ranks.
 *   sk_describe_colshard_plan: the per-rank plan (cols = shard width).
 *   sk_xchg_reset: zero an exchange block on `stream` (epoch back to 0).  The
 *       slot tags carry a 23-bit launch epoch, so a block must be reset at
 *       least every sk_xchg_reset_period() launches; sk_colshard_softmax_f32
 *       refuses (SK_ERR_ARGUMENT) a launch past that on a multi-rank block.
 *       With peers in other processes every rank must be quiescent around the
 *       reset (barrier, reset own block, synchronise, barrier);
 *       sharding.FusedColumnShard does this itself.  Single-process blocks
 *       (world 1, emulation) are reset automatically.
 */
#define SK_IPC_HANDLE_BYTES 64
size_t sk_xchg_block_bytes(void);
int sk_xchg_alloc(int device, void** block);
int sk_xchg_free(void* block);
int sk_xchg_reset(void* block, void* stream);
unsigned long long sk_xchg_reset_period(void);
int sk_ipc_handle(const void* dev_ptr, void* handle);
int sk_ipc_open(const void* handle, void** dev_ptr);
int sk_ipc_close(void* dev_ptr);
int sk_colshard_softmax_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                            int64_t ldy, int mode, int rank, int world, void* const* blocks,
                            unsigned long long* bad_row, void* stream);
int sk_colshard_emulate_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                            int64_t ldy, int mode, int world, void* const* blocks,
                            unsigned long long* bad_row, void* stream);
int sk_describe_colshard_plan(int64_t rows, int64_t cols, int world, int emulate, int device,
                              char* buf, int buflen);

/*
 * The reference's three phases as separate kernels (NOT the hot path; the
 * fused sk_softmax_f32 is).  They back variant_pipeline() / the GPU phase
 * profile (kernels.py:283-339, profiler.py:96-133):
 *   sk_maxsub_f32    y = x - rowmax, clamped at -64 if clip  (kernels.py:136-151)
 *   sk_exp_f32       buf = exp(buf) in place, mode as sk_softmax_f32 (kernels.py:171-174)
 *   sk_sumscale_f32  buf *= 1/(float)sum(row) (f64 sum), sub-normal -> +0 (kernels.py:177-189)
 */
int sk_maxsub_f32(const float* x, float* y, int64_t rows, int64_t cols, int64_t ldx,
                  int64_t ldy, int clip, void* stream);
int sk_exp_f32(float* buf, int64_t n, int mode, void* stream);
int sk_sumscale_f32(float* buf, int64_t rows, int64_t cols, int64_t ld, void* stream);

/*
 * The reference's 1-D component operations (kernels.py:229-276; test-level
 * API there) on the device, composed with the phase kernels above:
 *   sk_row_sum_f32      row_sum[r] = sum_c x[r,c] accumulated in f64
 *                       (row_sum_scalar kernels.py:258-260, rounded to f32 by the caller)
 *   sk_shift_scale_f32  y = (x - shift) * scale, IEEE: subtract_broadcast
 *                       (kernels.py:234-236, scale 1) and scale_reciprocal
 *                       (kernels.py:263-269, shift 0, scale = 1/(float)sum)
 * row_max_scalar / row_stats use sk_row_stats_f32; exp_batch uses sk_exp_f32.
 */
int sk_row_sum_f32(const float* x, int64_t rows, int64_t cols, int64_t ldx, double* row_sum,
                   void* stream);
/* row_max_scalar / row_stats of one row (kernels.py:119-126, 272-276) with
 * the reference's results for ANY input: max = NaN if x[0] is NaN, else the
 * largest non-NaN value; sum = f64 sum of expf(x - max), NaN / inf
 * propagating.  One block; the component ops use it for non-finite rows. */
int sk_row_stats_ref_f32(const float* x, int64_t n, float* row_max, double* row_sum,
                         void* stream);
int sk_shift_scale_f32(const float* x, float* y, int64_t n, float shift, float scale,
                       void* stream);

/*
 * Page-locked host memory for Matrix2D buffers (tensor.py:90-103 allocates
 * with np.zeros; pinned memory lets sk_softmax_f32_host reach full PCIe
 * bandwidth).  Returns NULL on failure (-> ResourceError).
 */
void* sk_alloc_pinned(size_t bytes);
void sk_free_pinned(void* p);
/*
 * Page-lock / release a caller-owned host range in place (cudaHostRegister,
 * portable).  A registered range is found by sk_softmax_f32_host per call
 * (cudaPointerGetAttributes) and then takes the direct-DMA path with no
 * staging copies.  The host mirror registers a caller's pageable Matrix2D
 * buffers (the reference's np.zeros, tensor.py:90-103) the second time it
 * sees them -- the owning array's whole range as ONE registration, since CUDA
 * rejects any copy (the caller's own, torch's) whose host side straddles two
 * registrations -- and releases them when the owning array dies (hostpin.py);
 * C callers own the lifetime themselves: unregister BEFORE freeing the memory.  SK_OK, or SK_ERR_CUDA (range already registered,
 * locked-memory limit, ...) -- the caller then simply stays on the staged path.
 */
int sk_host_register(void* p, size_t bytes);
int sk_host_unregister(void* p);

/*
 * Process-wide tuning / test hooks (not needed for normal use):
 *   "path"           -1 auto, 0 force K1 (rows in registers), 1 force the TMA
 *                    paths (K2 / K3g / K3c), 2 force split (K4), 3 force K1m
 *   "k1_lpr","k1_nv","k1_u"  force a K1 instantiation (lanes per row,
 *                    float4s per lane, rows per lane-group batch)
 *   "k1_pf", "pdl"   K1 register prefetch (-1 table default), PDL on launches (1)
 *   "vec8"           1: K1 uses 256-bit loads/stores when cols % 8 == 0 and rows
 *                    are 32-B aligned (measured no faster than 128-bit; default 0)
 *   "vec2_max"       widest even row (not a multiple of 4, 8-B pitch / bases) K1
 *                    loads as 64-bit pairs (default 128; 0: 32-bit accesses)
 *   "k1_threads"     K1 threads per block (default 128; halved down to 64 while a
 *                    job has fewer blocks than SMs)
 *   "k1_wide32"      32-bit rows up to this length take K1 with one warp per row
 *                    (36 / 40 floats per lane) instead of K1m (default 1280)
 *   "k1_fit"         1 (default): K1 / K1m shrink the vectors per lane to the fewest
 *                    that cover the row (no padded slots); 0: power-of-two shapes
 *   "grid_mult"      K1 grid = SMs * occupancy * grid_mult (default: one row batch
 *                    per warp, i.e. no grid-stride loop)
 *   "k1m"            1 (default): rows of 1025..8192 floats not taken by K1 go to
 *                    K1m (WPR warps hold a row in registers); 0: K2 / K4 instead
 *   "k1m_wpr","k1m_nv"  force a K1m instantiation (warps per row, vectors per thread)
 *   "k1m_threads"    K1m threads per block (0, default: one row = 32 * WPR threads)
 *   "k3_impl"        long rows (> 8192): 3 (default) K3g, else K3c; 5 K3c only
 *   "gres"           K3g: 1 (default) auto, 0 off, 2 force (also for C <= 8192)
 *   "gres_p","gres_st","gres_split"  force K3g CTAs per row, ring depth (2..5),
 *                    separate poller warp (-1 auto: depth >= 4)
 *   "gres_sleep"     K3g poller back-off (ns, default 128)
 *   "gres_timeout_spins"  polls before a missing peer aborts an exchange (0 = default)
 *   "gres_diag"      1: K3g waits for its own slot only, 2: K3g skips the math
 *                    (timing diagnostics; wrong results); 64 | seed << 8: timing
 *                    chaos -- pseudo-random per-warp delays at every hand-off of
 *                    K3g / K3c, results unchanged (tests/test_gpu_chaos.py)
 *   "colshard_sys"   1: the one-GPU column-shard emulation uses the cross-GPU
 *                    launch's system-scope slot stores / loads (test hook)
 *   "cluster_k3"     1 (default): K3c may serve rows K3g cannot (fallback)
 *   "cluster_size"   force the K3c cluster size (0 = auto: most SMs covered)
 *   "cluster_onex"   1: K3c exchanges one (max, sum) pair per row and recomputes
 *                    exp; 0 (default): two exchanges (max, then sum), exp kept in smem
 *   "cluster_tpb"    K3c threads per CTA (512 default, or 1024)
 *   "k4_fuse_combine" 1 (default): the split path merges each row's partial
 *                    statistics inside its normalize pass (2 launches) when the
 *                    job has <= 4096 (row, chunk) items; 2: always; 0: a separate
 *                    combine kernel (3 launches; same bits either way)
 *   "latency_steps"  K3g row steps per group up to which a long-row job takes the
 *                    latency path (cluster / split kernels) instead (default 3;
 *                    4-6 measured no better, profiles/r1d_latency_threshold_ab.jsonl)
 *   "host_chunk_kb"  sk_softmax_f32_host chunk size in KiB (0 = auto, ~1/4 of the job)
 *   "gres_epoch_reset" launches between zeroings of a K3g exchange block (the
 *                    library's per-stream block; the column-shard period); 0 =
 *                    default 2^22, the maximum (the 23-bit slot epoch never wraps)
 *   "host_threads"   host threads copying pageable caller buffers through the
 *                    page-locked staging slots of sk_softmax_f32_host (0 = auto,
 *                    min(16, hardware threads))
 *   "host_nt"        1 (default): those copies use non-temporal 16-B stores
 *                    (no read-for-ownership of the destination); 0: memcpy
 *   "host_zero_copy" 1: pinned host buffers with rows <= 8192 are read and written
 *                    by the kernel directly over PCIe (measured no faster than
 *                    staging on this box, so 0 by default)
 *   "skip_max_shift" 1: shift by 0 instead of the row max -- the reference's
 *                    _SKIP_MAX_SHIFT fault hook (kernels.py:103-105, :309-311);
 *                    large logits then overflow and verification must fail.
 */
int sk_set_tuning(const char* key, int value);

/*
 * Accuracy diagnostic of the kernels' exponential: sweeps every fp32 value in
 * [lo, hi] (hi <= 0) through the packed and scalar exp paths of `mode` and
 * reports the worst error vs the double-precision exp, in fp32 ulps of the
 * true result and as a relative error.  Synchronous.  (Reference exp:
 * kernels.py:171-174.)
 */
int sk_exp_accuracy(int mode, float lo, float hi, double* max_ulp, double* max_rel, int device);

/*
 * Diagnostic streaming copy y[0, n) = x[0, n) (n % 4 == 0, 16-B aligned) with
 * the softmax kernels' load/store hints and PDL: the same-run floor for a kernel
 * that moves 8 B/element (bound_probe.py:67-87 analogue).  blocks <= 0: auto.
 */
int sk_copy_f32(const float* x, float* y, int64_t n, int blocks, void* stream);

/*
 * Launch plan that sk_softmax_f32 would use for this shape/alignment, as a
 * short text ("k1_vec lpr=8 nv=4 u=2 grid=..." ...), for tests and bench logs.
 * Writes at most buflen bytes (NUL-terminated); returns SK_OK.
 */
int sk_describe_plan(int64_t rows, int64_t cols, int64_t ldx, int64_t ldy, uint64_t x_addr,
                     uint64_t y_addr, int device, char* buf, int buflen);

/*
 * Deterministic host-side input generators (tensor.py:106-121 and the
 * BASELINE configs).  Element i of a fill depends only on (seed, i), so
 * chunks [start, start+n) can be generated independently and in parallel.
 *   sk_fill_uniform_f32: fill_uniform (tensor.py:106-121): Philox4x64-10
 *       raw draw i (numpy np.random.Philox(key=seed)) -> ((u>>11)+0.5)*2^-53
 *       -> low+(high-low)u in f64 -> f32 -> clamp into the open interval.
 *   sk_fill_normal_f32: N(0, sigma^2): Box-Muller on raw draws (2i, 2i+1)
 *       giving elements 2i (cos) and 2i+1 (sin), in f64, then f32.
 *   sk_plant_f32: sets `count` distinct flat positions of x[0, total) to
 *       `value`; positions = first distinct (raw % total) of the Philox stream
 *       keyed by seed ^ 0x5EEDC0FFEE, in draw order.
 * nthreads <= 0: use all hardware threads.
 */
int sk_fill_uniform_f32(float* dst, int64_t n, uint64_t seed, double low, double high,
                        uint64_t start, int nthreads);
int sk_fill_normal_f32(float* dst, int64_t n, uint64_t seed, double sigma, uint64_t start,
                       int nthreads);
int sk_plant_f32(float* x, int64_t total, int64_t count, uint64_t seed, float value);

#ifdef __cplusplus
}
#endif
#endif /* SOFTMAX_B200_H_ */
