/*
 * icl.h -- C ABI of the B200-native ImageCL hot-path library (libicl.so).
 *
 * The library computes the per-pixel image filters of the three benchmarks
 * that ImageCL's compiler + auto-tuner exist to speed up (§6,
 * lines 546-603; NLM replaces non-separable convolution per BASELINE.json
 * north_star), over the tuned variant space of PAPER.md Table 1 (lines
 * 364-393, §5.2.1-5.2.5), re-designed for sm_100a.
 *
 * Conventions (all entry points):
 *  - extern "C", no C++ exceptions cross the ABI, no torch/CUDA types in the
 *    signatures: streams are passed as `void*` holding a cudaStream_t
 *    (NULL = legacy default stream).
 *  - Image pixel pointers are DEVICE pointers owned by the caller; the
 *    library never frees or retains them beyond the call.  Filter
 *    parameters (taps) are HOST pointers read during the call and copied by
 *    value into the kernel parameter block (the "constant memory" parameter
 *    of PAPER.md:477-482).
 *  - Filter calls only ENQUEUE work on `stream` and return; they never
 *    synchronise the host.  Asynchronous CUDA faults surface at the caller's
 *    next synchronisation.  icl_tune() synchronises.
 *  - On any non-OK status nothing has been enqueued, and icl_last_error()
 *    returns a thread-local human-readable message.
 *  - Image layout: fp32 (masks: uint8), row-major; pixel (x, y) of image b
 *    is at  data + b*batch_stride_bytes + y*pitch_bytes + x*elem_size
 *    (x = column = contiguous axis = ImageCL idx; y = row = idy;
 *    PAPER.md:289-296).
 *  - Environment (read once per process): ICL_TUNE_POLICY = off (default:
 *    cached winner, else the built-in default variant) | on_miss (tune an
 *    uncached problem at its first call) | require (ICL_ERR_NOT_TUNED when
 *    uncached); ICL_TUNE_CACHE = path of a tune cache loaded before the first
 *    call (when present and for this device/build) and saved after every
 *    tuning; ICL_FORCE_VARIANT = "filter=variant[,filter=variant]" forces
 *    variants process-wide (icl_force_variant, per thread, wins); ICL_LOG=1
 *    prints every dispatch decision (problem key -> variant, reason) to
 *    stderr; ICL_HOST_CHUNK_ROWS = rows per band of the host-image path.
 *    Each filter call's enqueue is an NVTX range "icl <filter> <variant>".
 *  - Boundary conditions: reads outside the image return the nearest edge
 *    pixel (CLAMP) or `border_value` (CONSTANT) -- PAPER.md:303-308 and
 *    Fig. 3 (lines 311-327).  Boundaries are applied in GLOBAL image
 *    coordinates, also for row bands (icl_band).
 *  - Aliasing between a source and any destination is rejected
 *    (ICL_ERR_ALIASING): "In ImageCL, we disallow aliasing".
 */
#ifndef ICL_H_
#define ICL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ICL_ABI_VERSION 1

typedef enum {
    ICL_OK = 0,
    ICL_ERR_INVALID_ARG = 1, /* null pointer, bad size/pitch/parameter */
    ICL_ERR_ALIASING = 2,    /* source and destination byte ranges overlap */
    ICL_ERR_UNSUPPORTED = 3, /* parameter outside the compiled variant space */
    ICL_ERR_WORKSPACE = 4,   /* forced variant needs more workspace than given */
    ICL_ERR_CUDA = 5,        /* CUDA launch/runtime error */
    ICL_ERR_NCCL = 6,        /* NCCL error (sharded calls) */
    ICL_ERR_NOT_TUNED = 7    /* ICL_TUNE_POLICY=require and no cache entry */
} icl_status;

typedef enum { ICL_BORDER_CONSTANT = 0, ICL_BORDER_CLAMP = 1 } icl_border;

typedef enum {
    ICL_FILTER_SEPCONV = 0,
    ICL_FILTER_HARRIS = 1,
    ICL_FILTER_NLM = 2,
    ICL_FILTER_CONV2D = 3,
    ICL_FILTER_SEPCONV3D = 4 /* icl_sepconv3d (variant registry / force / last only) */
} icl_filter;

/* A (batch of) 2-D image(s).  `data` is a device pointer or a HOST pointer
 * (fp32 pixels for images, uint8 for masks).  When any operand of
 * icl_sepconv / icl_harris / icl_nlm is host memory (pinned, or pageable --
 * pageable copies are staged synchronously by the driver), the call streams
 * the batch through the GPU in row bands of ~16 MiB: H2D of a band's input
 * rows (+ stencil halo) into library-owned device staging buffers, the filter
 * on that band (icl_band semantics: results equal the device-resident call,
 * bit for bit for sepconv and Harris), D2H of its output; the three stages of
 * consecutive bands overlap on three library streams forked from and joined
 * back into `stream`.  Host buffers must stay valid until `stream` reaches
 * the call (icl_transfer_bytes counts the bytes moved).  Device-resident
 * operands are used in place.  width, height >= 1 and < 2^31; pitch_bytes >=
 * width*elem_size and a multiple of elem_size; 1 <= batch < 2^31; when batch > 1,
 * batch_stride_bytes >= height*pitch_bytes (images must not overlap). */
typedef struct {
    void* data;
    int64_t width;
    int64_t height;
    int64_t pitch_bytes;
    int64_t batch;
    int64_t batch_stride_bytes;
} icl_image;

/* Row band of a taller GLOBAL image (row-band sharding).
 * src row 0 is global row src_y0; dst row 0 is global row dst_y0; the call
 * computes every dst row.  Every global row in [0, global_height) that a dst
 * row's stencil touches must be present in src.  NULL band == the whole
 * image: {global_height = src.height, src_y0 = 0, dst_y0 = 0} and
 * dst.height == src.height. */
typedef struct {
    int64_t global_height;
    int64_t src_y0;
    int64_t dst_y0;
} icl_band;

/* ------------------------------------------------------------------------
 * Separable convolution (§6; Table 2 R and C kernels,
 * lines 611-629).  Correlation form (Listing 1):
 *     out(x,y) = sum_{j=-ry..ry} taps_y[j+ry] * sum_{i=-rx..rx} taps_x[i+rx] * src_B(x+i, y+j)
 * Every variant evaluates, per output, the same fp32 FMA chain (inner over
 * i = -rx..rx, intermediate rounded to fp32, outer over j), so all variants
 * and all band splits are bit-identical (R16).
 * rx, ry in [0, 15]  (> 15 -> ICL_ERR_UNSUPPORTED); taps are HOST arrays of
 * 2r+1 floats.  src/dst: fp32, same width; dst.height = band rows.
 * workspace: optional device scratch for two-pass variants (size from
 * icl_sepconv_workspace_bytes); may be NULL, in which case only single-pass
 * variants are eligible.
 * ---------------------------------------------------------------------- */
icl_status icl_sepconv(const icl_image* src, const icl_image* dst, const float* taps_x, int rx,
                       const float* taps_y, int ry, icl_border border, float border_value,
                       const icl_band* band, void* workspace, size_t workspace_bytes, void* stream);

/* Workspace (bytes) that lets every sepconv variant run for these sizes. */
size_t icl_sepconv_workspace_bytes(int64_t width, int64_t height, int64_t batch, int ry);

/* ------------------------------------------------------------------------
 * Harris corner response (§6; Table 4 Sobel kernel,
 * Table 5 Harris kernel, lines 651-687), per-stage semantics (DESIGN.md
 * R6-R10):  dx = Kx * src_B, dy = Ky * src_B with the unnormalised 3x3
 * Sobel Kx = [1,2,1]^T[-1,0,1], Ky = Kx^T; dx/dy outside the image are
 * dx(clamp(q)) (CLAMP) or 0 (CONSTANT); window sums over
 * [-floor(B/2), B-1-floor(B/2)]^2;
 *     R = Sxx*Syy - Sxy^2 - k*(Sxx+Syy)^2.
 * block (window side B) in [1, 7]; k finite.
 * mask: optional uint8 device image (same width/height/batch as response,
 * own pitch); mask = (R > threshold) ? 1 : 0, decided in fp32.
 * ---------------------------------------------------------------------- */
icl_status icl_harris(const icl_image* src, const icl_image* response, int block, float k,
                      icl_border border, float border_value, const icl_image* mask, float threshold,
                      const icl_band* band, void* stream);

/* ------------------------------------------------------------------------
 * Non-local-means denoising (not in PAPER.md -- BASELINE.json north_star;
 * definition DESIGN.md R11-R14):
 *   d2(p,q) = (1/(2P+1)^2) sum_{t in [-P,P]^2} (src_B(p+t) - src_B(q+t))^2,
 *   w = exp(-d2/h^2), out(p) = sum_{q in p+[-S,S]^2} w src_B(q) / sum w.
 * patch_radius P in [0,3], search_radius S in [0,10]; h > 0 or +INF
 * (box mean); h <= 0 or NaN -> ICL_ERR_INVALID_ARG.
 * The box-sum variants re-associate d2 (sliding sums); "sym_tmem" /
 * "sym_ring" also use d_{-o}(p) = d_o(p-o) (R30: one weight per
 * pair of offsets) and hold num/den in tensor memory -- results agree with
 * the direct definition to the NLM tolerance, not bit for bit.
 * ---------------------------------------------------------------------- */
icl_status icl_nlm(const icl_image* src, const icl_image* dst, int patch_radius, int search_radius,
                   float h, icl_border border, float border_value, const icl_band* band,
                   void* stream);

/* ------------------------------------------------------------------------
 * Non-separable 2-D convolution of an 8-bit image -- the paper's third
 * benchmark (§6: "a 8192x8192 image with pixels of type
 * unsigned char, a 5x5 filter, and clamped boundary condition"; the filter
 * values are a run-time input; Table 3;
 * SURVEY.md §8(f) row 1):
 *     out(x,y) = sum_{j=-r..r} sum_{i=-r..r} filter[(j+r)*(2r+1) + (i+r)] * src_B(x+i, y+j)
 * (correlation, R1; fp32 output, R22).  src: uint8 pixels
 * (element size 1, own pitch); dst: fp32; same width / height / batch.
 * radius r in [0, 3] (> 3 -> ICL_ERR_UNSUPPORTED); filter: HOST array of
 * (2r+1)^2 finite floats, row j major, copied during the call (the
 * constant-memory analog).  border_value: the constant-mode pixel value
 * (any finite float).  Every variant evaluates, per output, one fp32 FMA
 * chain over j = -r..r then i = -r..r starting from +0 with the pixel
 * converted exactly to fp32, so variants and band splits are bit-identical.
 * ---------------------------------------------------------------------- */
icl_status icl_conv2d_u8(const icl_image* src, const icl_image* dst, const float* filter, int radius,
                         icl_border border, float border_value, const icl_band* band, void* stream);

/* ------------------------------------------------------------------------
 * Row-band sharding of one large image over the GPUs of a node (SURVEY.md
 * §8(b) "icl_comm_init / icl_*_sharded", §8(e); BASELINE.json configs[3]).
 * Rank k of N owns global rows [r0, r1) = [k*ceil(H/N), min(r0+ceil(H/N), H))
 * and keeps them in a BAND BUFFER holding rows [s0, s1) = [max(0, r0-up),
 * min(H, r1+down)), where up/down are the filter's stencil rows
 * (icl_halo_rows).  A sharded call exchanges the halo rows [s0, r0) and
 * [r1, s1) with ranks k-1 / k+1 by one grouped ncclSend / ncclRecv per
 * neighbour on the comm's stream, computes the rows that need no halo on
 * `stream` meanwhile, and the edge rows after the join.  The filter runs on
 * the band through icl_band (boundary in global coordinates), so the stitched
 * result equals the unsharded call (bit for bit for sepconv, Harris and
 * conv2d).  Collective: every rank calls with the same parameters.
 * NCCL is loaded at run time (libnccl.so.2; the copy torch mapped, if any).
 * ---------------------------------------------------------------------- */
typedef struct icl_comm icl_comm;

/* Stencil rows above / below an output row: sepconv p0 = ry; Harris p0 =
 * block (floor(B/2)+1 above, B-floor(B/2) below); NLM p0 = patch, p1 =
 * search radius (P+S each side); conv2d p0 = radius. */
icl_status icl_halo_rows(icl_filter filter, int p0, int p1, int* up, int* down);
/* out = {r0, r1, s0, s1} of `rank`; ICL_ERR_INVALID_ARG when N > 1 and a
 * band is thinner than max(up, down) (out is still filled). */
icl_status icl_shard_band(int64_t global_height, int nranks, int rank, int up, int down, int64_t out[4]);
/* The rank's exchange: *n <= 2 entries {peer, send_row0, send_row1,
 * recv_row0, recv_row1} (global rows), symmetric between neighbours. */
icl_status icl_shard_plan(int64_t global_height, int nranks, int rank, int up, int down, int64_t plan[10], int* n);
/* 128-byte NCCL unique id (rank 0 creates it; the caller broadcasts it). */
icl_status icl_comm_unique_id(void* id128);
icl_status icl_comm_init(icl_comm** comm, int nranks, int rank, const void* id128);
icl_status icl_comm_destroy(icl_comm* comm);
/* In-process loopback transport (test plumbing for the exchange path, SURVEY.md
 * §4(vi)): creates `nranks` communicators of ONE process on the current
 * device, written to comms[0..nranks-1].  The icl_*_sharded calls on them run
 * the same pack -> exchange -> unpack as over NCCL, the ncclSend / ncclRecv
 * pair replaced by device copies through per-(src, dst) mailboxes with NCCL's
 * matching and completion semantics.  Every rank must be driven by its OWN
 * host thread (a recv blocks the calling thread until the peer's matching
 * send is posted; a peer that never calls -> ICL_ERR_NCCL after 120 s).
 * nranks outside [1, ICL_LOCAL_MAX_RANKS] -> ICL_ERR_INVALID_ARG.  Each comm
 * is released with icl_comm_destroy. */
#define ICL_LOCAL_MAX_RANKS 16
icl_status icl_comm_init_local(icl_comm** comms, int nranks);
/* buf: the rank's band buffer (rows [s0, s1) of the global image, own rows
 * filled by the caller, halo rows filled by the call; device memory, batch
 * allowed); dst (and Harris mask): the rank's rows [r0, r1).  Shapes that do
 * not match the partition -> ICL_ERR_INVALID_ARG; NCCL failures ->
 * ICL_ERR_NCCL.  Ordered on `stream` (events on it bracket the exchange). */
icl_status icl_sepconv_sharded(icl_comm* comm, const icl_image* buf, const icl_image* dst, int64_t global_height,
                               const float* taps_x, int rx, const float* taps_y, int ry, icl_border border,
                               float border_value, void* stream);
icl_status icl_harris_sharded(icl_comm* comm, const icl_image* buf, const icl_image* response, int64_t global_height,
                              int block, float k, icl_border border, float border_value, const icl_image* mask,
                              float threshold, void* stream);
icl_status icl_nlm_sharded(icl_comm* comm, const icl_image* buf, const icl_image* dst, int64_t global_height,
                           int patch_radius, int search_radius, float h, icl_border border, float border_value,
                           void* stream);
icl_status icl_conv2d_u8_sharded(icl_comm* comm, const icl_image* buf, const icl_image* dst, int64_t global_height,
                                 const float* filter, int radius, icl_border border, float border_value,
                                 void* stream);

/* Separable convolution of a 3-D volume (ImageCL Images support "2D/3D
 * indexing"):
 *     out(x,y,z) = sum_k h_k sum_j g_j sum_i f_i in_B(x+i, y+j, z+k)
 * (correlation on every axis, the boundary per axis, R26).  A
 * volume is an icl_image whose batch axis is z: batch = depth,
 * batch_stride_bytes = the slice stride.  Taps: HOST pointers, 2r+1 each,
 * radii 0..7 (> 7 -> ICL_ERR_UNSUPPORTED; so are slices of 2 GiB or more).
 * Device volumes only; src and dst
 * must not overlap (ICL_ERR_ALIASING); shapes must match.  All variants
 * evaluate the same fp32 chains (bit-identical).  Enqueues on stream. */
icl_status icl_sepconv3d(const icl_image* src, const icl_image* dst, const float* taps_x, int rx, const float* taps_y,
                         int ry, const float* taps_z, int rz, icl_border border, float border_value, void* stream);

/* Two-filter pipeline in one pass (FAST-style filter
 * chains, §2.2): separable smoothing then Harris,
 *     blurred  = icl_sepconv(src, taps_x, rx, taps_y, ry, blur_border, ...)
 *     response = icl_harris(blurred, block, k, border, ...)   (+ mask)
 * without the intermediate image in memory (9 B/px of HBM traffic instead
 * of 8 + 9).  Every blurred value is the sepconv fp32 chain and the Harris
 * stage is the shfl kernel's, so the result equals the two calls bit for bit.
 * Layout/ownership as icl_harris; src must not alias response/mask.  Device
 * images only, 16-byte aligned data/pitches (mask 4-byte).  band: as
 * icl_harris, with the halo grown by max(rx, ry) rows (rows the blur needs).
 * Schedules: with workspace_bytes >= icl_blur_harris_workspace_bytes(...)
 * (device memory, 16-byte aligned, owned by the caller) the chain runs as
 * the two calls through that intermediate -- faster on B200, where Harris is
 * issue-bound; with no workspace (NULL / too small) it runs
 * fused.  Both give the same bits.
 * Errors: rx or ry > 3, block 6..7, batch > 65535 -> ICL_ERR_UNSUPPORTED;
 * host images, bad arguments -> ICL_ERR_INVALID_ARG (validation of
 * icl_sepconv + icl_harris); ICL_ERR_ALIASING as icl_harris, or a workspace
 * overlapping an image. */
icl_status icl_blur_harris(const icl_image* src, const icl_image* response, const float* taps_x, int rx,
                           const float* taps_y, int ry, icl_border blur_border, float blur_border_value, int block,
                           float k, icl_border border, float border_value, const icl_image* mask, float threshold,
                           const icl_band* band, void* workspace, size_t workspace_bytes, void* stream);
/* Bytes of intermediate icl_blur_harris's two-pass schedule needs for a
 * response of width x height x batch (height: the rows the call produces). */
size_t icl_blur_harris_workspace_bytes(int64_t width, int64_t height, int64_t batch, int block);

/* ------------------------------------------------------------------------
 * Row bands with the halo read in the kernel from the neighbours' memory
 * (in-kernel NVLink halo reads instead of send/recv).
 * ---------------------------------------------------------------------- */

/* CUDA IPC export of a device pointer: a 64-byte handle of its allocation
 * plus the pointer's byte offset inside it (send both to the other ranks). */
icl_status icl_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset);
/* Map a handle from another process of this node; *dev_ptr = base + offset.
 * Errors: ICL_ERR_CUDA with the runtime's message (e.g. same process). */
icl_status icl_ipc_open(const void* handle64, uint64_t offset, void** dev_ptr);
icl_status icl_ipc_close(void* dev_ptr, uint64_t offset);

/* Pull this rank's halo rows straight from the neighbours' bands (peer loads
 * in a copy kernel over NVLink; no NCCL, no staging): buf holds global rows
 * [buf_y0, buf_y0 + buf->height) with the owned rows [own_y0, own_y1) inside;
 * rows [buf_y0, own_y0) come from the last rows of `up` (the up neighbour's
 * owned rows, ending at own_y0), rows [own_y1, end) from the first rows of
 * `down` (starting at own_y1).  elem_bytes 4 (fp32) or 1 (uint8).  Then any
 * filter runs on buf through icl_band as in icl_*_sharded -- the generic
 * peer-memory form of the halo exchange for every filter; icl_sepconv_peer
 * goes further and reads the peers inside the filter kernel.  Ordering as
 * icl_sepconv_peer.  Errors: geometry -> ICL_ERR_INVALID_ARG; rows not
 * 4-byte aligned -> ICL_ERR_UNSUPPORTED. */
icl_status icl_halo_pull(const icl_image* buf, int64_t global_height, int64_t buf_y0, int64_t own_y0,
                         int64_t own_y1, const icl_image* up, const icl_image* down, int elem_bytes, void* stream);

/* ------------------------------------------------------------------------
 * The same in-kernel halo reads over NCCL symmetric memory (SURVEY.md
 * §8(f) row 3; NCCL >= 2.28): every rank allocates its band buffer with
 * icl_comm_mem_alloc (ncclMemAlloc) and registers it COLLECTIVELY as a
 * symmetric window (icl_comm_window_register: ncclCommWindowRegister with
 * NCCL_WIN_COLL_SYMMETRIC; every rank passes the same size).  A neighbour's
 * band is then named by (peer rank, byte offset of its first held row in the
 * peer's window, height, pitch, batch stride) -- icl_window_band -- and the
 * edge kernels resolve the address ON THE DEVICE with ncclGetPeerPointer(win,
 * offset, peer) (the NVLink mapping of the peer's buffer) and load the rows
 * directly: no staging buffer, send/recv or pack/unpack.  Semantics, results
 * (bit for bit) and ordering are those of icl_sepconv_peer /
 * icl_harris_peer / icl_halo_pull: the caller orders the writes of the bands
 * and the reads with a cross-rank barrier.  `peer` < 0: no neighbour on that
 * side.  The window API needs an NCCL communicator (icl_comm_init; not the
 * loopback one) and a libnccl.so.2 with the symmetric-memory symbols, else
 * ICL_ERR_UNSUPPORTED.  Tested here at N = 1 (one GPU per test box: NCCL
 * refuses two ranks on a device) with the neighbour bands placed in the
 * rank's own window (peer 0), which runs the device-side resolution and the
 * window loads end to end.
 * ---------------------------------------------------------------------- */
typedef struct icl_window icl_window;
typedef struct {
  int peer;                    /* rank holding the band; < 0: none */
  uint64_t offset;             /* byte offset of the band's first row (image 0) in that rank's window */
  int64_t height;              /* rows held */
  int64_t pitch_bytes, batch_stride_bytes;
} icl_window_band;
icl_status icl_comm_mem_alloc(icl_comm* comm, size_t bytes, void** ptr);
icl_status icl_comm_mem_free(icl_comm* comm, void* ptr);
icl_status icl_comm_window_register(icl_comm* comm, void* buf, size_t bytes, icl_window** win);
icl_status icl_comm_window_deregister(icl_comm* comm, icl_window* win);
icl_status icl_sepconv_window(const icl_window* win, const icl_image* own, const icl_image* dst,
                              int64_t global_height, int64_t own_y0, const icl_window_band* up,
                              const icl_window_band* down, const float* taps_x, int rx, const float* taps_y, int ry,
                              icl_border border, float border_value, void* stream);
icl_status icl_harris_window(const icl_window* win, const icl_image* own, const icl_image* response,
                             int64_t global_height, int64_t own_y0, const icl_window_band* up,
                             const icl_window_band* down, int block, float k, icl_border border, float border_value,
                             const icl_image* mask, float threshold, void* stream);
icl_status icl_halo_pull_window(const icl_window* win, const icl_image* buf, int64_t global_height, int64_t buf_y0,
                                int64_t own_y0, int64_t own_y1, const icl_window_band* up,
                                const icl_window_band* down, int elem_bytes, void* stream);

/* Separable convolution of the global rows [own_y0, own_y0 + own->height) of
 * an image of global_height rows whose row bands live on different GPUs.
 * own: this rank's rows ONLY (no halo rows); up / down: the neighbouring
 * ranks' bands (device pointers mapped with icl_ipc_open, or any device
 * memory this GPU can read) -- `up` ends at global row own_y0, `down` starts
 * at own_y0 + own->height; either may be NULL at the image edge.  The rows
 * that need no halo run on the ordinary kernels; the edge rows' kernel loads
 * its input rows from `own`, `up` or `down` directly (peer loads over NVLink):
 * no staging, no send/recv.  The boundary applies at the GLOBAL edges, so the
 * stitched outputs equal the unsharded icl_sepconv bit for bit.  Ordering: the
 * neighbours' rows must be complete before the call's kernels run and stay
 * unchanged until they finish (bracket the call with a cross-rank barrier).
 * Errors: geometry (dst shape != own, neighbour missing or thinner than ry
 * rows where needed, radius > 15) -> ICL_ERR_INVALID_ARG. */
icl_status icl_sepconv_peer(const icl_image* own, const icl_image* dst, int64_t global_height, int64_t own_y0,
                            const icl_image* up, const icl_image* down, const float* taps_x, int rx,
                            const float* taps_y, int ry, icl_border border, float border_value, void* stream);
/* Harris on one rank's rows, the same contract as icl_sepconv_peer: own holds
 * only this rank's rows; the edge rows (floor(block/2)+1 above and
 * block-floor(block/2) below, where a neighbour exists) run a kernel whose
 * input loads resolve to the own band or directly to `up` / `down`; the rest
 * runs on the ordinary Harris kernels.  Stitched responses and masks equal
 * the unsharded icl_harris bit for bit (one fp32 order, per-stage boundary in
 * GLOBAL coordinates).  Errors: geometry, block outside [1, 7] ->
 * ICL_ERR_INVALID_ARG; otherwise as icl_harris. */
icl_status icl_harris_peer(const icl_image* own, const icl_image* response, int64_t global_height, int64_t own_y0,
                          const icl_image* up, const icl_image* down, int block, float k, icl_border border,
                          float border_value, const icl_image* mask, float threshold, void* stream);

/* ------------------------------------------------------------------------
 * Variant space + auto-tuner (§4, Table 1 lines
 * 364-393).
 * ---------------------------------------------------------------------- */

/* Tagged union of the filter calls' arguments. */
typedef struct {
    icl_filter filter;
    icl_image src;
    icl_image dst; /* sepconv out / harris response / nlm out */
    icl_border border;
    float border_value;
    /* sepconv */
    const float* taps_x;
    int rx;
    const float* taps_y;
    int ry;
    void* workspace;
    size_t workspace_bytes;
    /* harris */
    int block;
    float k;
    icl_image mask; /* mask.data == NULL -> no mask */
    float threshold;
    /* nlm */
    int patch_radius;
    int search_radius;
    float h;
    /* conv2d (src is the uint8 image) */
    const float* filter2d;
    int radius2d;
} icl_problem;

typedef struct {
    int variant_id;
    char name[96];
    float median_us;  /* median of the timed launches of the winner */
    int n_candidates; /* eligible variants timed */
    int n_rejected;   /* variants whose output differed from the naive one */
    int from_cache;   /* 1 if the answer came from the cache */
} icl_variant_info;

#define ICL_TUNE_FORCE 1u     /* re-time even if the key is cached */
#define ICL_TUNE_NO_VERIFY 2u /* skip the equivalence check against the naive variant */

/* Time every eligible variant for this problem (CUDA events, median of >= 10
 * launches after warm-up), reject any whose output differs from the naive
 * variant (bit-exact for sepconv, tolerance for Harris/NLM), cache the
 * fastest per problem key (ties within 0.5% -> lower id).  Synchronises.
 * Leaves the winner's result in dst. */
/* (device-resident images only; host images -> ICL_ERR_INVALID_ARG) */
icl_status icl_tune(const icl_problem* problem, unsigned flags, void* stream, icl_variant_info* chosen);

/* Model-guided tuning (§4: "execute the code of several
 * randomly selected parameter configurations ... build an artificial neural
 * network performance model ... predict the execution time of all possible
 * configurations ... some of the configurations with the best predicted
 * execution times are executed, and the configuration with the best actual
 * execution time of these is returned").  Like icl_tune, but phase 1 times n1
 * randomly drawn eligible variants (seeded), phase 2 fits the surrogate
 * (ann.cu; R23) to their log median times and times the topk
 * best-predicted untimed variants; the fastest verified variant is cached.
 * n1 >= number of eligible variants degenerates to icl_tune (exhaustive).
 * chosen->n_candidates = variants actually timed.  Synchronises.
 * Errors: as icl_tune; n1 < 1 or topk < 0 -> ICL_ERR_INVALID_ARG. */
icl_status icl_tune_ann(const icl_problem* problem, int n1, int topk, uint64_t seed, void* stream,
                        icl_variant_info* chosen);

/* The surrogate and the two-phase search on their own, for any
 * configuration space (host only, no GPU).  features: row-major
 * [n_configs][n_features] numeric encoding of each configuration.
 * evaluate(ctx, i, &value) returns 0 and a value > 0 (e.g. a time) on success,
 * non-zero for a failed configuration (kept out of training).  evaluated
 * (nullable, n_configs ints) receives the indices in evaluation order.
 * Errors: bad arguments -> ICL_ERR_INVALID_ARG; every evaluation failed ->
 * ICL_ERR_UNSUPPORTED (best_index = -1). */
typedef int (*icl_eval_fn)(void* ctx, int index, double* value);
icl_status icl_ann_search(const double* features, int n_configs, int n_features, icl_eval_fn evaluate, void* ctx,
                          int n1, int topk, uint64_t seed, int* best_index, double* best_value, int* evaluated,
                          int* n_evaluated);
/* Fit the surrogate to n >= 10 samples (value > 0, modelled as log value) and
 * return its final standardised training MSE and (nullable) its predictions
 * at the training points.  Fewer than 10 samples -> ICL_ERR_INVALID_ARG. */
icl_status icl_ann_fit(const double* X, const double* value, int n, int n_features, uint64_t seed, double* final_loss,
                       double* pred_value);

/* Persist / restore the winner cache (JSON; keyed by device name, SM count
 * and library version + problem key -- the "final implementation" of
 * PAPER.md:233-234). */
icl_status icl_tune_cache_save(const char* path);
icl_status icl_tune_cache_load(const char* path);
void icl_tune_cache_clear(void);
int icl_tune_cache_size(void);

/* Variant registry.  Ids are stable within a library build. */
int icl_variant_count(icl_filter filter);
icl_status icl_variant_name(icl_filter filter, int variant_id, char* buf, size_t buf_len);

/* Force a variant for subsequent calls on the CALLING thread (the "force
 * on/off" directive analog); -1 restores automatic
 * dispatch.  A forced variant that is ineligible for a call makes that call
 * fail with ICL_ERR_UNSUPPORTED (or ICL_ERR_WORKSPACE). */
icl_status icl_force_variant(icl_filter filter, int variant_id);

/* Variant the last successful call of `filter` on this thread dispatched to. */
int icl_last_variant(icl_filter filter);

/* Number of kernel launches this library issued on the calling process since
 * load (for the bench's gpu_launches claim). */
uint64_t icl_launch_count(void);

/* Cumulative host->device / device->host bytes the host-image path copied
 * (either pointer may be NULL). */
void icl_transfer_bytes(uint64_t* h2d, uint64_t* d2h);

/* ------------------------------------------------------------------------
 * Misc
 * ---------------------------------------------------------------------- */
const char* icl_last_error(void);
const char* icl_version(void);
/* Fill a device fp32 image with the synthetic U[0,1) SplitMix64 stream of
 * synth.uniform_image(seed, ...) (input generation for large benches; holds
 * no filter arithmetic).  Pixel (x, y) of image b uses counter
 * (row0 + y)*width + x and seed (seed + b). */
icl_status icl_fill_uniform(const icl_image* img, uint64_t seed, int64_t row0, void* stream);
/* Enqueue a 2-D copy of `rows` rows of width_bytes between any two pointers the CUDA runtime
 * can address (device, pinned host, NCCL symmetric memory) on `stream` (plumbing for callers
 * holding raw allocations, e.g. icl_comm_mem_alloc buffers). */
icl_status icl_copy_2d(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width_bytes, int64_t rows,
                       void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ICL_H_ */
