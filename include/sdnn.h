/*
 * sdnn.h -- C ABI of libsdnn.so, the B200 (sm_100a) Sparse DNN inference
 * engine.  Plain pointers and sizes only; the caller owns every host buffer,
 * a handle owns its device memory.
 *
 * The reference (sdnnbench, /root/reference/pkg/src/sdnnbench) has no FFI:
 * its boundary is the Python functions below, so each entry point names the
 * reference function it replaces.  The Python mirror
 * (paper_1909_05631_b200/engine.py) binds them with ctypes; INTEGRATION.md
 * shows the binding a reference maintainer would add.
 *
 *   reference                                   this ABI
 *   engine.infer            engine.py:300-324   sdnn_net_* + sdnn_infer
 *                                               (sdnn_infer_streamed)
 *   engine.infer_timed      engine.py:327-340   sdnn_batch_upload + sdnn_run
 *                                               (+ sdnn_result_device_ms)
 *   engine._run_layers      engine.py:192-203   sdnn_run (all L layers on device)
 *   engine.spmm             engine.py:163-175   sdnn_spmm
 *   engine.apply_bias_relu_clamp  engine.py:178-184  sdnn_bias_relu_clamp
 *   challenge.categorize    challenge.py:60-67  sdnn_result_categories
 *   NetworkModel/LayerWeights model.py:128-162  sdnn_net_add_layer_csr
 *   FeatureBatch result     engine.py:158-160,324  sdnn_result_y_csr
 *   ingest.resize_threshold_flatten ingest.py:128-156  sdnn_batch_from_images
 *
 * Return codes map onto the reference's exception classes
 * (errors.py:12,46,50):  0 ok, 2 ParameterError, 3 CapacityError (also any
 * CUDA failure), 4 ShapeError.  sdnn_last_error() gives the message of the
 * calling thread's last failure.
 *
 * Threading: distinct handles may be used concurrently from different host
 * threads (one handle per GPU is the data-parallel layout); one handle must
 * not be used by two threads at once.
 */
#ifndef SDNN_H
#define SDNN_H

#include <stdint.h>

#include "sdnn_gen.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SDNN_OK 0
#define SDNN_ERR_PARAMETER 2
#define SDNN_ERR_CAPACITY 3
#define SDNN_ERR_SHAPE 4

#define SDNN_F32 0 /* activations and weights stored/computed in float  */
#define SDNN_F64 1 /* float64: bit-exact with the reference engine      */

typedef struct sdnn_net sdnn_net;       /* device-resident network      */
typedef struct sdnn_batch sdnn_batch;   /* device-resident input Y0     */
typedef struct sdnn_result sdnn_result; /* outputs of one run           */

int sdnn_version(void);
const char *sdnn_last_error(void);
int sdnn_device_count(int *n);

/* A network of n_neurons x n_neurons layers on CUDA device `device`. */
int sdnn_net_create(int device, int dtype, int64_t n_neurons, sdnn_net **out);
void sdnn_net_destroy(sdnn_net *net);

/* Append one layer given as the reference's LayerWeights: CSR by input row
 * (model.py:51-125: row_offsets[n+1], col_indices[nnz] ascending per row,
 * values[nnz]) and its scalar bias.  Converted once to the device layout
 * (ELL by output column, inputs ascending).  Untimed, like model loading
 * in the reference (engine.py:329-332). */
int sdnn_net_add_layer_csr(sdnn_net *net, const int64_t *w_off, const int64_t *w_cols,
                           const double *w_vals, int64_t nnz, double bias);

/* Append one layer already in ELL-by-output form: idx[j*width + s] is the
 * s-th smallest input feeding output j, vals likewise (n*width each). */
int sdnn_net_add_layer_ell(sdnn_net *net, int32_t width, const int32_t *idx,
                           const double *vals, double bias);

/* Generate `count` perm-union layers (sdnn_gen_permunion_ell) with `threads`
 * host threads and append them, every slot holding `value`. */
int sdnn_net_add_layers_permunion(sdnn_net *net, uint64_t seed, int64_t first_layer,
                                  int64_t count, int32_t width, double value,
                                  double bias, int threads);

/* Multi-GPU weight replication (weights are replicated once,
 * untimed, from GPU 0 over NVLink).  sdnn_net_add_layers_uninit appends
 * `count` layers of ELL width `width` whose device buffers are left for the
 * caller to fill (e.g. an NCCL broadcast from rank 0); sdnn_net_layer_buffers
 * exposes a layer's device buffers: idx int32 [n][wp] (-1 = padding) and
 * val (T) [n][wp], wp = width padded to a multiple of 32. */
int sdnn_net_add_layers_uninit(sdnn_net *net, int64_t count, int32_t width, double bias);
int sdnn_net_layer_buffers(const sdnn_net *net, int64_t layer, void **idx, void **val,
                           int32_t *wp, int64_t *val_bytes);

int sdnn_net_n_layers(const sdnn_net *net, int64_t *n);
/* Device bytes held by the weights (for the roofline byte model). */
int sdnn_net_weight_bytes(const sdnn_net *net, int64_t *bytes);

/* Stage Y0 (FeatureBatch, CSR) on the device.  Untimed input placement. */
int sdnn_batch_upload(sdnn_net *net, int64_t n_rows, const int64_t *y_off,
                      const int64_t *y_cols, const double *y_vals, sdnn_batch **out);
/* A batch lives in its network's stream and memory pool: free it before
 * sdnn_net_destroy of that network. */
void sdnn_batch_free(sdnn_batch *batch);
/* ingest.resize_threshold_flatten (ingest.py:128-156) on the device: n_images
 * square uint8 images of side x side pixels (ImageSet.pixels, row-major)
 * -> pixels / 255, bilinear resample to target_side (32, 64, 128 or 256, the
 * reference's TARGET_SIDES; ParameterError otherwise), threshold >= 0.5,
 * flatten row-major: a binary batch staged on the device, bit-identical to
 * the reference's FeatureBatch.  ShapeError unless target_side^2 equals the
 * network's neuron count. */
int sdnn_batch_from_images(sdnn_net *net, int64_t n_images, int32_t side, const uint8_t *pixels,
                           int32_t target_side, sdnn_batch **out);
/* The pipeline hand-off (engine._infer_pipeline, engine.py:254-297): the
 * final Y of a run made with sdnn_run_y becomes the staged input of the
 * next layer range on `net` without leaving the device -- a device-to-device
 * copy, or a peer copy over NVLink when `net` is on another GPU.  ShapeError
 * unless the result's width equals the network's neuron count. */
int sdnn_batch_from_result(sdnn_net *net, const sdnn_result *result, sdnn_batch **out);
/* A staged batch back as host CSR (values 1.0 for a binary batch; cols and
 * vals may be null): query nnz first. */
int sdnn_batch_nnz(const sdnn_batch *batch, int64_t *nnz);
int sdnn_batch_csr(const sdnn_batch *batch, int64_t *off, int64_t *cols, double *vals);
/* Bytes the upload copied host -> device (offsets, columns as uint16 when
 * the row length is <= 65536 else int32, values unless all are 1.0). */
int sdnn_batch_h2d_bytes(const sdnn_batch *batch, int64_t *bytes);

/* Run layers [first_layer, first_layer + n_layers) over a staged batch and
 * build the category list (the reference's timed region,
 * engine.py:336-339).  n_layers < 0 means all remaining layers. */
int sdnn_run(sdnn_net *net, const sdnn_batch *batch, double ymax, int64_t first_layer,
             int64_t n_layers, sdnn_result **out);

/* sdnn_run that also materialises the final Y for sdnn_result_y_csr. */
int sdnn_run_y(sdnn_net *net, const sdnn_batch *batch, double ymax, int64_t first_layer,
               int64_t n_layers, sdnn_result **out);

/* engine.infer end to end: host CSR in, result (with Y) out. */
int sdnn_infer(sdnn_net *net, int64_t n_rows, const int64_t *y_off, const int64_t *y_cols,
               const double *y_vals, double ymax, sdnn_result **out);

/* engine.infer end to end with the upload hidden behind the run: Y0 is cut
 * into `segments` row segments of about equal nnz (0 = automatic: one per
 * ~96M entries, at most 6); a second host thread converts and uploads
 * segment s+1 on its own stream while segment s runs.  Rows are independent
 * (engine.py:237-251), so the result equals the one-shot run bit for bit.
 * want_y = 0 skips materialising Y (categories only).  sdnn_infer is this
 * call with want_y = 1 and automatic segments. */
int sdnn_infer_streamed(sdnn_net *net, int64_t n_rows, const int64_t *y_off, const int64_t *y_cols,
                        const double *y_vals, double ymax, int want_y, int segments, sdnn_result **out);
/* Host -> device bytes an end-to-end call copied, and its row segments. */
int sdnn_result_h2d_bytes(const sdnn_result *r, int64_t *bytes);
int sdnn_result_segments(const sdnn_result *r, int64_t *n);

/* Category list: 1-based rows of the final Y holding any entry, ascending. */
int sdnn_result_n_categories(const sdnn_result *r, int64_t *n);
int sdnn_result_categories(const sdnn_result *r, int64_t *buf);
/* Device time of the layer loop (CUDA events) and host wall time of the
 * whole call, milliseconds. */
double sdnn_result_device_ms(const sdnn_result *r);
double sdnn_result_wall_ms(const sdnn_result *r);
/* live_rows[l] = rows with an entry entering layer l (l = 0..n_layers),
 * live_rows[n_layers] = rows alive at the end. */
int sdnn_result_n_layers(const sdnn_result *r, int64_t *n);
int sdnn_result_live_rows(const sdnn_result *r, int64_t *live_rows);
/* Profiling pass: record a CUDA event around every layer launch of later
 * runs on this handle (off by default; adds one event per layer). */
int sdnn_net_set_layer_timing(sdnn_net *net, int on);
/* Per-layer device milliseconds of a run made with layer timing on. */
int sdnn_result_layer_ms(const sdnn_result *r, double *ms);
/* Device milliseconds of the run's launches, from CUDA events recorded on
 * the engine's stream in every run: ms[0] = live-row select + Y0 expansion into tiles
 * (densify), ms[1] = the first layer's own launch over bit-line tiles (0
 * when Y0 is not binary), ms[2] = the persistent launch over the remaining
 * layers. */
int sdnn_result_stage_ms(const sdnn_result *r, double *ms);
/* Kernel launches the run issued (evidence for bench gpu_launches). */
int sdnn_result_launches(const sdnn_result *r, int64_t *n);
/* Live-row compaction: before a layer, the live rows
 * are repacked densely into tiles when that frees at least `pct` % of the
 * live tiles (default 10; <= 0 never; the SDNN_COMPACT environment variable
 * overrides) and at least 16 tiles (SDNN_COMPACT_MIN).  Results are
 * bit-identical either way.  No reference
 * counterpart: the reference's CSR rows carry no dead-row cost. */
int sdnn_net_set_compaction(sdnn_net *net, int pct);
/* Row compactions the run performed (summed over waves / segments). */
int sdnn_result_compactions(const sdnn_result *r, int64_t *n);
/* Output pruning by line bounds.  Every stored line of activations (one
 * neuron over a tile of rows) carries an upper bound of its largest |value|.
 * For one output neuron of a tile, |chain| <= sum over its weight slots of
 * |w| * (bound of the slot's input line); when that sum, with a margin far
 * above the rounding of the chain, stays below -bias, the epilogue
 * (engine.py:129-133: keep v = z + bias only when v > 0) stores nothing for
 * any row of the tile, so the column gathers no line at all.  Data-dependent
 * and exact: results are bit-identical with pruning off (on by default;
 * `on` = 0 or SDNN_PRUNE=0 turns it off).  It uses no property of the weight
 * values or of the layers beyond this run's own activations (PAPER.md
 * avoid-list).  No reference counterpart: the reference's Gustavson product
 * only ever touches stored entries. */
int sdnn_net_set_pruning(sdnn_net *net, int on);
/* (tile, output) columns the run pruned (summed over layers / waves). */
int sdnn_result_pruned(const sdnn_result *r, int64_t *n);
/* Final Y as canonical CSR (ascending columns, no zeros) widened to
 * float64: query nnz first, then fill caller buffers. */
int sdnn_result_y_nnz(sdnn_result *r, int64_t *nnz);
int sdnn_result_y_csr(sdnn_result *r, int64_t *off, int64_t *cols, double *vals);
void sdnn_result_free(sdnn_result *r);

/* ---- One handle over several GPUs -------------------
 * engine._infer_data_parallel (engine.py:237-251) with one GPU per worker:
 * every member holds a full weight replica; sdnn_group_infer splits the
 * batch into contiguous row blocks of ceil(B / G) rows (engine.py:240), runs
 * each block on its GPU from its own host thread (sdnn_infer_streamed:
 * upload overlapped with the run), and merges the results in row order --
 * bit-identical to one GPU.  Device time of a group result is the slowest
 * member's (they run concurrently); launches, live rows, H2D bytes add up. */
typedef struct sdnn_group sdnn_group;
/* GPUs 0 .. n_gpus-1 (n_gpus <= 0: every visible GPU). */
int sdnn_open(int n_gpus, int dtype, int64_t n_neurons, sdnn_group **out);
/* An explicit device list (a device may appear more than once). */
int sdnn_open_devices(const int *devices, int n_devices, int dtype, int64_t n_neurons,
                      sdnn_group **out);
void sdnn_close(sdnn_group *group);
int sdnn_group_size(const sdnn_group *group, int *n);
/* Member i's single-GPU handle (owned by the group; NULL if out of range). */
sdnn_net *sdnn_group_net(sdnn_group *group, int i);
/* Layers are converted once on the first member and replicated to the
 * others device to device (peer copies over NVLink/NVSwitch). */
int sdnn_group_add_layer_csr(sdnn_group *group, const int64_t *w_off, const int64_t *w_cols,
                             const double *w_vals, int64_t nnz, double bias);
int sdnn_group_add_layers_permunion(sdnn_group *group, uint64_t seed, int64_t first_layer,
                                    int64_t count, int32_t width, double value, double bias,
                                    int threads);
int sdnn_group_infer(sdnn_group *group, int64_t n_rows, const int64_t *y_off,
                     const int64_t *y_cols, const double *y_vals, double ymax, int want_y,
                     sdnn_result **out);

/* engine.spmm: Z = Y * W (n_rows x n_inner times n_inner x n_out), exact
 * zeros dropped, no epilogue.  Result Y is Z. */
int sdnn_spmm(int device, int dtype, int64_t n_rows, int64_t n_inner, int64_t n_out,
              const int64_t *y_off, const int64_t *y_cols, const double *y_vals,
              const int64_t *w_off, const int64_t *w_cols, const double *w_vals,
              sdnn_result **out);

/* engine.apply_bias_relu_clamp on a CSR matrix. */
int sdnn_bias_relu_clamp(int device, int dtype, int64_t n_rows, int64_t n_cols,
                         const int64_t *off, const int64_t *cols, const double *vals,
                         double bias, double ymax, sdnn_result **out);

#ifdef __cplusplus
}
#endif

#endif
