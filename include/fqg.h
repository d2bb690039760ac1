/* fqg.h — C ABI of the B200 (sm_100a) FlattenQuant linear-layer hot path.
 *
 * This is the drop-in boundary for the reference's operator API
 * (/root/reference/proj/core/include/fq/{flatten,quantize,pipeline}.hpp, namespace fq). Every entry point
 * names the reference interface it replaces. Plain pointers and sizes only;
 * device pointers are marked *_dev, streams are cudaStream_t passed as void*.
 *
 * Errors: every function returns an fqg_status. The message of the last
 * failure on the calling thread is in fqg_last_error(). The C++ shim
 * (include/fq_gpu.hpp) maps FQG_ERR_INVALID -> std::invalid_argument and
 * FQG_ERR_RUNTIME -> std::runtime_error, the exception types the reference
 * throws for the same conditions (pipeline.cpp:161-163, flatten.cpp:92-94,
 * quantize.cpp:37). There is no CPU fallback: without a usable sm_100 device
 * every compute entry point fails with FQG_ERR_CUDA.
 *
 * Layer handles are immutable after creation; fqg_layer_forward is
 * stream-ordered and may be called concurrently on different streams.
 */
#ifndef FQG_H
#define FQG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fqg_status {
    FQG_OK = 0,
    FQG_ERR_INVALID = -2,     /* std::invalid_argument in the reference */
    FQG_ERR_RUNTIME = -3,     /* std::runtime_error in the reference   */
    FQG_ERR_CUDA = -4,        /* CUDA / device failure (no fallback)   */
    FQG_ERR_UNSUPPORTED = -5  /* shape/format outside this build       */
} fqg_status;

typedef enum fqg_dtype {
    FQG_F64 = 0,
    FQG_F32 = 1,
    FQG_F16 = 2,
    FQG_BF16 = 3,
    FQG_I32 = 4, /* raw INT32 accumulators (bit-exact debug dump)          */
    FQG_I8 = 5,  /* int8 operand, one value per byte                       */
    FQG_I4 = 6,  /* packed int4 operand: per group g of 32 consecutive k,
                    byte 16g + i = q[32g + i] & 15 | q[32g + 16 + i] << 4 */
    FQG_NONE = 7
} fqg_dtype;

/* Activation-scale mode. STATIC is the reference inference path
 * (act_scale = T_x / qmax, pipeline.cpp:138,167). DYNAMIC is the opt-in
 * per-tensor absmax mode whose oracle is quantize_per_tensor without an
 * override (quantize.cpp:34-40), computed per call on the device. */
typedef enum fqg_scale_mode { FQG_SCALE_STATIC = 0, FQG_SCALE_DYNAMIC = 1 } fqg_scale_mode;

typedef struct fqg_layer_s* fqg_layer_t;

/* The frozen recipe of one linear layer: the fields of fq::LayerQuantConfig
 * (pipeline.hpp:37-49) that fq::run_layer reads, as plain arrays. */
typedef struct fqg_layer_desc {
    int bits;                     /* 4 or 8 (LayerQuantConfig::bits)              */
    int64_t k;                    /* input channels K                              */
    int64_t n;                    /* output channels of THIS shard                 */
    const double* smooth_scales;  /* [k] host, SmoothingScales::s                  */
    double t_x;                   /* plan_x.threshold                              */
    const int64_t* ext_x;         /* [k] host, plan_x.extensions                   */
    int64_t block_x;              /* plan_x.block (32)                             */
    double t_w;                   /* plan_w.threshold                              */
    const int64_t* ext_w;         /* [plan_x.padded_width] host, plan_w.extensions */
    int64_t block_w;              /* plan_w.block                                  */
    double act_scale;             /* LayerQuantConfig::act_scale (static s_x)      */
    /* Weights, one of:
     *  (a) weight_q != NULL: reference weight_q.q, int32 [K'][n_total] row-major
     *      (host), with w_scale = weight_q.params.scale;
     *  (b) weight != NULL: the unquantized layer weight W, f64 [k][n_total]
     *      row-major (host). The offline tail of quantize_layer
     *      (pipeline.cpp:100,114-120,139-150) runs on the device: scale_rows,
     *      repeat_channels, strict flatten_rows, per-tensor absmax -> s_w,
     *      round-to-nearest quantization; w_scale is ignored (computed). */
    const int32_t* weight_q;
    const double* weight;
    double w_scale;
    int64_t n_total;              /* columns of the full layer (== n unsharded)    */
    int64_t n_begin;              /* first column of this shard                    */
    int a_format;                 /* FQG_I8, or FQG_I4 (packed activations; bits=4) */
    int b_format;                 /* FQG_I8, or FQG_I4 (packed weights; bits=4)    */
    int scale_mode;               /* fqg_scale_mode                                */
    int device;                   /* CUDA device ordinal                           */
} fqg_layer_desc;

typedef struct fqg_layer_info {
    int bits, a_format, b_format, scale_mode;
    int64_t k, n, c1, kp, n_total, n_begin;
    double t_x, t_w, act_scale, w_scale;
    int64_t weight_bytes;         /* device bytes of the packed weight operand     */
} fqg_layer_info;

const char* fqg_last_error(void);
int fqg_version(void);

/* Replaces the construction of a runnable LayerQuantConfig (cmd_infer's
 * load_recipes, flattenquant_cli.cpp:241-252, and the weight tail of
 * fq::quantize_layer, pipeline.cpp:100,114-120,139-150): compiles the
 * composite gather map from plan_x/plan_w, quantizes/packs the weights
 * K-major on the device, uploads the per-channel tables. */
int fqg_layer_create(const fqg_layer_desc* desc, fqg_layer_t* out);
int fqg_layer_destroy(fqg_layer_t layer);
int fqg_layer_get_info(fqg_layer_t layer, fqg_layer_info* info);
/* Device copy of the quantized weight (int32 [K'][n] row-major, the
 * reference's weight_q layout for this shard) and s_w, for parity checks. */
int fqg_layer_weight_q(fqg_layer_t layer, int32_t* wq_host, double* w_scale);

/* Replaces fq::run_layer (pipeline.hpp:83-84, pipeline.cpp:159-169) on
 * device-resident data: y = dequant(int_gemm(quant(repeat(flatten(x / s))))).
 * x_dev: [m][k] of x_dtype (F64/F32/F16/BF16), y_dev: [m][ldy] of y_dtype
 * (F64/F32/F16/BF16, or I32 for the raw accumulators). bias_dev: optional
 * [n] of bias_dtype (build extension; the reference has no bias).
 * saturation_dev: optional device uint64 the call ADDS its saturation events
 * to (pipeline.hpp:80-82). Asynchronous on `stream`. */
int fqg_layer_forward(fqg_layer_t layer, const void* x_dev, int x_dtype, int64_t m, void* y_dev,
                      int y_dtype, int64_t ldy, const void* bias_dev, int bias_dtype,
                      unsigned long long* saturation_dev, void* stream);

/* N-sharding across the GPUs of a node. The layer shards along
 * N: rank r of `world` holds columns [b0, b1) = fqg_shard_bounds(n_total, world,
 * r) (create it with desc.n_begin = b0, desc.n = b1 - b0; the device weight tail
 * uses the GLOBAL s_w, so every shard is an exact column slice). Widths are
 * 32-aligned except possibly the last; `width` is the common slot width. */
int fqg_shard_bounds(int64_t n_total, int world, int rank, int64_t* b0, int64_t* b1,
                     int64_t* width);

/* The collective the caller supplies: ncclAllGather itself fits this type
 * (sendbuff, recvbuff, sendcount, ncclDataType_t, ncclComm_t, cudaStream_t; the
 * return value is ncclResult_t, 0 = success), so the library does not link or
 * load any NCCL and the caller's communicator stays with the NCCL that made it. */
typedef int (*fqg_allgather_fn)(const void* sendbuff, void* recvbuff, size_t sendcount,
                                int nccl_datatype, void* comm, void* stream);

/* Sharded fq::run_layer on device data: this rank's K1 + K4 write its column
 * shard straight into its slot of the shard-major gather buffer
 * gather_dev [world][m][width] (y_dtype F16/BF16/F32/F64), then `allgather`
 * fills the other ranks' slots in place (sendbuff = this rank's slot, count
 * m * width elements). Column c of the full output is slot c / width (for the
 * 32-aligned widths of fqg_shard_bounds: slot r holds [b0_r, b1_r)), row i at
 * [r][i][c - b0_r]; no reassembly copy is made. allgather may be NULL (world 1,
 * or a caller that gathers later). Stream-ordered. */
int fqg_layer_forward_sharded(fqg_layer_t layer, const void* x_dev, int x_dtype, int64_t m,
                              void* gather_dev, int y_dtype, int world, int rank,
                              const void* bias_dev, int bias_dtype,
                              unsigned long long* saturation_dev, fqg_allgather_fn allgather,
                              void* comm, void* stream);

/* The drop-in host call: same contract as fq::run_layer(cfg, x, saturation)
 * (pipeline.hpp:84) on host f64 buffers; copies in, runs, copies out,
 * synchronizes. y_host: [m][n] f64, equal to the reference bit for bit. */
int fqg_layer_run_host(fqg_layer_t layer, const double* x_host, int64_t m, double* y_host,
                       int64_t* saturation);

/* The activation half of run_layer (pipeline.cpp:164-167, i.e. divide_columns
 * -> flatten_tensor(saturating) -> repeat_columns -> quantize_per_tensor):
 * writes the quantized operand q_dev [m][K'] int8 (a_format I8) or
 * [m][K'/2] packed int4 (a_format I4). */
int fqg_layer_quantize_acts(fqg_layer_t layer, const void* x_dev, int x_dtype, int64_t m,
                            void* q_dev, unsigned long long* saturation_dev, void* stream);

/* The GEMM half (int_matmul, quantize.cpp:190-198) on an operand produced by
 * fqg_layer_quantize_acts. */
int fqg_layer_gemm(fqg_layer_t layer, const void* q_dev, int64_t m, void* y_dev, int y_dtype,
                   int64_t ldy, const void* bias_dev, int bias_dtype, void* stream);

/* Same two halves with the operand row sums passed between them (optional
 * rowsum_dev [m] int32). Int4 weights are stored with biased nibbles
 * (q + 8) and multiplied as unsigned; the GEMM epilogue subtracts 8 * rowsum
 * per row. fqg_layer_quantize_acts_ex writes the sums as a by-product;
 * fqg_layer_gemm (or _ex with NULL) recomputes them with an extra pass. */
int fqg_layer_quantize_acts_ex(fqg_layer_t layer, const void* x_dev, int x_dtype, int64_t m,
                               void* q_dev, int32_t* rowsum_dev, unsigned long long* saturation_dev,
                               void* stream);
int fqg_layer_gemm_ex(fqg_layer_t layer, const void* q_dev, const int32_t* rowsum_dev, int64_t m,
                      void* y_dev, int y_dtype, int64_t ldy, const void* bias_dev, int bias_dtype,
                      void* stream);

/* Standalone integer GEMM (int_matmul_raw / int_matmul, quantize.cpp:166-198):
 * a_dev [m][lda] and b_dev [n][ldb] K-major int8 (or packed int4), y as in
 * fqg_layer_forward; scale_dev: device double[2] = {s_x, s_w}; the epilogue forms s_x*s_w once in FP64 (quantize.cpp:193). */
int fqg_gemm(const void* a_dev, int a_fmt, int64_t lda, const void* b_dev, int b_fmt, int64_t ldb,
             int64_t m, int64_t n, int64_t kp, void* y_dev, int y_dtype, int64_t ldy,
             const double* scale_dev, const void* bias_dev, int bias_dtype, void* stream);

/* The launch fqg_gemm (and a layer's GEMM) makes for a shape, on the current
 * device; host-only query for tests and tooling. kernel 1: 1-CTA 128 x tile_n
 * tiles; kernel 2: CTA pair (cta_group::2) tile_m x tile_n tiles (tile_m 512:
 * two A sub-tiles); kernel 3: decode-size M (<= 4 rows) on CUDA cores, tile_n
 * columns per warp; splits >= 2: split-K with the fix-up inside the kernel;
 * ctas: grid size. */
typedef struct fqg_gemm_plan_info {
    int kernel, tile_m, tile_n, splits, ctas;
} fqg_gemm_plan_info;
int fqg_gemm_plan(int64_t m, int64_t n, int64_t kp, int a_fmt, int b_fmt, int y_dtype,
                  fqg_gemm_plan_info* out);

/* fq::quantize_layer (pipeline.cpp:76-152) for modes O1/O2/O3 with its scans on
 * the device: calibration channel maxima (collect_channel_maxes,
 * calibration.cpp:9-28), weight row maxima, and the KL bit-width selection
 * (select_bit_width, quantize.cpp:145-158: P / INT4 / INT8 round-trip
 * histograms of the flattened calibration activations and of the flattened
 * weight). Smoothing scales, boxplot truncation and the plans are host
 * arithmetic on K values. The recipe (bits, s, plans, T_x, T_w, act_scale, s_w,
 * KL ratios) equals the reference's bit for bit; the layer is then created with
 * desc.weight = W (the device weight tail computes the same weight_q).
 * weight: host f64 [k][n]; calib: host f64 [samples][rows][k]. */
typedef struct fqg_quant_options {
    int mode;            /* 1 = O1 (8 bits pinned), 2 = O2 (KL choice), 3 = O3 (O2 + GPTQ) */
    double alpha, beta, gamma;
    int64_t block, bins;
    int smooth, clip;
    double damping;      /* O3: Hessian damping (hessian_from_calibration) */
} fqg_quant_options;
void fqg_quant_options_default(fqg_quant_options* o);  /* pipeline.hpp:24-34 */
typedef struct fqg_recipe_s* fqg_recipe_t;
int fqg_calibrate(const double* weight, int64_t k, int64_t n, const double* calib, int64_t samples,
                  int64_t rows, const fqg_quant_options* options, int device, fqg_recipe_t* out);
/* The recipe as a layer description (arrays owned by the recipe). O1/O2:
 * weight_q is NULL, set desc.weight = W before fqg_layer_create. O3: weight_q
 * is the GPTQ result (gptq.cpp:106-161, computed on the device). */
int fqg_recipe_get(fqg_recipe_t recipe, fqg_layer_desc* desc, double* kl_ratio_act,
                   double* kl_ratio_w);
int fqg_recipe_free(fqg_recipe_t recipe);

/* The reference's on-disk contract (recipe JSON + FQTA archive) -> device
 * layers: replaces the CLI's load_recipes (flattenquant_cli.cpp:241-252, over
 * schemas.cpp:268-298 parse_recipe_json and archive.cpp:144-192
 * decode_archive). One layer per recipe entry, weights from
 * "<layer>.qweight" (int32 [K'][N]); 4-bit layers keep int4 weights packed in
 * HBM and take activations as `a_format` (FQG_I8 or FQG_I4). device < 0 parses
 * only (no layers; qmodel_path may be NULL). Errors carry the reference's texts
 * ("missing tensor: ...", "plan: inconsistent extension counts", ...). */
typedef struct fqg_model_s* fqg_model_t;
int fqg_model_load(const char* recipe_path, const char* qmodel_path, int device, int a_format,
                   fqg_model_t* out);
int fqg_model_destroy(fqg_model_t model);
int fqg_model_num_layers(fqg_model_t model, int64_t* n);
int fqg_model_layer_name(fqg_model_t model, int64_t index, char* buf, int64_t cap);
/* The parsed recipe of layer `index` (arrays owned by the model). */
int fqg_model_layer_recipe(fqg_model_t model, int64_t index, fqg_layer_desc* desc,
                           double* kl_ratio_act, double* kl_ratio_w);
/* The device layer of a recipe entry (owned by the model). */
int fqg_model_layer(fqg_model_t model, const char* name, fqg_layer_t* layer);
/* cmd_infer (flattenquant_cli.cpp:254-281): every f64 "<layer>/<name>" tensor of
 * the input FQTA archive through its layer; outputs (same names, f64 [rows][N],
 * equal to the reference bit for bit) written as an FQTA archive. */
int fqg_model_infer(fqg_model_t model, const char* input_path, const char* out_path,
                    int64_t* saturated_total, int64_t* ran);

/* 64-bit content hash (host, parallel over fixed 1 MiB blocks; the value does
 * not depend on the thread count). The C++ shim keys its layer cache on the
 * hash of every recipe field and the weights, so an edited recipe or a reused
 * address never returns a stale device layer. */
uint64_t fqg_hash64(const void* data, size_t bytes, uint64_t seed);

/* Host-side plan arithmetic (pure integer/FP64 work, no device):
 * fq::build_flatten_plan (flatten.cpp:17-45). e/off: [k]. */
int fqg_build_flatten_plan(const double* maxes, int64_t k, double t, int64_t block, int64_t* e,
                           int64_t* off, int64_t* c_extend, int64_t* padded_width);
/* fq::split_against_threshold (flatten.cpp:8-15). */
void fqg_split_against_threshold(double abs_value, double t, int64_t* count, double* rem);

/* The composite gather maps the layer compiles from plan_x / plan_w (host
 * only): for every final column k' of the flattened operands,
 *   amap[k'] = j << 12 | p_x : activation column k' is piece p_x of channel j
 *             (divide_columns -> flatten_tensor -> repeat_columns),
 *   wmap[k'] = j << 12 | p_w : weight row k' is piece p_w of smoothed row j
 *             (scale_rows -> repeat_channels -> flatten_rows),
 *   wcap[k'] = the plan_w capacity E_w + 1 of that row; -1 marks padding.
 * Arrays sized by `capacity` >= K' (returned in *kp). */
int fqg_gather_maps(const int64_t* ext_x, int64_t k, int64_t block_x, const int64_t* ext_w,
                    int64_t block_w, int32_t* amap, int32_t* wmap, int32_t* wcap, int64_t* kp,
                    int64_t capacity);

/* Offline recipe builder for modes O1/O2 with the bit width pinned by the
 * caller (KL bit selection, select_bit_width, is out of scope): the same
 * stage order as fq::quantize_layer (pipeline.cpp:76-152). Channel maxima of
 * the calibration set are given (collect_channel_maxes, calibration.cpp:9-28,
 * see fqg_collect_channel_maxes); the weight W is host f64 [k][n]. Writes the
 * recipe arrays: s[k], *t_x, e_x[k], *t_w, e_w[c1] (caller sizes e_w with
 * fqg_recipe_plan_sizes), *act_scale. The weight tail then runs in
 * fqg_layer_create with desc.weight = W. */
int fqg_recipe_plan(const double* weight, int64_t k, int64_t n, const double* act_maxes, int bits,
                    double alpha, double beta, int64_t block, int smooth, int clip, double* s,
                    double* t_x, int64_t* e_x, int64_t* c1, double* t_w, int64_t* e_w,
                    int64_t e_w_capacity, int64_t* kp, double* act_scale);
void fqg_collect_channel_maxes(const double* calib, int64_t rows, int64_t k, double* maxes_inout);

/* Deterministic synthetic layer generator with planted outlier channels, the
 * reference's input substrate (fq::make_synthetic_layer, synthetic.cpp:54-92,
 * mt19937_64 + Box-Muller). weight [k][n], calib [samples][rows][k],
 * test_input [test_rows][k] (test_rows may differ from rows). */
typedef struct fqg_synth_opts {
    int64_t rows, samples, in_channels, out_channels;
    double outlier_fraction, outlier_min, outlier_max, channel_spread;
    double act_tail_prob_max, act_tail_scale, weight_row_spread;
    uint64_t seed;
} fqg_synth_opts;
void fqg_synth_default(fqg_synth_opts* o);
int fqg_synthetic_layer(const fqg_synth_opts* o, int64_t index, double* weight, double* calib,
                        double* test_input, int64_t test_rows);

#ifdef __cplusplus
}
#endif
#endif /* FQG_H */
