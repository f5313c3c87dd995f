/* SPDX-License-Identifier: Apache-2.0
 *
 * henet_b200.h -- C ABI of the B200-native encrypted-inference hot path.
 *
 * This is the drop-in boundary for the `henet` reference library (nGraph-HE2
 * restatement, /root/reference/proj/include/henet).  The reference has no
 * plugin registry: its public surface is the header API itself.  Every entry
 * point below replaces one reference call on the hot path (cited as
 * `henet/<file>:<line>`, relative to proj/include/).  All arguments are plain
 * old data: pointers, sizes, doubles.  No torch or CUDA types appear in the
 * signatures; streams are passed as `void*` (a cudaStream_t, NULL = the
 * context's own stream).
 *
 * Conventions
 *  - Every function returns an `int` status (HG_OK == 0).  On failure a
 *    thread-local message is available from hg_last_error().  The C++ shim
 *    (henet_b200.hpp) maps HG_ERR_VALIDATION to henet::ValidationError, the
 *    reference's only error type on this path (henet/common.hpp:25-42).
 *  - Residues cross the boundary as little-endian u64 words in the
 *    reference's RingElement order: polynomial-major, then limb, then
 *    coefficient (henet/modmath.hpp:257-296, henet/serialize.hpp:61-63),
 *    NTT domain, one array per ciphertext, ciphertexts concatenated.
 *  - Device storage is u32 per residue (every supported prime is < 2^30).
 *  - There is no CPU fallback: if no sm_100 device is present, hg_ctx_create
 *    fails with HG_ERR_CUDA.
 */
#ifndef HENET_B200_H_
#define HENET_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_ABI_VERSION 1

enum hg_status {
  HG_OK = 0,
  HG_ERR_VALIDATION = 1,  /* henet::ValidationError */
  HG_ERR_CUDA = 2,        /* CUDA runtime / launch failure */
  HG_ERR_UNSUPPORTED = 3, /* parameters outside what the B200 kernels implement */
  HG_ERR_ALLOC = 4,       /* device or host allocation failure */
  HG_ERR_INTERNAL = 5
};

/* Packing mode, henet/encoding.hpp:12 */
enum hg_packing { HG_PACKING_REAL = 0, HG_PACKING_COMPLEX = 1 };

/* OpKind, henet/graph.hpp:109-121 (same numbering) */
enum hg_op {
  HG_OP_INPUT = 0,
  HG_OP_CONST_WEIGHT = 1,
  HG_OP_ADD = 2,
  HG_OP_MULTIPLY = 3,
  HG_OP_SQUARE = 4,
  HG_OP_DOT = 5,
  HG_OP_CONVOLUTION = 6,
  HG_OP_RESHAPE = 7,
  HG_OP_RELU = 8,
  HG_OP_MAXPOOL = 9,
  HG_OP_OUTPUT = 10
};

/* RescaleMode / RescaleDecision, henet/graph.hpp:447-448 */
enum hg_rescale_mode { HG_RESCALE_LAZY = 0, HG_RESCALE_NAIVE = 1 };
enum hg_rescale_decision { HG_SKIP = 0, HG_RESCALE_AFTER = 1 };

/* NonlinKind, henet/graph.hpp:687 */
enum hg_nonlin_kind { HG_NONLIN_RELU = 1, HG_NONLIN_MAXPOOL = 2 };

typedef struct hg_ctx hg_ctx;           /* CkksContext + device tables (henet/params.hpp:110-167) */
typedef struct hg_tensor hg_tensor;     /* device-resident CipherTensor (henet/graph.hpp:50-60) */
typedef struct hg_relin_key hg_relin_key; /* RelinKey (henet/ckks.hpp:25-27) on device */
typedef struct hg_model hg_model;       /* PlainModel (henet/graph.hpp:154-182) */
typedef struct hg_plan hg_plan;         /* RescalePlan (henet/graph.hpp:457-461) */

/* ------------------------------------------------------------------ */
/* Errors                                                              */
/* ------------------------------------------------------------------ */
const char* hg_last_error(void);
int hg_abi_version(void);

/* ------------------------------------------------------------------ */
/* Context: replaces CkksContext(EncryptionParameters)                 */
/* henet/params.hpp:112-129 (tables) with the parameter fields of      */
/* henet/params.hpp:21-27.  `special` == 0 means no special prime.     */
/* The scale<=q check of the checked constructor (henet/params.hpp:44) */
/* is NOT applied, matching field-assignment construction. */
/* ------------------------------------------------------------------ */
int hg_ctx_create(uint32_t poly_degree, const uint64_t* chain, uint32_t chain_len,
                  uint64_t special, double default_scale, int device, hg_ctx** out);
void hg_ctx_destroy(hg_ctx* ctx);
/* psi (primitive 2N-th root) used for basis index i; i == chain_len is the special prime.
 * find_ntt_root, henet/modmath.hpp:195-222 */
int hg_ctx_ntt_root(const hg_ctx* ctx, uint32_t basis_index, uint64_t* root);
/* cudaStream_t the context enqueues on when a call passes stream == NULL. */
void* hg_ctx_stream(hg_ctx* ctx);
int hg_ctx_synchronize(hg_ctx* ctx);
/* Kernel launches issued by this library in this process (all contexts; differences
 * around a region count the region's launches). */
uint64_t hg_ctx_launch_count(const hg_ctx* ctx);

/* ------------------------------------------------------------------ */
/* Ciphertext tensors: `count` ciphertexts of `polys` (2 or 3)          */
/* polynomials at `level`, one tensor-wide scale (Ciphertext::scale,    */
/* henet/ckks.hpp:34-42).  Device layout [elem][poly][limb][N] u32.     */
/* ------------------------------------------------------------------ */
int hg_tensor_create(hg_ctx* ctx, uint64_t count, uint32_t polys, uint32_t level, double scale,
                     int packing, hg_tensor** out);
void hg_tensor_destroy(hg_tensor* t);
int hg_tensor_info(const hg_tensor* t, uint64_t* count, uint32_t* polys, uint32_t* level,
                   double* scale, int* packing);
int hg_tensor_set_scale(hg_tensor* t, double scale);
/* Shape metadata (CipherTensor::shape); elem count must equal `count`. */
int hg_tensor_set_shape(hg_tensor* t, const uint32_t* dims, uint32_t ndims);
int hg_tensor_get_shape(const hg_tensor* t, uint32_t* dims, uint32_t* ndims /* in: cap, out: n */);
/* Host <-> device in the reference's u64 word order (see header).  Words are
 * checked < q_limb on upload, like deserialize_ciphertext (henet/serialize.hpp:66-77). */
int hg_tensor_upload(hg_tensor* t, const uint64_t* words, void* stream);
int hg_tensor_download(const hg_tensor* t, uint64_t* words, void* stream);
/* Wire format (put_tensor / get_tensor, henet/protocol.hpp:335-358, around
 * serialize_ciphertext, henet/serialize.hpp:95-124): u8 ndims, u32 dims, u32 count, then
 * per ciphertext u64 length + "NGH2" header + moduli + little-endian u64 residues.
 * Deserialisation validates every header and residue like deserialize_ciphertext (same
 * messages) and packs the words straight into a new device tensor; every element must share
 * level, size, packing and scale (HG_ERR_UNSUPPORTED otherwise).  *consumed = bytes read. */
int hg_tensor_deserialize(hg_ctx* ctx, const uint8_t* bytes, uint64_t len, uint64_t* consumed,
                          hg_tensor** out, void* stream);
uint64_t hg_tensor_serialized_size(const hg_tensor* t);
int hg_tensor_serialize(const hg_tensor* t, uint8_t* out, uint64_t cap, void* stream);
/* dst takes src's contents (count, polys, level, scale, packing, shape and residues; the
 * device buffer is shared, not copied).  Both tensors must belong to one context.  Lets an
 * hg_nonlin_fn hand back a tensor it obtained elsewhere (e.g. from hg_tensor_deserialize). */
int hg_tensor_assign(hg_tensor* dst, const hg_tensor* src);
/* Same word order, one pointer per polynomial (RingElement) instead of one contiguous array:
 * segs[e * polys + k] -> level * N words of polynomial k of element e.  The upload's packer
 * threads read each segment in place, so a caller holding std::vector<Ciphertext> (the
 * reference's CipherTensor) never builds a contiguous copy; checked like hg_tensor_upload. */
int hg_tensor_upload_segments(hg_tensor* t, const uint64_t* const* segs, void* stream);
int hg_tensor_download_segments(const hg_tensor* t, uint64_t* const* segs, void* stream);
/* Same, in the device's compact u32 word order (no widening). */
int hg_tensor_upload_u32(hg_tensor* t, const uint32_t* words, void* stream);
int hg_tensor_download_u32(const hg_tensor* t, uint32_t* words, void* stream);
/* Raw device pointer to the residues (for zero-copy interop, e.g. NCCL): u32 words, or
 * u64 words when the context has a prime >= 2^30 (hg_tensor_word_bytes says which);
 * hg_tensor_words = count * polys * level * N residues in [elem][poly][limb][N] order. */
void* hg_tensor_device_ptr(hg_tensor* t);
uint64_t hg_tensor_words(const hg_tensor* t);
uint32_t hg_tensor_word_bytes(const hg_tensor* t);

/* ------------------------------------------------------------------ */
/* Relinearization key, words in serialize_relin_key order             */
/* (henet/serialize.hpp:148-158): for j in chain: c0 then c1, each      */
/* (chain_len + 1) limbs x N u64 words, special limb last, NTT domain.  */
/* ------------------------------------------------------------------ */
int hg_relin_key_upload(hg_ctx* ctx, const uint64_t* words, uint64_t n_words, hg_relin_key** out);
void hg_relin_key_destroy(hg_relin_key* rk);

/* ------------------------------------------------------------------ */
/* Op-level evaluator (henet/ckks.hpp:281-524).  `out` must be a       */
/* distinct tensor created with the right count; its polys/level/scale  */
/* are overwritten to the result's.  Scales follow the reference's      */
/* double arithmetic exactly.                                           */
/* ------------------------------------------------------------------ */
/* add_ct_ct, henet/ckks.hpp:281-290 */
int hg_add_ct_ct(hg_ctx* ctx, const hg_tensor* a, const hg_tensor* b, hg_tensor* out, void* stream);
/* mul_ct_pt_scalar, henet/ckks.hpp:363-392: residues[e*level + i] is the scalar plaintext of
 * element e (or of every element when per_element == 0), each < q_i. */
int hg_mul_ct_pt_scalar(hg_ctx* ctx, const hg_tensor* ct, const uint64_t* residues,
                        int per_element, double pt_scale, hg_tensor* out, void* stream);
/* add_ct_pt_scalar, henet/ckks.hpp:315-330 (same residue convention). */
int hg_add_ct_pt_scalar(hg_ctx* ctx, const hg_tensor* ct, const uint64_t* residues,
                        int per_element, double pt_scale, hg_tensor* out, void* stream);
/* add_ct_pt_vector, henet/ckks.hpp:300-311: plaintext words level*N (u64, NTT domain),
 * one plaintext for every element (per_element == 0) or count plaintexts. */
int hg_add_ct_pt_vector(hg_ctx* ctx, const hg_tensor* ct, const uint64_t* pt_words,
                        int per_element, double pt_scale, hg_tensor* out, void* stream);
/* square, henet/ckks.hpp:424-437 (size-3 output). */
int hg_square(hg_ctx* ctx, const hg_tensor* ct, hg_tensor* out, void* stream);
/* mul_ct_ct, henet/ckks.hpp:407-422 (size-3 output). */
int hg_mul_ct_ct(hg_ctx* ctx, const hg_tensor* a, const hg_tensor* b, hg_tensor* out, void* stream);
/* relinearize, henet/ckks.hpp:442-499 (size-3 in, size-2 out). */
int hg_relinearize(hg_ctx* ctx, const hg_tensor* ct, const hg_relin_key* rk, hg_tensor* out,
                   void* stream);
/* Fused relinearize(square(ct)) [+ rescale_next] -- the Square node body of
 * eval_square, henet/graph.hpp:995-1008. */
int hg_square_relin(hg_ctx* ctx, const hg_tensor* ct, const hg_relin_key* rk, int rescale,
                    hg_tensor* out, void* stream);
/* rescale, henet/ckks.hpp:504-519 (drops limbs down to target_level). */
int hg_rescale(hg_ctx* ctx, const hg_tensor* ct, uint32_t target_level, hg_tensor* out,
               void* stream);

/* Negacyclic NTT of every limb of every polynomial of the tensor, in place
 * (ntt_forward / ntt_inverse, henet/modmath.hpp:382-398).  Only the domain
 * changes; hg tensors carry no domain flag, so the caller tracks it. */
int hg_ntt_forward(hg_ctx* ctx, hg_tensor* t, void* stream);
int hg_ntt_inverse(hg_ctx* ctx, hg_tensor* t, void* stream);

/* ------------------------------------------------------------------ */
/* Encoding                                                            */
/* ------------------------------------------------------------------ */
/* encode_scalar, henet/encoding.hpp:180-197, batched: out[v*level + i] = residue of
 * values[v] under chain prime i.  Computed on the GPU with exact x87 long-double rounding. */
int hg_encode_scalars(hg_ctx* ctx, const double* values, uint64_t count, uint32_t level,
                      double scale, uint64_t* out_residues);
/* encode_vector, henet/encoding.hpp:144-171 (+ fft.hpp:57-105): slots as interleaved
 * (re, im) doubles, n_slots <= N/2, per plaintext; `count` plaintexts back to back.
 * Output words: count x level x N u64 (NTT domain). */
int hg_encode_vector(hg_ctx* ctx, const double* slots_re_im, uint32_t n_slots, uint64_t count,
                     uint32_t level, double scale, uint64_t* out_words);

/* ------------------------------------------------------------------ */
/* Client side on the GPU                                              */
/* ------------------------------------------------------------------ */
typedef struct hg_secret_key hg_secret_key; /* SecretKey (henet/ckks.hpp:21-23) on device */
/* s in NTT form over the full basis, chain limbs then the special limb, in the word order
 * of serialize_secret_key (henet/serialize.hpp:129-136): (chain_len + 1) x N words. */
int hg_secret_key_upload(hg_ctx* ctx, const uint64_t* words, uint64_t n_words, hg_secret_key** out);
void hg_secret_key_destroy(hg_secret_key* sk);
/* encrypt_tensor (henet/graph.hpp:68-91): samples[s * count + e] is element e of sample s
 * (BatchInput::samples); ciphertext e = encrypt_batch(values of element e, sk,
 * derive_seed(seed, e)) at the top level and default scale (henet/ckks.hpp:229-254).
 * `out` is overwritten with the count ciphertexts. */
int hg_encrypt_tensor(hg_ctx* ctx, const hg_secret_key* sk, const double* samples, uint32_t batch,
                      uint64_t count, uint64_t seed, int packing, hg_tensor* out, void* stream);
/* decrypt (henet/ckks.hpp:256-268): plaintext residues count x level x N (u64, NTT domain). */
int hg_decrypt(hg_ctx* ctx, const hg_secret_key* sk, const hg_tensor* ct, uint64_t* pt_words,
               void* stream);
/* decrypt_tensor (henet/graph.hpp:93-103): out[s * count + e], s < batch. */
int hg_decrypt_tensor(hg_ctx* ctx, const hg_secret_key* sk, const hg_tensor* ct, uint32_t batch,
                      double* out, void* stream);

/* decode_slots (henet/encoding.hpp:223-264) of `count` plaintexts (level x N u64 words each,
 * NTT domain) at `scale`: N/2 slots per plaintext as interleaved (re, im), bit-exact. */
int hg_decode_vector(hg_ctx* ctx, const uint64_t* pt_words, uint64_t count, uint32_t level, double scale,
                     double* out_re_im);

/* ------------------------------------------------------------------ */
/* Graph level: PlainModel / RescalePlan / execute                     */
/* ------------------------------------------------------------------ */
typedef struct hg_node_desc {
  const char* id;
  int op;                    /* enum hg_op */
  const char* const* inputs; /* node ids */
  uint32_t n_inputs;
  const uint32_t* shape;     /* attrs.shape (Input / Reshape) */
  uint32_t shape_len;
  uint32_t stride;           /* NodeAttrs, henet/graph.hpp:136-143 */
  uint32_t window;
  uint32_t filters;
  uint32_t pad[4];           /* top, left, bottom, right */
  uint32_t pool_stride;
  const char* weight_ref;    /* may be NULL / "" */
  const char* bias_ref;      /* may be NULL / "" */
} hg_node_desc;

int hg_model_create(int packing, hg_model** out);
void hg_model_destroy(hg_model* m);
/* PlainTensor (henet/graph.hpp:45-48): row-major f32 */
int hg_model_add_weight(hg_model* m, const char* name, const uint32_t* dims, uint32_t ndims,
                        const float* data);
int hg_model_add_node(hg_model* m, const hg_node_desc* node);
/* Topological sort, shape inference and structural checks of load_model
 * (henet/graph.hpp:297-436). */
int hg_model_finalize(hg_model* m);
/* on != 0: weight encodings (residues at each consumer's level and scale, tensor-core byte
 * planes) are built on the first execute and reused by later ones -- the reference's shared
 * WeightEncoder cache after precompile_weights (henet/graph.hpp:595-679); results are
 * identical either way.  on == 0 (default): encoded per execute, like a per-call encoder. */
int hg_model_keep_encodings(hg_model* m, int on);
int hg_model_node_count(const hg_model* m, uint32_t* n);
int hg_model_shape(const hg_model* m, const char* id, uint32_t* dims, uint32_t* ndims);

/* plan_rescaling, henet/graph.hpp:504-584 */
int hg_plan_rescaling(const hg_ctx* ctx, const hg_model* m, int mode, hg_plan** out);
/* Same planner from the parameter fields alone (no device needed). */
int hg_plan_rescaling_params(const uint64_t* chain, uint32_t chain_len, double default_scale,
                             const hg_model* m, int mode, hg_plan** out);
/* An externally built plan (the reference's own RescalePlan, or a patched one). */
int hg_plan_create(int mode, uint64_t planned_rescale_ops, hg_plan** out);
int hg_plan_set_node(hg_plan* p, const char* id, int decision, uint32_t level_in,
                     uint32_t level_out, double scale_out);
int hg_plan_get_node(const hg_plan* p, const char* id, int* decision, uint32_t* level_in,
                     uint32_t* level_out, double* scale_out);
uint64_t hg_plan_planned_rescales(const hg_plan* p);
void hg_plan_destroy(hg_plan* p);

/* NonlinearityProvider::apply (henet/graph.hpp:689-697).  `request` holds groups
 * of `window` ciphertexts; the callback must fill `response` (already created with
 * one ciphertext per group) with fresh top-level encryptions and return 0. */
typedef int (*hg_nonlin_fn)(void* user, int kind, uint32_t window, uint32_t layer_seq,
                            const hg_tensor* request, hg_tensor* response);

/* ExecutionStats, henet/graph.hpp:776-782 (layer timings via CUDA events). */
typedef struct hg_exec_stats {
  uint64_t rescale_ops;
  uint64_t relin_ops;
  uint64_t nonlin_elements;
  double wall_ms;
  uint64_t kernel_launches;
} hg_exec_stats;

/* execute, henet/graph.hpp:1121-1126.  `input` must be at the top level with the
 * model's packing and input shape; *output is a fresh tensor owned by the caller. */
int hg_execute(hg_ctx* ctx, const hg_model* m, const hg_plan* plan, const hg_tensor* input,
               const hg_relin_key* rk, hg_nonlin_fn provider, void* provider_user,
               hg_tensor** output, hg_exec_stats* stats, void* stream);

/* ExecutionStats::layer_ms (henet/graph.hpp:776-782, filled at :860-866): one (node id, ms)
 * entry per node in execution order, from CUDA events around each node on the execute's
 * stream, for the most recent hg_execute on the calling thread that passed `stats` (or ran
 * with HG_NODE_TIMING set).  `*id` stays valid until the next hg_execute on this thread. */
int hg_last_exec_layer_count(uint32_t* n);
int hg_last_exec_layer(uint32_t index, const char** id, double* ms);

/* Host -> device bytes the most recent host-packed upload in this process put on the bus
 * (hg_tensor_upload / _upload_segments / hg_tensor_deserialize of a u32 context): the packed
 * chunks (3 bytes per residue of a prime < 2^24 when the host packs 24-bit words, else 4)
 * plus the raw u64 share.  0 before any such upload.  (bench.py's h2d_bytes_per_step.) */
int hg_last_upload_h2d_bytes(uint64_t* bytes);

/* NonlinearityEngine / LocalProvider (henet/graph.hpp:699-752) on the GPU: decrypt and
 * decode every request ciphertext, ReLU or the per-slot window max, encode_vector at the
 * top level and default scale, encrypt with derive_seed(derive_seed(seed, layer_seq), g).
 * Pass hg_refresh_engine_apply as hg_execute's provider with the engine as provider_user. */
typedef struct hg_refresh_engine hg_refresh_engine;
int hg_refresh_engine_create(hg_ctx* ctx, const hg_secret_key* sk, uint64_t seed, hg_refresh_engine** out);
void hg_refresh_engine_destroy(hg_refresh_engine* e);
int hg_refresh_engine_apply(void* engine, int kind, uint32_t window, uint32_t layer_seq,
                            const hg_tensor* request, hg_tensor* response);
/* hi > 0: ReLU refreshes clamp each slot to [0, hi] instead (v < 0 ? 0 : v > hi ? hi : v) --
 * the client-aided ReLU6 of BASELINE config 4; hi <= 0 restores ReLU. */
int hg_refresh_engine_set_relu_clip(hg_refresh_engine* e, double hi);

/* ------------------------------------------------------------------ */
/* Multi-GPU, one process per GPU.  The reference has no  */
/* multi-device executor; these are the pieces a C/C++ caller needs to  */
/* shard a layer's output neurons (BASELINE c5b) without torch: a       */
/* contiguous block partition, an NCCL communicator bound to a context, */
/* and a byte-exact all-gather of the ranks' output ciphertexts.  NCCL  */
/* is loaded at run time (libnccl.so.2); without it these return        */
/* HG_ERR_UNSUPPORTED.                                                  */
/* ------------------------------------------------------------------ */
#define HG_COMM_ID_BYTES 128
typedef struct hg_comm hg_comm;
/* Block partition of `total` items over `nranks` (sizes differ by <= 1, lower ranks larger):
 * rank owns [*begin, *begin + *count). */
int hg_shard_range(uint64_t total, int rank, int nranks, uint64_t* begin, uint64_t* count);
/* ncclGetUniqueId: call on one rank and pass the bytes to every rank (any side channel). */
int hg_comm_unique_id(uint8_t* id /* HG_COMM_ID_BYTES */);
/* ncclCommInitRank on the context's device (collective over the nranks processes). */
int hg_comm_create(hg_ctx* ctx, const uint8_t* id, int nranks, int rank, hg_comm** out);
void hg_comm_destroy(hg_comm* c);
/* `local` holds this rank's block hg_shard_range(total, rank, nranks) of a tensor of `total`
 * ciphertexts (same polys / level / scale on every rank); *out (new, shape [total]) receives
 * every rank's block in place, stream-ordered (no host synchronisation).  Residue words are
 * copied, never recomputed, so the gathered tensor is bit-identical to an unsharded run. */
int hg_allgather_tensor(hg_comm* c, const hg_tensor* local, uint64_t total, hg_tensor** out, void* stream);
/* ncclBroadcast of a tensor's residues from `root` (every rank's tensor has the same
 * count / polys / level), e.g. the c5b input ciphertexts staged on one rank. */
int hg_broadcast_tensor(hg_comm* c, hg_tensor* t, int root, void* stream);

/* ------------------------------------------------------------------ */
/* Measurement helpers (not part of the reference surface)             */
/* ------------------------------------------------------------------ */
/* Register-only integer-pipe microbenchmark (the INT32 roofline denominator):
 * kind 0 = IMAD (mad.lo.u32), 1 = IMAD.WIDE (mul.wide.u32, high word consumed: the cost of
 * one 32x32->64 MAC), 2 = IMAD.HI, 3 = Shoup lazy
 * modular product (IMAD.HI + 2 IMAD, the NTT butterfly's multiply), 4 = int8 tensor-core MACs
 * (tcgen05.mma.kind::i8, M=128 x N=256 x K=32, one CTA per SM); lane-ops/s (MAC/s for 4). */
int hg_bench_int_peak(int device, int kind, double* ops_per_s);
/* Per-kernel CUDA-event profiler: when enabled, every kernel launch is bracketed by
 * events on its stream; hg_prof_report writes {"kernel": {"ms": total, "launches": n}}
 * as JSON and clears the log. */
int hg_prof_enable(int on);
int hg_prof_report(char* buf, uint64_t cap);
/* Times the most recent execute's kernels (sum of per-node CUDA-event ms) by node op kind. */
int hg_last_exec_node_ms(hg_ctx* ctx, double* ms_by_op /* 11 entries, indexed by hg_op */);

#ifdef __cplusplus
}
#endif

#endif /* HENET_B200_H_ */
