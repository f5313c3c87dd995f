// SPDX-License-Identifier: Apache-2.0
//
// Host runtime objects behind the C ABI: the device context (CkksContext
// mirror), device ciphertext batches (CipherTensor mirror), the relin key,
// the plain model (PlainModel mirror) and the rescale plan.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstdint>
#include <map>
#include <mutex>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/henet_b200.h"
#include "hg_kernels.hpp"
#include "hg_wide.hpp"
#include "hg_tc.hpp"
#include "hg_client.hpp"

namespace hg {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
inline void require(bool cond, const std::string& what) {
  if (!cond) throw Error(HG_ERR_VALIDATION, what);
}
void cuda_check(cudaError_t e, const char* what);

// hg_upload.cpp: reference u64 words -> device u32 residues, validated and packed by host
// threads and DMA'd chunk by chunk (HG_UPLOAD_HOST_NARROW=0: copy u64, narrow on the GPU).
bool host_narrow_enabled();
// Optional share of the words (the tail, whole limb runs at a ciphertext boundary) sent as
// raw u64 through `stage` and narrowed + validated on the GPU while the host packs the rest.
struct DirectShare {
  uint64_t words;
  uint64_t* stage;  // device, words * 8 bytes
  int* bad;         // device flag
  const Basis* basis;
};
// fraction of ciphertexts hg_tensor_upload sends raw (HG_UPLOAD_DIRECT_FRAC, default 0.15)
double upload_direct_fraction();
extern std::atomic<uint64_t> g_last_upload_h2d;  // bytes of the last host-packed upload (hg_upload.cpp)
bool host_narrow_upload(int device, const uint64_t* words, uint32_t* dst, uint64_t n_words, uint32_t level,
                        uint32_t N, const uint64_t* chain, cudaStream_t s, const uint8_t* const* segs = nullptr,
                        uint64_t seg_words = 0, const DirectShare* direct = nullptr);

// Shared device state: the stream and device; kept alive by every buffer.
struct DeviceCore {
  int device = 0;
  cudaStream_t stream = nullptr;
  // Buffer cache: buffers >= 1 MB (HG_BUF_CACHE_MIN_MB) allocated on `stream` are kept on
  // release and handed to the next request of exactly that size (stream-ordered like
  // cudaFreeAsync / cudaMallocAsync on the same stream).  A layer-sized cudaMallocAsync can
  // otherwise stall the host: 30-130 ms at a workload's memory peak (the c4 block), 10-500 ms
  // now and then with two contexts executing concurrently.
  std::mutex cache_mu;
  std::multimap<size_t, void*> cache;
  size_t cached = 0;
  void* take(size_t bytes);
  bool put(void* p, size_t bytes);
  void flush();  // cudaFreeAsync every cached buffer on `stream`
  void enroll();  // registers the core with its device's cache accounting (after `device` is set)
  ~DeviceCore();
};

struct DeviceBuffer {
  std::shared_ptr<DeviceCore> core;
  void* ptr = nullptr;
  size_t bytes = 0;
  cudaStream_t stream = nullptr;  // allocation stream; the free is ordered on it
  DeviceBuffer(std::shared_ptr<DeviceCore> c, size_t b, cudaStream_t s);
  ~DeviceBuffer();
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
};
using BufPtr = std::shared_ptr<DeviceBuffer>;

struct Context {
  std::shared_ptr<DeviceCore> core;
  u32 n = 0, logn = 0;
  std::vector<u64> chain;
  u64 special = 0;
  bool has_special = false;
  double default_scale = 0;
  std::vector<u64> roots;                    // psi per basis index
  std::vector<long double> modulus_products;  // q_l, henet/params.hpp:236-242
  Basis basis{};
  bool wide = false;  // some basis prime >= 2^30: every residue is stored as u64 (hg_wide.cu)
  bool dense_tc = false;  // Dot on tcgen05 int8 tensor cores (hg_tc.cu) instead of IMAD
  BasisW basisw{};
  BufPtr tables;      // twiddles for all basis moduli
  BufPtr wide_tables; // u64 twiddles (wide mode)
  BufPtr fft_tables;  // dft roots (N/2) + twist (N), double2
  std::vector<double> host_roots, host_twist;  // interleaved re/im

  size_t chain_len() const { return chain.size(); }
  size_t word_bytes() const { return wide ? 8 : 4; }
  u64 basis_mod(size_t i) const { return i < chain.size() ? chain[i] : special; }
  cudaStream_t pick(void* s) const { return s ? static_cast<cudaStream_t>(s) : core->stream; }
  BufPtr alloc(size_t bytes, cudaStream_t s) const { return std::make_shared<DeviceBuffer>(core, bytes, s); }
  // Device tables that depend only on a layer's geometry (convolution valid-tap lists),
  // built and uploaded once per distinct key.
  mutable std::mutex geo_mu;
  mutable std::map<std::vector<u32>, BufPtr> geo_cache;
};

// A batch of ciphertexts with one scale (Ciphertext::scale is identical
// across the elements of every tensor the executor produces).
struct CtBatch {
  BufPtr buf;
  u64 count = 0;
  u32 polys = 2, level = 0;
  double scale = 0;
  int packing = HG_PACKING_REAL;
  std::vector<u32> shape;
  u64 words(u32 n) const { return count * polys * level * static_cast<u64>(n); }
  u32* data() const { return buf ? static_cast<u32*>(buf->ptr) : nullptr; }
  u64* data64() const { return buf ? static_cast<u64*>(buf->ptr) : nullptr; }
};

struct RelinKeyDev {
  BufPtr key;  // [chain][2][chain+1][N]: u32 values, or (value, shoup) pairs (kKeyShoup)
  u32 chain_len = 0;
};

// A device buffer shared between executes, with the event its producing work recorded:
// a later execute on another stream waits on `ready` before reading it.
struct KeptBuf {
  BufPtr buf;
  std::shared_ptr<CUevent_st> ready;
};

struct WeightTensor {
  std::vector<u32> dims;
  std::vector<float> data;
  float max_abs = 0;
  // f32 device copy, uploaded lazily once per device (keyed by the context's DeviceCore)
  std::map<const DeviceCore*, KeptBuf> dev;
  // encodings kept across executes when the model caches weights (Model::keep_encodings):
  // (context, layout, level, scale bits, ...) -> device residues / packed planes
  std::map<std::vector<u64>, KeptBuf> enc;
  int depthwise = -1;  // conv weights (F, C, k, k) with F == C and zero off-diagonal taps; -1 unknown
};

struct NodeAttrs {
  std::vector<u32> shape;
  u32 stride = 1, window = 0, filters = 0, pool_stride = 0;
  std::array<u32, 4> pad{0, 0, 0, 0};
};

struct Node {
  std::string id;
  int op = HG_OP_INPUT;
  NodeAttrs attrs;
  std::vector<std::string> inputs;
  std::string weight_ref, bias_ref;
};

struct Model {
  int packing = HG_PACKING_REAL;
  std::vector<Node> nodes;
  std::map<std::string, WeightTensor> weights;
  std::map<std::string, std::vector<u32>> shapes;
  std::map<std::string, size_t> index;
  bool finalized = false;
  // Weight encodings persist across executes, like the reference's shared WeightEncoder
  // cache filled by precompile_weights (henet/graph.hpp:595-679); off = per-call encoding.
  bool keep_encodings = false;
  // Guards the lazily built per-weight state above (dev, enc, depthwise) and keep_encodings:
  // concurrent executes of one model (the reference allows them, henet/graph.hpp:601,616)
  // share it.
  std::shared_ptr<std::mutex> mu = std::make_shared<std::mutex>();
  const Node& node(const std::string& id) const { return nodes[index.at(id)]; }
};

struct NodePlan {
  int decision = HG_SKIP;
  u32 level_in = 0, level_out = 0;
  double scale_out = 0;
};

struct Plan {
  int mode = HG_RESCALE_LAZY;
  std::map<std::string, NodePlan> nodes;
  u64 planned_rescale_ops = 0;
};

}  // namespace hg

// C ABI handle types
struct hg_ctx {
  std::shared_ptr<hg::Context> c;
  std::array<double, 11> last_node_ms{};
};
struct hg_tensor {
  std::shared_ptr<hg::Context> ctx;
  hg::CtBatch b;
  // upload staging (u64 words + validation flag), kept across uploads: a fresh 617 MB
  // stream-ordered allocation per call cannot always reuse a block freed on another stream
  hg::BufPtr stage;
};
struct hg_relin_key {
  std::shared_ptr<hg::Context> ctx;
  hg::RelinKeyDev k;
};
struct hg_secret_key {
  std::shared_ptr<hg::Context> ctx;
  hg::BufPtr s;  // [full][N] u32, NTT domain (SecretKey::s, henet/ckks.hpp:21-23)
};
struct hg_model {
  hg::Model m;
};
struct hg_plan {
  hg::Plan p;
};
