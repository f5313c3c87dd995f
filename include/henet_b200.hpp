// SPDX-License-Identifier: Apache-2.0
//
// henet_b200.hpp -- C++ drop-in for the reference's hot path, over the C ABI.
//
// Include this AFTER the reference's own headers ("henet/henet.hpp"); it only
// uses their public types.  A reference user switches the evaluator by calling
// henet::gpu::execute instead of henet::execute -- same signature, same
// argument meaning, same exceptions (henet::ValidationError), bit-identical
// output ciphertexts (tests/test_gpu_dropin.py runs oracle/ref/dropin_test.cpp,
// which checks exactly that against the unmodified reference).
//
//   henet::execute        henet/graph.hpp:1121-1126   -> henet::gpu::execute
//   henet::relinearize    henet/ckks.hpp:442-499      -> henet::gpu::relinearize
//   henet::rescale        henet/ckks.hpp:504-519      -> henet::gpu::rescale
//   henet::mul_ct_pt_scalar henet/ckks.hpp:387-392    -> henet::gpu::mul_ct_pt_scalar
//   henet::encrypt_tensor henet/graph.hpp:68-91       -> henet::gpu::encrypt_tensor
//   henet::decrypt_tensor henet/graph.hpp:93-103      -> henet::gpu::decrypt_tensor
//   henet::LocalProvider  henet/graph.hpp:743-752     -> henet::gpu::LocalProvider (its
//       NonlinearityEngine on the GPU; gpu::execute hands it device tensors directly)
//
// Device state (context tables, relin key, model weights) is cached per
// CkksContext / RelinKey / PlainModel object, so repeated calls -- the
// InferenceServer pattern (henet/protocol.hpp:528) -- upload only ciphertexts.
#pragma once

#include <array>
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <map>
#include <thread>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "henet_b200.h"

namespace henet {
namespace gpu {

inline void check(int rc) {
  if (rc == HG_OK) return;
  const std::string msg = hg_last_error();
  if (rc == HG_ERR_VALIDATION) throw ValidationError(msg);
  throw std::runtime_error("henet::gpu: " + msg);
}

// Device mirror of one CkksContext (+ its relin keys and models), created lazily.
// Device caches are keyed by content, never by address (a freed object's address can be
// reused by a different model or key).  The content hash reads the words in place, four
// independent xxHash64-style lanes of 8-byte words (~10+ GB/s), so keying a 5.5 MB relin
// key or 64 MB of c5b weights costs well under the upload it saves.
inline u64 hash_bytes(const void* p, std::size_t n, u64 h = 0x9E3779B97F4A7C15ull) {
  constexpr u64 P1 = 0x9E3779B185EBCA87ull, P2 = 0xC2B2AE3D27D4EB4Full;
  auto rotl = [](u64 x, int r) { return (x << r) | (x >> (64 - r)); };
  auto round = [&](u64 acc, u64 w) { return rotl(acc + w * P2, 31) * P1; };
  const auto* b = static_cast<const unsigned char*>(p);
  u64 v[4] = {h + P1 + P2, h + P2, h, h - P1};
  std::size_t i = 0;
  for (; i + 32 <= n; i += 32) {
    u64 w[4];
    std::memcpy(w, b + i, 32);
    for (int k = 0; k < 4; ++k) v[k] = round(v[k], w[k]);
  }
  u64 acc = rotl(v[0], 1) + rotl(v[1], 7) + rotl(v[2], 12) + rotl(v[3], 18) + n;
  for (; i < n; ++i) acc = (acc ^ b[i]) * 1099511628211ull;
  acc ^= acc >> 33;
  acc *= P2;
  acc ^= acc >> 29;
  return acc;
}
inline u64 fnv(const void* p, std::size_t n, u64 h = 1469598103934665603ull) { return hash_bytes(p, n, h); }

class Device {
 public:
  explicit Device(const CkksContext& ctx, int device = 0) {
    std::vector<u64> chain;
    for (std::size_t i = 0; i < ctx.chain_length(); ++i) chain.push_back(ctx.modulus(i).value);
    check(hg_ctx_create(ctx.degree(), chain.data(), static_cast<uint32_t>(chain.size()),
                        ctx.has_special() ? ctx.special().value : 0, ctx.params().default_scale, device, &ctx_));
    n_ = ctx.degree();
  }
  ~Device() {
    for (auto& kv : keys_) hg_relin_key_destroy(kv.second);
    for (auto& kv : secrets_) hg_secret_key_destroy(kv.second);
    for (auto& kv : engines_) hg_refresh_engine_destroy(kv.second);
    for (auto& kv : models_) hg_model_destroy(kv.second);
    hg_ctx_destroy(ctx_);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  hg_ctx* ctx() const { return ctx_; }
  u32 degree() const { return n_; }

  // Relinearisation keys are keyed by identity (the words' addresses and sizes) plus a
  // sampled checksum (up to 64 words of every RingElement): a uniform-random key never
  // collides on the sample, and a key rebuilt at the same address differs in it.  Hashing
  // all 5.5 MB of a BASELINE key on every execute cost ~0.5 ms of the call.
  const hg_relin_key* relin(const RelinKey& rk) {
    u64 key = 0x52454c494eull;
    for (const auto& part : rk.parts)
      for (const auto& p : part) {
        const auto& w = p.words();
        const void* addr = w.data();
        const std::size_t n = w.size();
        key = hash_bytes(&addr, sizeof(addr), key);
        key = hash_bytes(&n, sizeof(n), key);
        const std::size_t stride = n > 64 ? n / 64 : 1;
        for (std::size_t i = 0; i < n; i += stride) key = (key ^ w[i]) * 0x9E3779B185EBCA87ull;
      }
    std::lock_guard<std::mutex> g(mu_);
    auto it = keys_.find(key);
    if (it != keys_.end()) return it->second;
    std::vector<u64> w;
    for (const auto& part : rk.parts)
      for (const auto& p : part) w.insert(w.end(), p.words().begin(), p.words().end());
    hg_relin_key* k = nullptr;
    check(hg_relin_key_upload(ctx_, w.data(), w.size(), &k));
    keys_[key] = k;
    return k;
  }

  const hg_secret_key* secret(const SecretKey& sk) {
    const auto& w = sk.s.words();
    const u64 key = fnv(w.data(), w.size() * sizeof(u64));
    std::lock_guard<std::mutex> g(mu_);
    auto it = secrets_.find(key);
    if (it != secrets_.end()) return it->second;
    hg_secret_key* k = nullptr;
    check(hg_secret_key_upload(ctx_, w.data(), w.size(), &k));
    secrets_[key] = k;
    return k;
  }

  // one device NonlinearityEngine per (secret key, refresh seed)
  hg_refresh_engine* engine(const SecretKey& sk, u64 seed) {
    const hg_secret_key* k = secret(sk);
    const u64 key = fnv(&seed, sizeof(seed), fnv(&k, sizeof(k)));
    std::lock_guard<std::mutex> g(mu_);
    auto it = engines_.find(key);
    if (it != engines_.end()) return it->second;
    hg_refresh_engine* e = nullptr;
    check(hg_refresh_engine_create(ctx_, k, seed, &e));
    engines_[key] = e;
    return e;
  }

  static u64 fingerprint(const PlainModel& m) {
    u64 h = fnv(&m.packing, sizeof(m.packing));
    for (const auto& [name, t] : m.weights) {
      h = fnv(name.data(), name.size(), h);
      h = fnv(t.shape.dims.data(), t.shape.dims.size() * sizeof(u32), h);
      h = fnv(t.data.data(), t.data.size() * sizeof(float), h);
    }
    for (const auto& n : m.nodes) {
      h = fnv(n.id.data(), n.id.size(), h);
      h = fnv(&n.op, sizeof(n.op), h);
      for (const auto& i : n.inputs) h = fnv(i.data(), i.size(), h);
      h = fnv(n.attrs.shape.data(), n.attrs.shape.size() * sizeof(u32), h);
      const u32 a[8] = {n.attrs.stride, n.attrs.window, n.attrs.filters, n.attrs.pool_stride,
                        n.attrs.pad[0], n.attrs.pad[1], n.attrs.pad[2], n.attrs.pad[3]};
      h = fnv(a, sizeof(a), h);
      h = fnv(n.weight_ref.data(), n.weight_ref.size(), h);
      h = fnv(n.bias_ref.data(), n.bias_ref.size(), h);
    }
    return h;
  }

  // PlainModel -> hg_model (weights + nodes); load_model's checks rerun device-side.  One
  // device model per (content, keep_encodings): the flag is fixed when the model is created,
  // so concurrent executes with and without a shared WeightEncoder never toggle it.
  const hg_model* model(const PlainModel& m, bool keep_encodings) {
    const u64 key = fingerprint(m) ^ (keep_encodings ? 0x4b454550ull : 0);
    std::lock_guard<std::mutex> g(mu_);
    auto it = models_.find(key);
    if (it != models_.end()) return it->second;
    hg_model* hm = nullptr;
    check(hg_model_create(static_cast<int>(m.packing), &hm));
    for (const auto& [name, t] : m.weights) {
      check(hg_model_add_weight(hm, name.c_str(), t.shape.dims.data(), static_cast<uint32_t>(t.shape.dims.size()),
                                t.data.data()));
    }
    for (const auto& n : m.nodes) {
      std::vector<const char*> ins;
      for (const auto& s : n.inputs) ins.push_back(s.c_str());
      hg_node_desc d{};
      d.id = n.id.c_str();
      d.op = static_cast<int>(n.op);
      d.inputs = ins.data();
      d.n_inputs = static_cast<uint32_t>(ins.size());
      d.shape = n.attrs.shape.data();
      d.shape_len = static_cast<uint32_t>(n.attrs.shape.size());
      d.stride = n.attrs.stride;
      d.window = n.attrs.window;
      d.filters = n.attrs.filters;
      for (int i = 0; i < 4; ++i) d.pad[i] = n.attrs.pad[i];
      d.pool_stride = n.attrs.pool_stride;
      d.weight_ref = n.weight_ref.c_str();
      d.bias_ref = n.bias_ref.c_str();
      check(hg_model_add_node(hm, &d));
    }
    check(hg_model_finalize(hm));
    check(hg_model_keep_encodings(hm, keep_encodings ? 1 : 0));
    models_[key] = hm;
    return hm;
  }

 private:
  hg_ctx* ctx_ = nullptr;
  u32 n_ = 0;
  std::mutex mu_;
  std::map<u64, hg_relin_key*> keys_;
  std::map<u64, hg_model*> models_;
  std::map<u64, hg_secret_key*> secrets_;
  std::map<u64, hg_refresh_engine*> engines_;
};

inline Device& device_for(const CkksContext& ctx) {
  static std::mutex mu;
  static std::map<u64, std::unique_ptr<Device>> devs;
  u64 key = fnv(&ctx.params().poly_degree, sizeof(u32));
  key = fnv(&ctx.params().default_scale, sizeof(double), key);
  for (std::size_t i = 0; i < ctx.chain_length(); ++i) key = fnv(&ctx.modulus(i).value, sizeof(u64), key);
  if (ctx.has_special()) key = fnv(&ctx.special().value, sizeof(u64), key);
  std::lock_guard<std::mutex> g(mu);
  auto& d = devs[key];
  if (!d) d = std::make_unique<Device>(ctx);
  return *d;
}

namespace detail {

// RAII tensor handle
struct Tensor {
  hg_tensor* t = nullptr;
  ~Tensor() { hg_tensor_destroy(t); }
};

// Ciphertexts -> device tensor.  The library's packer threads read every RingElement's words
// in place (hg_tensor_upload_segments), so no contiguous host copy of the tensor is built.
inline void upload(Device& dev, const std::vector<Ciphertext>& cts, const std::vector<u32>& shape, Tensor& out) {
  require(!cts.empty(), "empty cipher tensor");
  const u32 polys = static_cast<u32>(cts[0].size());
  const u32 level = static_cast<u32>(cts[0].level());
  check(hg_tensor_create(dev.ctx(), cts.size(), polys, level, cts[0].scale, static_cast<int>(cts[0].packing), &out.t));
  std::vector<const uint64_t*> segs;
  segs.reserve(cts.size() * polys);
  for (const auto& ct : cts) {
    require(ct.size() == polys && ct.level() == level, "ciphertext shape mismatch inside tensor");
    for (const auto& p : ct.polys) segs.push_back(p.words().data());
  }
  check(hg_tensor_upload_segments(out.t, segs.data(), nullptr));
  if (!shape.empty()) check(hg_tensor_set_shape(out.t, shape.data(), static_cast<uint32_t>(shape.size())));
}

// Device tensor -> ciphertexts, written straight into each RingElement's words.
inline std::vector<Ciphertext> download(Device& dev, const hg_tensor* t) {
  uint64_t count = 0;
  uint32_t polys = 0, level = 0;
  double scale = 0;
  int packing = 0;
  check(hg_tensor_info(t, &count, &polys, &level, &scale, &packing));
  std::vector<Ciphertext> out(count);
  std::vector<uint64_t*> segs;
  segs.reserve(count * polys);
  for (uint64_t e = 0; e < count; ++e) {
    out[e].polys.reserve(polys);
    for (u32 p = 0; p < polys; ++p) {
      out[e].polys.emplace_back(dev.degree(), level, PolyDomain::Ntt);
      segs.push_back(out[e].polys.back().words().data());
    }
    out[e].scale = scale;
    out[e].packing = static_cast<PackingMode>(packing);
    out[e].slots = dev.degree() / 2;
  }
  check(hg_tensor_download_segments(t, segs.data(), nullptr));
  return out;
}

struct ProviderCtx {
  Device* dev;
  NonlinearityProvider* provider;
};

// hg_nonlin_fn trampoline onto the reference NonlinearityProvider interface.
inline int provider_trampoline(void* user, int kind, uint32_t window, uint32_t layer_seq, const hg_tensor* request,
                               hg_tensor* response) {
  auto* pc = static_cast<ProviderCtx*>(user);
  try {
    auto req = download(*pc->dev, request);
    auto fresh = pc->provider->apply(kind == HG_NONLIN_RELU ? NonlinKind::Relu : NonlinKind::MaxPool, window,
                                     layer_seq, req);
    std::vector<const uint64_t*> segs;
    for (const auto& ct : fresh)
      for (const auto& p : ct.polys) segs.push_back(p.words().data());
    return hg_tensor_upload_segments(response, segs.data(), nullptr);
  } catch (...) {
    return 1;
  }
}

}  // namespace detail

// LocalProvider (henet/graph.hpp:743-752) whose NonlinearityEngine (decrypt, decode, ReLU /
// window max, encode, encrypt with derive_seed(derive_seed(seed, layer), group)) runs on
// the GPU.  gpu::execute recognises it and refreshes on device; any other caller gets the
// usual host-Ciphertext NonlinearityProvider interface.  Output bit-identical to
// henet::LocalProvider(NonlinearityEngine(ctx, sk, seed)).
class LocalProvider : public NonlinearityProvider {
 public:
  LocalProvider(std::shared_ptr<const CkksContext> ctx, SecretKey sk, u64 seed)
      : ctx_(std::move(ctx)), sk_(std::move(sk)), seed_(seed) {}
  hg_refresh_engine* engine(Device& dev) const { return dev.engine(sk_, seed_); }
  const CkksContext& context() const { return *ctx_; }

  std::vector<Ciphertext> apply(NonlinKind kind, u32 window, u32 layer_seq,
                                const std::vector<Ciphertext>& cts) override {
    Device& dev = device_for(*ctx_);
    detail::Tensor in, out;
    detail::upload(dev, cts, {}, in);
    check(hg_tensor_create(dev.ctx(), cts.size() / (window ? window : 1), 2, 1, 1.0, 0, &out.t));
    check(hg_refresh_engine_apply(engine(dev), kind == NonlinKind::Relu ? HG_NONLIN_RELU : HG_NONLIN_MAXPOOL, window,
                                  layer_seq, in.t, out.t));
    return detail::download(dev, out.t);
  }

 private:
  std::shared_ptr<const CkksContext> ctx_;
  SecretKey sk_;
  u64 seed_;
};

// encrypt_tensor, henet/graph.hpp:68-91 (threads is ignored: the GPU does the parallelism).
inline CipherTensor encrypt_tensor(const CkksContext& ctx, const BatchInput& input, const SecretKey& sk, u64 seed,
                                   PackingMode packing, unsigned threads = 1) {
  (void)threads;
  require(!input.samples.empty(), "batch must be non-empty");
  Device& dev = device_for(ctx);
  const std::size_t batch = input.samples.size(), count = input.shape.elem_count();
  std::vector<double> flat(batch * count);
  for (std::size_t s = 0; s < batch; ++s) {
    require(input.samples[s].size() == count, "sample size does not match the tensor shape");
    std::memcpy(&flat[s * count], input.samples[s].data(), count * sizeof(double));
  }
  detail::Tensor out;
  check(hg_tensor_create(dev.ctx(), count, 2, 1, 1.0, 0, &out.t));
  check(hg_encrypt_tensor(dev.ctx(), dev.secret(sk), flat.data(), static_cast<uint32_t>(batch), count, seed,
                          static_cast<int>(packing), out.t, nullptr));
  CipherTensor t;
  t.shape = input.shape;
  t.elems = detail::download(dev, out.t);
  return t;
}

// decrypt_tensor, henet/graph.hpp:93-103.
inline std::vector<std::vector<double>> decrypt_tensor(const CkksContext& ctx, const CipherTensor& ct,
                                                       const SecretKey& sk, std::size_t batch) {
  Device& dev = device_for(ctx);
  detail::Tensor in;
  detail::upload(dev, ct.elems, {}, in);
  const std::size_t count = ct.elems.size();
  std::vector<double> flat(batch * count);
  check(hg_decrypt_tensor(dev.ctx(), dev.secret(sk), in.t, static_cast<uint32_t>(batch), flat.data(), nullptr));
  std::vector<std::vector<double>> samples(batch, std::vector<double>(ct.shape.elem_count()));
  for (std::size_t s = 0; s < batch; ++s)
    for (std::size_t e = 0; e < count; ++e) samples[s][e] = flat[s * count + e];
  return samples;
}

namespace detail {
// RescalePlan -> hg_plan (the reference's plan passes through unchanged)
inline std::unique_ptr<hg_plan, void (*)(hg_plan*)> device_plan(const RescalePlan& plan) {
  hg_plan* hp = nullptr;
  check(hg_plan_create(static_cast<int>(plan.mode), plan.planned_rescale_ops, &hp));
  std::unique_ptr<hg_plan, void (*)(hg_plan*)> guard(hp, hg_plan_destroy);
  for (const auto& [id, np] : plan.nodes) {
    check(hg_plan_set_node(hp, id.c_str(), static_cast<int>(np.decision), static_cast<uint32_t>(np.level_in),
                           static_cast<uint32_t>(np.level_out), np.scale_out));
  }
  return guard;
}

inline std::vector<std::pair<std::string, double>> last_layers() {
  std::vector<std::pair<std::string, double>> out;
  uint32_t nl = 0;
  check(hg_last_exec_layer_count(&nl));
  for (uint32_t i = 0; i < nl; ++i) {
    const char* id = nullptr;
    double ms = 0;
    check(hg_last_exec_layer(i, &id, &ms));
    out.emplace_back(id, ms);
  }
  return out;
}
}  // namespace detail

// execute, henet/graph.hpp:1121-1126 -- the whole graph on the B200.
inline CipherTensor execute(std::shared_ptr<const CkksContext> ctx, const PlainModel& model, const RescalePlan& plan,
                            const CipherTensor& input, const ExecutionConfig& cfg, ExecutionStats* stats = nullptr) {
  Device& dev = device_for(*ctx);
  // a shared WeightEncoder (ExecutionConfig::encoder, henet/graph.hpp:773) keeps encodings
  // across calls; without one the reference encodes per call -- mirrored on the device
  const hg_model* hm = dev.model(model, cfg.encoder != nullptr);
  auto plan_guard = detail::device_plan(plan);
  hg_plan* hp = plan_guard.get();
  require(input.elems.size() == input.shape.elem_count(), "input shape does not match the model");
  detail::Tensor in;
  detail::upload(dev, input.elems, input.shape.dims, in);
  const hg_relin_key* rk = cfg.relin ? dev.relin(*cfg.relin) : nullptr;
  detail::ProviderCtx pc{&dev, cfg.provider};
  hg_exec_stats st{};
  detail::Tensor out;
  hg_nonlin_fn fn = cfg.provider ? detail::provider_trampoline : nullptr;
  void* user = &pc;
  if (auto* lp = dynamic_cast<LocalProvider*>(cfg.provider)) {  // refresh on device
    fn = hg_refresh_engine_apply;
    user = lp->engine(dev);
  }
  check(hg_execute(dev.ctx(), hm, hp, in.t, rk, fn, user, &out.t, stats ? &st : nullptr, nullptr));
  CipherTensor result;
  uint32_t dims[8], nd = 8;
  check(hg_tensor_get_shape(out.t, dims, &nd));
  result.shape = TensorShape{std::vector<u32>(dims, dims + nd)};
  result.elems = detail::download(dev, out.t);
  if (stats) {
    stats->rescale_ops = st.rescale_ops;
    stats->relin_ops = st.relin_ops;
    stats->nonlin_elements = st.nonlin_elements;
    stats->wall_ms = st.wall_ms;
    // layer_ms: one (node id, ms) per node in execution order (henet/graph.hpp:860-866),
    // from CUDA events around each node
    stats->layer_ms = detail::last_layers();
  }
  return result;
}

// InferenceServer (henet/protocol.hpp:449-598) with the evaluator on the B200: the same
// sessions, frames, checks, error codes and byte accounting, but the ciphertexts never become
// host Ciphertext objects.  INFER_REQ payloads are validated and packed straight into a device
// tensor (hg_tensor_deserialize, the checks of deserialize_ciphertext), the graph runs through
// hg_execute, every NONLIN_REQ is serialized from the device tensor (hg_tensor_serialize) and
// its NONLIN_RESP deserialized back onto the device, and the RESULT frame is
// hg_tensor_serialize of the output.  Bytes on the wire are identical to the reference
// server's (oracle/ref/dropin_test.cpp checks a loopback session against it).
class InferenceServer {
 public:
  struct ModelEntry {
    std::shared_ptr<const CkksContext> ctx;
    PlainModel model;
    RescalePlan plan;
  };

  void add_model(const std::string& id, PlainModel model, std::shared_ptr<const CkksContext> ctx = nullptr) {
    if (!ctx) ctx = CkksContext::create(model.preset);
    auto plan = plan_lazy_rescaling(*ctx, model);
    models_.emplace(id, ModelEntry{std::move(ctx), std::move(model), std::move(plan)});
  }

  // kept for interface parity: the GPU does the parallelism
  void set_threads(unsigned threads) { threads_ = threads; }

  const ModelEntry& entry(const std::string& id) const { return models_.at(id); }

  SessionStats handle_session(Stream& stream) const {
    SessionStats stats;
    auto t0 = std::chrono::steady_clock::now();
    try {
      Frame hello = read_frame(stream, &stats);
      if (hello.type != FrameType::Hello) {
        fail(stream, stats, 4, "expected HELLO");
        return stats;
      }
      SessionConfig config;
      try {
        config = henet::detail::decode_hello(hello.payload);
      } catch (const ValidationError& e) {
        fail(stream, stats, 3, std::string("bad HELLO: ") + e.what());
        return stats;
      }
      if (config.version != kProtocolVersion) {
        fail(stream, stats, 1, "protocol version mismatch");
        return stats;
      }
      auto it = models_.find(config.model_id);
      if (it == models_.end()) {
        fail(stream, stats, 2, "unknown model: " + config.model_id);
        return stats;
      }
      const ModelEntry& entry = it->second;
      if (config.preset != entry.model.preset) {
        fail(stream, stats, 2, "model is registered under a different preset");
        return stats;
      }
      if (config.packing != entry.model.packing) {
        fail(stream, stats, 2, "model is registered under a different packing");
        return stats;
      }
      if (config.batch == 0 || config.batch > batch_capacity(*entry.ctx, config.packing)) {
        fail(stream, stats, 3, "batch size outside slot capacity");
        return stats;
      }
      stats.batch = config.batch;
      write_frame(stream, FrameType::HelloAck, henet::detail::encode_hello(config), &stats);

      Frame infer = read_frame(stream, &stats);
      if (infer.type != FrameType::InferReq) {
        fail(stream, stats, 4, infer.type == FrameType::Hello ? "HELLO replayed mid-session" : "expected INFER_REQ");
        return stats;
      }
      Device& dev = device_for(*entry.ctx);
      detail::Tensor input;
      {
        uint64_t consumed = 0;
        const int rc = hg_tensor_deserialize(dev.ctx(), infer.payload.data(), infer.payload.size(), &consumed,
                                             &input.t, nullptr);
        if (rc == HG_ERR_VALIDATION) {
          fail(stream, stats, 3, std::string("bad INFER_REQ: ") + hg_last_error());
          return stats;
        }
        check(rc);
      }
      const hg_model* hm = dev.model(entry.model, false);
      auto plan = detail::device_plan(entry.plan);
      Remote remote{&dev, &stream, &stats, nullptr};
      hg_exec_stats st{};
      detail::Tensor out;
      const int rc = hg_execute(dev.ctx(), hm, plan.get(), input.t, nullptr, remote_apply, &remote, &out.t, &st,
                                nullptr);
      if (remote.error) std::rethrow_exception(remote.error);
      check(rc);
      stats.layer_ms = detail::last_layers();
      std::vector<u8> result(hg_tensor_serialized_size(out.t));
      check(hg_tensor_serialize(out.t, result.data(), result.size(), nullptr));
      write_frame(stream, FrameType::Result, result, &stats);
    } catch (const TransportError&) {
      // peer went away
    } catch (const ValidationError& e) {
      try {
        fail(stream, stats, 3, e.what());
      } catch (...) {
      }
    }
    stats.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return stats;
  }

  // Accept loop: one thread per connection, sessions independent (henet/protocol.hpp:548-560).
  void serve(TcpListener& listener, const std::atomic<bool>& stop) const {
    std::vector<std::thread> sessions;
    while (!stop.load()) {
      std::unique_ptr<TcpStream> conn;
      try {
        conn = listener.accept();
      } catch (const TransportError&) {
        break;
      }
      sessions.emplace_back([this, c = std::move(conn)]() mutable { handle_session(*c); });
    }
    for (auto& t : sessions) t.join();
  }

 private:
  struct Remote {
    Device* dev;
    Stream* stream;
    SessionStats* stats;
    std::exception_ptr error;
  };

  // RemoteProvider::apply (henet/protocol.hpp:566-583) over device tensors: NONLIN_REQ =
  // kind u8 | layer u32 | window u32 | the request's ciphertext list; NONLIN_RESP = the fresh
  // ciphertext list, deserialized onto the device.
  static int remote_apply(void* user, int kind, uint32_t window, uint32_t layer_seq, const hg_tensor* request,
                          hg_tensor* response) {
    auto* r = static_cast<Remote*>(user);
    try {
      std::vector<u8> tensor(hg_tensor_serialized_size(request));
      check(hg_tensor_serialize(request, tensor.data(), tensor.size(), nullptr));
      uint32_t dims[16], nd = 16;
      check(hg_tensor_get_shape(request, dims, &nd));
      const std::size_t skip = 1 + 4 * static_cast<std::size_t>(nd);  // put_tensor's shape prefix
      std::vector<u8> payload;
      payload.reserve(9 + tensor.size() - skip);
      put_u8(payload, static_cast<u8>(kind));
      put_u32(payload, layer_seq);
      put_u32(payload, window);
      payload.insert(payload.end(), tensor.begin() + static_cast<std::ptrdiff_t>(skip), tensor.end());
      write_frame(*r->stream, FrameType::NonlinReq, payload, r->stats, /*interactive=*/true);
      Frame resp = read_frame(*r->stream, r->stats, /*interactive=*/true);
      if (resp.type != FrameType::NonlinResp)
        throw TransportError("expected NONLIN_RESP at layer " + std::to_string(layer_seq));
      require(resp.payload.size() >= 4, "serialized data truncated");
      const u32 count = static_cast<u32>(resp.payload[0]) | static_cast<u32>(resp.payload[1]) << 8 |
                        static_cast<u32>(resp.payload[2]) << 16 | static_cast<u32>(resp.payload[3]) << 24;
      std::vector<u8> msg;  // the list as a put_tensor message of shape [count]
      msg.reserve(5 + resp.payload.size());
      put_u8(msg, 1);
      put_u32(msg, count);
      msg.insert(msg.end(), resp.payload.begin(), resp.payload.end());
      detail::Tensor fresh;
      uint64_t consumed = 0;
      check(hg_tensor_deserialize(r->dev->ctx(), msg.data(), msg.size(), &consumed, &fresh.t, nullptr));
      uint64_t req_count = 0;
      uint32_t polys = 0, level = 0;
      double scale = 0;
      int packing = 0;
      check(hg_tensor_info(request, &req_count, &polys, &level, &scale, &packing));
      const uint64_t expected = kind == HG_NONLIN_RELU ? req_count : req_count / window;
      require(count == expected, "provider returned the wrong element count");
      ++r->stats->nonlin_round_trips;
      check(hg_tensor_assign(response, fresh.t));
      return 0;
    } catch (...) {
      r->error = std::current_exception();
      return 1;
    }
  }

  void fail(Stream& stream, SessionStats& stats, u16 code, const std::string& message) const {
    write_frame(stream, FrameType::Error, henet::detail::encode_error(code, message), &stats);
    stream.close();
  }

  std::map<std::string, ModelEntry> models_;
  unsigned threads_ = 1;
};

// ---- multi-GPU: one process per GPU, NCCL inside the library ----
using CommId = std::array<uint8_t, HG_COMM_ID_BYTES>;
inline CommId comm_unique_id() {
  CommId id{};
  check(hg_comm_unique_id(id.data()));
  return id;
}

class Communicator {
 public:
  Communicator(const CkksContext& ctx, const CommId& id, int nranks, int rank)
      : dev_(&device_for(ctx)), nranks_(nranks), rank_(rank) {
    check(hg_comm_create(dev_->ctx(), id.data(), nranks, rank, &c_));
  }
  ~Communicator() { hg_comm_destroy(c_); }
  Communicator(const Communicator&) = delete;
  Communicator& operator=(const Communicator&) = delete;
  hg_comm* get() const { return c_; }
  Device& device() const { return *dev_; }
  int nranks() const { return nranks_; }
  int rank() const { return rank_; }

 private:
  Device* dev_;
  hg_comm* c_ = nullptr;
  int nranks_, rank_;
};

// A single-Dot model (Input -> Dot [+bias] -> Output, BASELINE c5b) evaluated with its output
// neurons split over the ranks: rank r runs the reference's eval_dot on the column block
// hg_shard_range(M, r, n) of W (same plan decisions, so the same arithmetic per output), and
// hg_allgather_tensor assembles all M output ciphertexts on every rank.  Bit-identical to
// henet::execute on the whole layer.  Lazy plans only (naive rescale counts differ per
// shard in a way the plan does not record).
inline CipherTensor execute_output_sharded(std::shared_ptr<const CkksContext> ctx, const PlainModel& model,
                                           const RescalePlan& plan, const CipherTensor& input, Communicator& comm) {
  require(plan.mode == RescaleMode::Lazy, "output sharding needs a lazy plan");
  const Node* dot = nullptr;
  for (const auto& n : model.nodes)
    if (n.op == OpKind::Dot) {
      require(dot == nullptr, "output sharding expects a single Dot node");
      dot = &n;
    }
  require(dot != nullptr, "output sharding expects a Dot node");
  const PlainTensor& w = model.weights.at(dot->weight_ref);
  const u32 K = w.shape.dims[0], M = w.shape.dims[1];
  uint64_t b0 = 0, cnt = 0;
  check(hg_shard_range(M, comm.rank(), comm.nranks(), &b0, &cnt));
  PlainModel part = model;  // the rank's column block of W (and of the bias)
  PlainTensor& pw = part.weights.at(dot->weight_ref);
  pw.shape.dims = {K, static_cast<u32>(cnt)};
  pw.data.assign(static_cast<std::size_t>(K) * cnt, 0.0f);
  for (u32 k = 0; k < K; ++k)
    for (uint64_t j = 0; j < cnt; ++j) pw.data[k * cnt + j] = w.data[static_cast<std::size_t>(k) * M + b0 + j];
  if (!dot->bias_ref.empty()) {
    const PlainTensor& b = model.weights.at(dot->bias_ref);
    PlainTensor& pb = part.weights.at(dot->bias_ref);
    pb.shape.dims = {static_cast<u32>(cnt)};
    pb.data.assign(b.data.begin() + static_cast<std::ptrdiff_t>(b0), b.data.begin() + static_cast<std::ptrdiff_t>(b0 + cnt));
  }
  RescalePlan pplan = plan;  // one rescale per output of a RescaleAfter Dot
  if (plan.nodes.at(dot->id).decision == RescaleDecision::RescaleAfter)
    pplan.planned_rescale_ops = plan.planned_rescale_ops - (M - cnt);
  Device& dev = comm.device();
  const hg_model* hm = dev.model(part, false);
  auto hp = detail::device_plan(pplan);
  detail::Tensor in;
  detail::upload(dev, input.elems, input.shape.dims, in);
  detail::Tensor local, full;
  hg_exec_stats st{};
  check(hg_execute(dev.ctx(), hm, hp.get(), in.t, nullptr, nullptr, nullptr, &local.t, &st, nullptr));
  check(hg_allgather_tensor(comm.get(), local.t, M, &full.t, nullptr));
  CipherTensor out;
  out.shape = model.shapes.at(model.output_node().id);
  out.elems = detail::download(dev, full.t);
  return out;
}

// ---- op level ----
inline Ciphertext relinearize(const CkksContext& ctx, const Ciphertext& ct, const RelinKey& rk) {
  Device& dev = device_for(ctx);
  detail::Tensor in, out;
  detail::upload(dev, {ct}, {}, in);
  check(hg_tensor_create(dev.ctx(), 1, 2, 1, 1.0, 0, &out.t));
  check(hg_relinearize(dev.ctx(), in.t, dev.relin(rk), out.t, nullptr));
  return detail::download(dev, out.t)[0];
}

inline Ciphertext rescale(const CkksContext& ctx, const Ciphertext& ct, std::size_t target_level) {
  Device& dev = device_for(ctx);
  detail::Tensor in, out;
  detail::upload(dev, {ct}, {}, in);
  check(hg_tensor_create(dev.ctx(), 1, 2, 1, 1.0, 0, &out.t));
  check(hg_rescale(dev.ctx(), in.t, static_cast<uint32_t>(target_level), out.t, nullptr));
  return detail::download(dev, out.t)[0];
}

inline Ciphertext mul_ct_pt_scalar(const CkksContext& ctx, const Ciphertext& ct, const ScalarPlaintext& pt) {
  Device& dev = device_for(ctx);
  detail::Tensor in, out;
  detail::upload(dev, {ct}, {}, in);
  check(hg_tensor_create(dev.ctx(), 1, 2, 1, 1.0, 0, &out.t));
  require(pt.level() == ct.level(), "ciphertext/plaintext level mismatch");
  check(hg_mul_ct_pt_scalar(dev.ctx(), in.t, pt.residues.data(), 0, pt.scale, out.t, nullptr));
  return detail::download(dev, out.t)[0];
}

}  // namespace gpu
}  // namespace henet
