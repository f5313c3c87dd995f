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

#include <cstring>
#include <map>
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

  const hg_relin_key* relin(const RelinKey& rk) {
    u64 key = 0x52454c494eull;
    for (const auto& part : rk.parts)
      for (const auto& p : part) key = hash_bytes(p.words().data(), p.words().size() * sizeof(u64), key);
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

// execute, henet/graph.hpp:1121-1126 -- the whole graph on the B200.
inline CipherTensor execute(std::shared_ptr<const CkksContext> ctx, const PlainModel& model, const RescalePlan& plan,
                            const CipherTensor& input, const ExecutionConfig& cfg, ExecutionStats* stats = nullptr) {
  Device& dev = device_for(*ctx);
  // a shared WeightEncoder (ExecutionConfig::encoder, henet/graph.hpp:773) keeps encodings
  // across calls; without one the reference encodes per call -- mirrored on the device
  const hg_model* hm = dev.model(model, cfg.encoder != nullptr);
  hg_plan* hp = nullptr;
  check(hg_plan_create(static_cast<int>(plan.mode), plan.planned_rescale_ops, &hp));
  std::unique_ptr<hg_plan, void (*)(hg_plan*)> plan_guard(hp, hg_plan_destroy);
  for (const auto& [id, np] : plan.nodes) {
    check(hg_plan_set_node(hp, id.c_str(), static_cast<int>(np.decision), static_cast<uint32_t>(np.level_in),
                           static_cast<uint32_t>(np.level_out), np.scale_out));
  }
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
    uint32_t nl = 0;
    check(hg_last_exec_layer_count(&nl));
    for (uint32_t i = 0; i < nl; ++i) {
      const char* id = nullptr;
      double ms = 0;
      check(hg_last_exec_layer(i, &id, &ms));
      stats->layer_ms.emplace_back(id, ms);
    }
  }
  return result;
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
