// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// A C ABI over the UNMODIFIED reference library (the header-only `henet`
// under /root/reference/proj/include), compiled by oracle/Makefile into
// oracle/_ref/libhenet_ref.so.  The reference sources are included where they
// lie; nothing from them is copied into this repository.
//
// Used by: the parity tests (as the ground-truth oracle, and to generate the
// committed golden fixtures under tests/golden/), and by bench.py --impl
// reference (the reference's own CPU `execute()` timed on the host cores).
//
// Contexts are built by field assignment because the checked
// constructor rejects scale > prime (henet/params.hpp:44).
#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "henet/henet.hpp"

using namespace henet;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct RefCtx {
  std::shared_ptr<const CkksContext> ctx;
};

struct RefKeys {
  KeyPair kp;
};

RingElement poly_from(const u64* w, u32 n, std::size_t level) {
  RingElement p(n, level, PolyDomain::Ntt);
  std::memcpy(p.words().data(), w, sizeof(u64) * n * level);
  return p;
}

std::vector<Ciphertext> cts_from(const CkksContext& ctx, const u64* words, u64 count, u32 polys, u32 level,
                                 double scale, int packing) {
  std::vector<Ciphertext> out(count);
  const u64 per_poly = static_cast<u64>(ctx.degree()) * level;
  for (u64 e = 0; e < count; ++e) {
    Ciphertext& ct = out[e];
    for (u32 p = 0; p < polys; ++p) ct.polys.push_back(poly_from(words + (e * polys + p) * per_poly, ctx.degree(), level));
    ct.scale = scale;
    ct.packing = static_cast<PackingMode>(packing);
    ct.slots = ctx.slot_count();
  }
  return out;
}

void cts_to(const std::vector<Ciphertext>& cts, u64* words) {
  u64 off = 0;
  for (const auto& ct : cts)
    for (const auto& p : ct.polys) {
      std::memcpy(words + off, p.words().data(), sizeof(u64) * p.words().size());
      off += p.words().size();
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_ctx_create(uint32_t n, const uint64_t* chain, uint32_t L, uint64_t special, double scale) {
  RefCtx* r = nullptr;
  int rc = guard([&] {
    EncryptionParameters p;
    p.poly_degree = n;
    p.default_scale = scale;
    std::vector<PrimeModulus> moduli;
    for (uint32_t i = 0; i < L; ++i) moduli.emplace_back(chain[i]);
    std::optional<PrimeModulus> sp;
    if (special) sp = PrimeModulus(special);
    p.basis = RnsBasis(std::move(moduli), std::move(sp));
    r = new RefCtx{std::make_shared<const CkksContext>(p)};
  });
  return rc == 0 ? r : nullptr;
}

void ref_ctx_destroy(void* c) { delete static_cast<RefCtx*>(c); }

uint64_t ref_ntt_root(void* c, uint32_t basis_index) {
  auto& ctx = *static_cast<RefCtx*>(c)->ctx;
  return basis_index < ctx.chain_length() ? ctx.modulus(basis_index).ntt_root : ctx.special().ntt_root;
}

int ref_ntt(void* c, uint32_t basis_index, uint64_t* limb, int inverse) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    const NttTables& t = basis_index < ctx.chain_length() ? ctx.chain_tables()[basis_index] : ctx.special_table();
    std::span<u64> s(limb, ctx.degree());
    if (inverse) detail::ntt_inverse_limb(s, t);
    else detail::ntt_forward_limb(s, t);
  });
}

int ref_barrett(void* c, uint32_t basis_index, const uint64_t* lo, const uint64_t* hi, uint64_t count, int b64,
                uint64_t* out) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    const PrimeModulus& q = basis_index < ctx.chain_length() ? ctx.modulus(basis_index) : ctx.special();
    for (uint64_t i = 0; i < count; ++i) out[i] = b64 ? barrett_reduce_64(lo[i], q) : barrett_reduce_128(lo[i], hi[i], q);
  });
}

void* ref_keygen(void* c, uint64_t seed, int with_relin) {
  RefKeys* k = nullptr;
  int rc = guard([&] { k = new RefKeys{keygen(*static_cast<RefCtx*>(c)->ctx, seed, with_relin != 0)}; });
  return rc == 0 ? k : nullptr;
}

void ref_keys_destroy(void* k) { delete static_cast<RefKeys*>(k); }

int ref_sk_words(void* k, uint64_t* out) {
  return guard([&] {
    const auto& w = static_cast<RefKeys*>(k)->kp.secret.s.words();
    std::memcpy(out, w.data(), w.size() * 8);
  });
}

int ref_rk_words(void* k, uint64_t* out) {
  return guard([&] {
    const auto& rk = *static_cast<RefKeys*>(k)->kp.relin;
    u64 off = 0;
    for (const auto& part : rk.parts)
      for (const auto& p : part) {
        std::memcpy(out + off, p.words().data(), p.words().size() * 8);
        off += p.words().size();
      }
  });
}

// samples: batch x count (sample-major), like BatchInput::samples
int ref_encrypt_tensor(void* c, void* k, const double* samples, uint32_t batch, uint64_t count, uint64_t seed,
                       int packing, unsigned threads, uint64_t* out_words, double* out_scale) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    BatchInput in;
    in.shape = TensorShape{{static_cast<u32>(count)}};
    in.samples.resize(batch);
    for (uint32_t s = 0; s < batch; ++s) in.samples[s].assign(samples + s * count, samples + (s + 1) * count);
    auto t = encrypt_tensor(ctx, in, static_cast<RefKeys*>(k)->kp.secret, seed, static_cast<PackingMode>(packing),
                            threads ? threads : 1);
    cts_to(t.elems, out_words);
    *out_scale = t.elems[0].scale;
  });
}

int ref_decrypt_tensor(void* c, void* k, const uint64_t* words, uint64_t count, uint32_t polys, uint32_t level,
                       double scale, int packing, uint32_t batch, double* out) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    CipherTensor t;
    t.shape = TensorShape{{static_cast<u32>(count)}};
    t.elems = cts_from(ctx, words, count, polys, level, scale, packing);
    auto v = decrypt_tensor(ctx, t, static_cast<RefKeys*>(k)->kp.secret, batch);
    for (uint32_t s = 0; s < batch; ++s) std::memcpy(out + s * count, v[s].data(), count * 8);
  });
}

int ref_encode_scalar(void* c, double value, uint32_t level, double scale, uint64_t* out) {
  return guard([&] {
    auto pt = encode_scalar(*static_cast<RefCtx*>(c)->ctx, value, level, scale);
    std::memcpy(out, pt.residues.data(), level * 8);
  });
}

int ref_encode_vector(void* c, const double* re_im, uint32_t n_slots, uint32_t level, double scale, uint64_t* out) {
  return guard([&] {
    std::vector<std::complex<double>> slots(n_slots);
    for (uint32_t i = 0; i < n_slots; ++i) slots[i] = {re_im[2 * i], re_im[2 * i + 1]};
    auto pt = encode_vector(*static_cast<RefCtx*>(c)->ctx, slots, level, scale);
    std::memcpy(out, pt.poly.words().data(), pt.poly.words().size() * 8);
  });
}

int ref_decode(void* c, const uint64_t* words, uint32_t level, double scale, double* out_re_im) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    PackedPlaintext pt{poly_from(words, ctx.degree(), level), scale};
    auto s = decode_slots(ctx, pt);
    for (std::size_t i = 0; i < s.size(); ++i) {
      out_re_im[2 * i] = s[i].real();
      out_re_im[2 * i + 1] = s[i].imag();
    }
  });
}

// ---- ciphertext ops on `count` ciphertexts ----
int ref_mul_ct_pt_scalar(void* c, const uint64_t* words, uint64_t count, uint32_t polys, uint32_t level, double scale,
                         int packing, const uint64_t* residues, double pt_scale, uint64_t* out, double* out_scale) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto cts = cts_from(ctx, words, count, polys, level, scale, packing);
    ScalarPlaintext pt;
    pt.residues.assign(residues, residues + level);
    pt.scale = pt_scale;
    for (auto& ct : cts) ct = mul_ct_pt_scalar(ctx, ct, pt);
    cts_to(cts, out);
    *out_scale = cts[0].scale;
  });
}

int ref_add_ct_ct(void* c, const uint64_t* a, const uint64_t* b, uint64_t count, uint32_t polys, uint32_t level,
                  double scale, int packing, uint64_t* out) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto ca = cts_from(ctx, a, count, polys, level, scale, packing);
    auto cb = cts_from(ctx, b, count, polys, level, scale, packing);
    for (u64 i = 0; i < count; ++i) ca[i] = add_ct_ct(ctx, ca[i], cb[i]);
    cts_to(ca, out);
  });
}

int ref_add_ct_pt_vector(void* c, const uint64_t* words, uint64_t count, uint32_t polys, uint32_t level, double scale,
                         int packing, const uint64_t* pt_words, double pt_scale, uint64_t* out) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto cts = cts_from(ctx, words, count, polys, level, scale, packing);
    PackedPlaintext pt{poly_from(pt_words, ctx.degree(), level), pt_scale};
    for (auto& ct : cts) ct = add_ct_pt_vector(ctx, ct, pt);
    cts_to(cts, out);
  });
}

int ref_rescale(void* c, const uint64_t* words, uint64_t count, uint32_t polys, uint32_t level, double scale,
                int packing, uint32_t target, uint64_t* out, double* out_scale) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto cts = cts_from(ctx, words, count, polys, level, scale, packing);
    for (auto& ct : cts) ct = rescale(ctx, ct, target);
    cts_to(cts, out);
    *out_scale = cts[0].scale;
  });
}

int ref_square(void* c, const uint64_t* words, uint64_t count, uint32_t level, double scale, int packing,
               uint64_t* out, double* out_scale) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto cts = cts_from(ctx, words, count, 2, level, scale, packing);
    for (auto& ct : cts) ct = square(ctx, ct);
    cts_to(cts, out);
    *out_scale = cts[0].scale;
  });
}

int ref_mul_ct_ct(void* c, const uint64_t* a, const uint64_t* b, uint64_t count, uint32_t level, double scale_a,
                  double scale_b, int packing, uint64_t* out, double* out_scale) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto ca = cts_from(ctx, a, count, 2, level, scale_a, packing);
    auto cb = cts_from(ctx, b, count, 2, level, scale_b, packing);
    for (u64 i = 0; i < count; ++i) ca[i] = mul_ct_ct(ctx, ca[i], cb[i]);
    cts_to(ca, out);
    *out_scale = ca[0].scale;
  });
}

int ref_relinearize(void* c, void* k, const uint64_t* words, uint64_t count, uint32_t level, double scale, int packing,
                    uint64_t* out) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto cts = cts_from(ctx, words, count, 3, level, scale, packing);
    for (auto& ct : cts) ct = relinearize(ctx, ct, *static_cast<RefKeys*>(k)->kp.relin);
    cts_to(cts, out);
  });
}

// ---- graph level ----
namespace {
// Forces RescaleAfter on Dot/Convolution nodes the lazy planner marked Skip
// (BASELINE config 1: "one lazy rescale per output").
void patch_terminal_rescale(const CkksContext& ctx, const PlainModel& model, RescalePlan& plan) {
  const double s = ctx.params().default_scale;
  for (const auto& n : model.nodes) {
    auto& np = plan.nodes.at(n.id);
    if ((n.op == OpKind::Dot || n.op == OpKind::Convolution) && np.decision == RescaleDecision::Skip) {
      const auto& in = plan.nodes.at(n.inputs[0]);
      const double raised = in.scale_out * s;
      np.decision = RescaleDecision::RescaleAfter;
      np.level_out = np.level_in - 1;
      np.scale_out = raised / static_cast<double>(ctx.modulus(np.level_in - 1).value);
      plan.planned_rescale_ops += model.shapes.at(n.id).elem_count();
    } else if (!n.inputs.empty() && n.op != OpKind::Dot && n.op != OpKind::Convolution) {
      // propagate levels/scales of pass-through nodes
      if (n.op == OpKind::Reshape || n.op == OpKind::Output) {
        const auto& in = plan.nodes.at(n.inputs[0]);
        np.level_in = in.level_out;
        np.level_out = in.level_out;
        np.scale_out = in.scale_out;
      }
    }
  }
}

std::string plan_json(const PlainModel& model, const RescalePlan& plan) {
  nlohmann::json j;
  j["mode"] = plan.mode == RescaleMode::Lazy ? "lazy" : "naive";
  j["planned_rescale_ops"] = plan.planned_rescale_ops;
  nlohmann::json nodes = nlohmann::json::array();
  for (const auto& n : model.nodes) {
    const auto& np = plan.nodes.at(n.id);
    nodes.push_back({{"id", n.id},
                     {"decision", np.decision == RescaleDecision::Skip ? 0 : 1},
                     {"level_in", np.level_in},
                     {"level_out", np.level_out},
                     {"scale_out_bits", std::bit_cast<u64>(np.scale_out)}});
  }
  j["nodes"] = nodes;
  return j.dump();
}
}  // namespace

int ref_plan_json(void* c, const char* manifest, const uint8_t* blob, uint64_t blob_len, int mode, int patch,
                  char* out, uint64_t cap) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    auto model = load_model(manifest, std::span<const u8>(blob, blob_len));
    auto plan = plan_rescaling(ctx, model, mode ? RescaleMode::Naive : RescaleMode::Lazy);
    if (patch) patch_terminal_rescale(ctx, model, plan);
    std::string s = plan_json(model, plan);
    if (s.size() + 1 > cap) throw ValidationError("plan buffer too small");
    std::memcpy(out, s.c_str(), s.size() + 1);
  });
}

namespace {
// ReLU6 for config 4: the reference graph has no ReLU6 op; its Relu nodes
// run through a NonlinearityProvider.  With a clip bound set (ref_set_relu_clip), Relu
// clamps each decrypted slot component to [0, hi] instead of [0, inf); everything else
// (decode, encode at (L, default scale), per-group seeds) follows
// NonlinearityEngine::apply (henet/graph.hpp:707-741).  MaxPool is unchanged.
double g_relu_clip_hi = 0.0;  // 0: plain ReLU

std::vector<Ciphertext> clip_apply(const std::shared_ptr<const CkksContext>& sctx, const SecretKey& sk, u64 seed,
                                   NonlinKind kind, u32 window, u32 layer_seq, const std::vector<Ciphertext>& cts) {
  if (kind != NonlinKind::Relu || g_relu_clip_hi <= 0.0)
    return NonlinearityEngine(sctx, sk, seed).apply(kind, window, layer_seq, cts);
  require(window == 1, "ReLU is element-wise");
  const CkksContext& ctx = *sctx;
  const double hi = g_relu_clip_hi;
  auto clamp = [hi](double v) { return v < 0.0 ? 0.0 : (v > hi ? hi : v); };
  std::vector<Ciphertext> out(cts.size());
  // Groups are independent and seeded per group (derive_seed(derive_seed(seed, layer), g)),
  // so the harness spreads them over the host threads with the reference's parallel_for;
  // the result is identical to the serial loop.
  parallel_for(cts.size(), std::thread::hardware_concurrency(), [&](std::size_t g) {
    auto slots = decode_slots(ctx, decrypt(ctx, cts[g], sk));
    for (auto& z : slots) z = {clamp(z.real()), clamp(z.imag())};
    auto pt = encode_vector(ctx, slots, ctx.chain_length(), ctx.params().default_scale);
    out[g] = encrypt(ctx, pt, sk, derive_seed(derive_seed(seed, layer_seq), g), cts[g].packing);
  });
  return out;
}

class ClipProvider : public NonlinearityProvider {
 public:
  ClipProvider(std::shared_ptr<const CkksContext> ctx, SecretKey sk, u64 seed)
      : ctx_(std::move(ctx)), sk_(std::move(sk)), seed_(seed) {}
  std::vector<Ciphertext> apply(NonlinKind kind, u32 window, u32 layer_seq,
                                const std::vector<Ciphertext>& cts) override {
    return clip_apply(ctx_, sk_, seed_, kind, window, layer_seq, cts);
  }

 private:
  std::shared_ptr<const CkksContext> ctx_;
  SecretKey sk_;
  u64 seed_;
};
}  // namespace

void ref_set_relu_clip(double hi) { g_relu_clip_hi = hi; }

int ref_execute(void* c, void* k, const char* manifest, const uint8_t* blob, uint64_t blob_len, int mode, int patch,
                const uint64_t* in_words, uint64_t in_count, double in_scale, unsigned threads, uint64_t refresh_seed,
                uint64_t* out_words, uint64_t out_capacity_words, uint64_t* out_count, uint32_t* out_level,
                double* out_scale, double* exec_ms, uint64_t* rescales, uint64_t* relins) {
  return guard([&] {
    auto sctx = static_cast<RefCtx*>(c)->ctx;
    auto& ctx = *sctx;
    auto* keys = static_cast<RefKeys*>(k);
    auto model = load_model(manifest, std::span<const u8>(blob, blob_len));
    auto plan = plan_rescaling(ctx, model, mode ? RescaleMode::Naive : RescaleMode::Lazy);
    if (patch) patch_terminal_rescale(ctx, model, plan);
    CipherTensor input;
    input.shape = model.shapes.at(model.input_node().id);
    require(input.shape.elem_count() == in_count, "input count does not match the model");
    input.elems = cts_from(ctx, in_words, in_count, 2, static_cast<u32>(ctx.chain_length()), in_scale,
                           static_cast<int>(model.packing));
    ExecutionConfig cfg;
    cfg.threads = threads ? threads : std::thread::hardware_concurrency();
    if (keys && keys->kp.relin) cfg.relin = &*keys->kp.relin;
    std::unique_ptr<ClipProvider> prov;
    if (keys) {
      prov = std::make_unique<ClipProvider>(sctx, keys->kp.secret, refresh_seed);
      cfg.provider = prov.get();
    }
    ExecutionStats st;
    const auto t0 = std::chrono::steady_clock::now();
    auto out = execute(sctx, model, plan, input, cfg, &st);
    const auto t1 = std::chrono::steady_clock::now();
    if (exec_ms) *exec_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    const u64 words = out.elems.size() * out.elems[0].size() * out.level() * ctx.degree();
    require(words <= out_capacity_words, "output buffer too small");
    cts_to(out.elems, out_words);
    *out_count = out.elems.size();
    *out_level = static_cast<uint32_t>(out.level());
    *out_scale = out.scale();
    if (rescales) *rescales = st.rescale_ops;
    if (relins) *relins = st.relin_ops;
  });
}

// NonlinearityEngine::apply for the GPU path's provider callback in tests:
// decrypt -> relu (or ReLU6 when a clip bound is set)/maxpool -> re-encrypt at the top
// level, seeded like the reference.
int ref_nonlin_apply(void* c, void* k, int kind, uint32_t window, uint32_t layer_seq, uint64_t refresh_seed,
                     const uint64_t* words, uint64_t count, uint32_t level, double scale, int packing,
                     uint64_t* out_words) {
  return guard([&] {
    auto sctx = static_cast<RefCtx*>(c)->ctx;
    auto& ctx = *sctx;
    auto* keys = static_cast<RefKeys*>(k);
    auto cts = cts_from(ctx, words, count, 2, level, scale, packing);
    auto out = clip_apply(sctx, keys->kp.secret, refresh_seed, kind == 1 ? NonlinKind::Relu : NonlinKind::MaxPool,
                          window, layer_seq, cts);
    cts_to(out, out_words);
  });
}

// Wire format (test fixture side): detail::put_tensor / get_tensor, henet/protocol.hpp:335-358.
int ref_put_tensor(void* c, const uint64_t* words, uint64_t count, uint32_t polys, uint32_t level, double scale,
                   int packing, const uint32_t* dims, uint32_t ndims, uint8_t* out, uint64_t cap, uint64_t* out_len) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    CipherTensor t;
    for (uint32_t i = 0; i < ndims; ++i) t.shape.dims.push_back(dims[i]);
    t.elems = cts_from(ctx, words, count, polys, level, scale, packing);
    std::vector<u8> bytes;
    detail::put_tensor(bytes, ctx, t);
    *out_len = bytes.size();
    if (out != nullptr) {
      require(cap >= bytes.size(), "buffer too small");
      std::memcpy(out, bytes.data(), bytes.size());
    }
  });
}

int ref_get_tensor(void* c, const uint8_t* bytes, uint64_t len, uint64_t* out_words, uint64_t cap_words,
                   uint64_t* count, uint32_t* polys, uint32_t* level, double* scale) {
  return guard([&] {
    auto& ctx = *static_cast<RefCtx*>(c)->ctx;
    ByteReader in(bytes, len);
    CipherTensor t = detail::get_tensor(in, ctx);
    *count = t.elems.size();
    *polys = static_cast<uint32_t>(t.elems[0].size());
    *level = static_cast<uint32_t>(t.elems[0].level());
    *scale = t.elems[0].scale;
    u64 need = 0;
    for (const auto& ct : t.elems)
      for (const auto& p : ct.polys) need += p.words().size();
    require(need <= cap_words, "buffer too small");
    cts_to(t.elems, out_words);
  });
}

}  // extern "C"
