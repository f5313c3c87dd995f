// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY -- the drop-in check.  Compiled against the
// UNMODIFIED reference headers (/root/reference/proj/include) plus
// include/henet_b200.hpp, linked to the product libhenet_b200.so.  Runs the
// reference's own model generators through henet::execute (CPU) and
// henet::gpu::execute (B200) with identical arguments and requires
// bit-identical ciphertexts, scales and statistics; likewise the client side
// (encrypt_tensor, decrypt_tensor, LocalProvider).  Exit code 0 = pass.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <future>
#include <tuple>
#include <string>
#include <thread>

#include "henet/henet.hpp"
#include "henet_b200.hpp"

using namespace henet;

static std::shared_ptr<const CkksContext> baseline_ctx() {
  EncryptionParameters p;  // field assignment: scale 2^24 > 24-bit primes
  p.poly_degree = 8192;
  p.default_scale = std::ldexp(1.0, 24);
  std::vector<PrimeModulus> chain;
  for (u64 q : {1073692673ull, 16760833ull, 16580609ull, 16515073ull, 16465921ull, 16384001ull}) chain.emplace_back(q);
  p.basis = RnsBasis(std::move(chain), PrimeModulus(1073643521ull));
  return std::make_shared<const CkksContext>(p);
}

static bool same(const CipherTensor& a, const CipherTensor& b, const char* what) {
  bool ok = a.shape == b.shape && a.elems.size() == b.elems.size();
  for (std::size_t e = 0; ok && e < a.elems.size(); ++e) {
    ok = a.elems[e].scale == b.elems[e].scale && a.elems[e].packing == b.elems[e].packing &&
         a.elems[e].polys.size() == b.elems[e].polys.size();
    for (std::size_t k = 0; ok && k < a.elems[e].polys.size(); ++k) ok = a.elems[e].polys[k] == b.elems[e].polys[k];
  }
  std::printf("%-40s %s (%zu ciphertexts at level %zu)\n", what, ok ? "bit-identical" : "MISMATCH", a.elems.size(),
              a.elems.empty() ? 0 : a.level());
  return ok;
}

static bool run_model(std::shared_ptr<const CkksContext> ctx, const KeyPair& keys, const GeneratedModel& gm,
                      PackingMode packing, std::size_t batch, const char* name) {
  PlainModel model = load_model(gm.manifest, std::span<const u8>(gm.blob.data(), gm.blob.size()));
  RescalePlan plan = plan_lazy_rescaling(*ctx, model);
  BatchInput in = make_random_input(model.shapes.at(model.input_node().id), batch, 5);
  CipherTensor x = encrypt_tensor(*ctx, in, keys.secret, 77, packing, std::thread::hardware_concurrency());
  LocalProvider prov(NonlinearityEngine(ctx, keys.secret, 99));
  ExecutionConfig cfg;
  cfg.threads = std::thread::hardware_concurrency();
  cfg.relin = keys.relin ? &*keys.relin : nullptr;
  cfg.provider = &prov;
  ExecutionStats s_cpu, s_gpu;
  CipherTensor want = henet::execute(ctx, model, plan, x, cfg, &s_cpu);
  CipherTensor got = henet::gpu::execute(ctx, model, plan, x, cfg, &s_gpu);
  bool ok = same(want, got, name);
  ok = ok && s_cpu.rescale_ops == s_gpu.rescale_ops && s_cpu.relin_ops == s_gpu.relin_ops &&
       s_cpu.nonlin_elements == s_gpu.nonlin_elements;
  // layer_ms: one entry per node, same ids in the same order (henet/graph.hpp:860-866)
  bool layers_ok = s_cpu.layer_ms.size() == s_gpu.layer_ms.size();
  for (std::size_t i = 0; layers_ok && i < s_cpu.layer_ms.size(); ++i)
    layers_ok = s_cpu.layer_ms[i].first == s_gpu.layer_ms[i].first && s_gpu.layer_ms[i].second >= 0.0;
  std::printf("  layer_ms: %zu entries %s\n", s_gpu.layer_ms.size(), layers_ok ? "ids match" : "MISMATCH");
  ok = ok && layers_ok;
  std::printf("  stats cpu (rescale %llu relin %llu nonlin %llu, %.0f ms)  gpu (rescale %llu relin %llu nonlin %llu)\n",
              (unsigned long long)s_cpu.rescale_ops, (unsigned long long)s_cpu.relin_ops,
              (unsigned long long)s_cpu.nonlin_elements, s_cpu.wall_ms, (unsigned long long)s_gpu.rescale_ops,
              (unsigned long long)s_gpu.relin_ops, (unsigned long long)s_gpu.nonlin_elements);
  return ok;
}

// --bench K: the drop-in's end-to-end time per call -- henet::gpu::execute on the c2
// CryptoNets-shaped network (make_cryptonets, 4096 images, BASELINE context) with host
// CipherTensors in and out, i.e. upload + execute + download as a reference user sees it.
static int bench(int steps) {
  auto ctx = baseline_ctx();
  KeyPair keys = keygen(*ctx, 2024, true);
  auto gm = make_cryptonets(Preset::P13, 1);
  PlainModel model = load_model(gm.manifest, std::span<const u8>(gm.blob.data(), gm.blob.size()));
  RescalePlan plan = plan_lazy_rescaling(*ctx, model);
  BatchInput in = make_random_input(model.shapes.at(model.input_node().id), 4096, 5);
  CipherTensor x = henet::gpu::encrypt_tensor(*ctx, in, keys.secret, 77, PackingMode::Real);
  ExecutionConfig cfg;
  cfg.relin = &*keys.relin;
  std::vector<double> ms;
  for (int i = 0; i < steps + 3; ++i) {
    const auto t0 = std::chrono::steady_clock::now();
    CipherTensor y = henet::gpu::execute(ctx, model, plan, x, cfg);
    const auto t1 = std::chrono::steady_clock::now();
    if (i >= 3) ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    if (y.elems.size() != 10) return 1;
  }
  // the upload alone (hg_tensor_upload_segments from the RingElements), for the breakdown
  std::vector<double> up;
  henet::gpu::Device& dev = henet::gpu::device_for(*ctx);
  for (int i = 0; i < steps; ++i) {
    henet::gpu::detail::Tensor t;
    const auto t0 = std::chrono::steady_clock::now();
    henet::gpu::detail::upload(dev, x.elems, x.shape.dims, t);
    up.push_back(std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  // per-phase host times of the call, for the breakdown: the device-cache lookups (relin key,
  // model, plan) and the upload; the remainder of the call is hg_execute + the download
  std::vector<double> t_key, t_model, t_plan;
  for (int i = 0; i < steps; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    dev.relin(*keys.relin);
    auto t1 = std::chrono::steady_clock::now();
    dev.model(model, false);
    auto t2 = std::chrono::steady_clock::now();
    auto pg = henet::gpu::detail::device_plan(plan);
    auto t3 = std::chrono::steady_clock::now();
    t_key.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
    t_model.push_back(std::chrono::duration<double, std::milli>(t2 - t1).count());
    t_plan.push_back(std::chrono::duration<double, std::milli>(t3 - t2).count());
  }
  auto med = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::fprintf(stderr, "dropin breakdown [ms]: relin key lookup %.3f, model lookup %.3f, plan %.3f\n", med(t_key),
               med(t_model), med(t_plan));
  std::sort(ms.begin(), ms.end());
  std::sort(up.begin(), up.end());
  double sum = 0;
  for (double v : ms) sum += v;
  std::printf("{\"dropin_ms_median\": %.4f, \"dropin_ms_mean\": %.4f, \"dropin_ms_min\": %.4f, "
              "\"upload_ms_median\": %.4f, \"steps\": %d, \"images\": 4096, \"input_cts\": %zu}\n",
              ms[ms.size() / 2], sum / ms.size(), ms[0], up[up.size() / 2], steps, x.elems.size());
  return 0;
}

// One client session (the reference's client_infer) against a server over the in-process
// pipe (ServerRun, proj/tests/test_protocol.cpp:32-46); returns the client's result, or the
// rejection message, and the server's accounting.
template <class Server>
static std::pair<ClientResult, SessionStats> session(const Server& server, std::shared_ptr<const CkksContext> ctx,
                                                     const SessionConfig& config, const BatchInput& input,
                                                     const SecretKey& sk, u64 seed, std::string* error) {
  auto [a, b] = make_pipe();
  std::shared_ptr<Stream> server_end(std::move(b));
  auto fut = std::async(std::launch::async, [&server, server_end] {
    auto st = server.handle_session(*server_end);
    server_end->close();
    return st;
  });
  ClientResult r;
  try {
    r = client_infer(*a, ctx, config, input, sk, seed);
  } catch (const std::exception& e) {
    if (error) *error = e.what();
  }
  a->close();
  return {r, fut.get()};
}

static bool same_stats(const SessionStats& x, const SessionStats& y) {
  return x.bytes_sent == y.bytes_sent && x.bytes_received == y.bytes_received &&
         x.interactive_bytes == y.interactive_bytes && x.nonlin_round_trips == y.nonlin_round_trips &&
         x.batch == y.batch && x.layer_ms.size() == y.layer_ms.size();
}

// InferenceServer::handle_session (henet/protocol.hpp:465-545) with the GPU evaluator against
// the reference server: the loopback case of proj/tests/test_protocol.cpp:207-246 (P11,
// client-aided ReLU network, bit-exact decrypted outputs, one round trip per ReLU layer),
// the same at P13 under complex packing, and rejected sessions; wire bytes and accounting
// must be identical.
static bool protocol_checks() {
  bool ok = true;
  for (auto [pr, packing, batch] : {std::tuple{Preset::P11, PackingMode::Real, 4u},
                                    std::tuple{Preset::P13, PackingMode::Complex, 64u}}) {
    auto ctx = CkksContext::create(pr);
    KeyPair keys = keygen(*ctx, 11, false);
    auto gm = make_cryptonets_relu(pr, packing, 71);
    PlainModel model = load_model(gm.manifest, std::span<const u8>(gm.blob.data(), gm.blob.size()));
    auto input = make_random_input(model.shapes.at("input"), batch, 99);
    InferenceServer ref_server;
    ref_server.set_threads(std::thread::hardware_concurrency());
    ref_server.add_model("cryptonets-relu", model, ctx);
    henet::gpu::InferenceServer gpu_server;
    gpu_server.add_model("cryptonets-relu", model, ctx);
    SessionConfig config;
    config.preset = pr;
    config.packing = packing;
    config.model_id = "cryptonets-relu";
    config.batch = batch;
    std::string e1, e2;
    auto [rc, rs] = session(ref_server, ctx, config, input, keys.secret, 1234, &e1);
    auto [gc, gs] = session(gpu_server, ctx, config, input, keys.secret, 1234, &e2);
    const bool good = e1.empty() && e2.empty() && rc.outputs == gc.outputs && !gc.outputs.empty() &&
                      gc.stats.nonlin_round_trips == 2 && same_stats(rc.stats, gc.stats) && same_stats(rs, gs) &&
                      gs.interactive_bytes == gc.stats.interactive_bytes;
    std::printf("%-40s %s (%zu outputs x %zu, %llu bytes sent by the server, %zu layer timings)\n",
                (std::string("server session ") + preset_name(pr)).c_str(), good ? "bit-identical" : "MISMATCH",
                gc.outputs.size(), gc.outputs.empty() ? 0 : gc.outputs[0].size(),
                (unsigned long long)gs.bytes_sent, gs.layer_ms.size());
    if (!good) std::printf("  ref error '%s' gpu error '%s'\n", e1.c_str(), e2.c_str());
    ok &= good;
    // rejected sessions: unknown model, wrong preset, batch outside capacity
    for (int k = 0; k < 3; ++k) {
      SessionConfig bad = config;
      if (k == 0) bad.model_id = "nope";
      if (k == 1) bad.preset = pr == Preset::P11 ? Preset::P13 : Preset::P11;
      if (k == 2) bad.batch = batch_capacity(*ctx, packing) + 1;
      std::string r1, r2;
      auto in2 = make_random_input(model.shapes.at("input"), bad.batch, 5);
      auto [x1, y1] = session(ref_server, ctx, bad, in2, keys.secret, 1, &r1);
      auto [x2, y2] = session(gpu_server, ctx, bad, in2, keys.secret, 1, &r2);
      const bool same = r1 == r2 && same_stats(y1, y2);
      std::printf("  rejected session %d: %s (%s)\n", k, same ? "identical" : "MISMATCH", r2.c_str());
      ok &= same;
    }
  }
  return ok;
}

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[1]) == "--bench") return bench(std::atoi(argv[2]));
  auto ctx = baseline_ctx();
  KeyPair keys = keygen(*ctx, 2024, true);
  bool ok = true;
  ok &= run_model(ctx, keys, make_cryptonets(Preset::P13, 1), PackingMode::Real, 4096, "make_cryptonets (c2 topology)");
  ok &= run_model(ctx, keys, make_cryptonets_relu(Preset::P13, PackingMode::Complex, 2), PackingMode::Complex, 8192,
                  "make_cryptonets_relu complex (c3)");
  ok &= run_model(ctx, keys, make_cryptonets_shaped_toy(Preset::P13, 3), PackingMode::Real, 64, "cryptonets toy");
  // the reference's own parameter presets (henet/params.hpp:74-101) through
  // CkksContext::create, as `henet run` builds them (proj/tools/henet.cpp:377): 41/51-bit
  // primes (P13, P14), a 41-bit special prime over ~2^30 primes (P12), and N = 2^11 with a
  // single 54-bit prime and no special prime (P11, client-aided ReLU network)
  for (Preset pr : {Preset::P12, Preset::P13, Preset::P14, Preset::P11}) {
    auto pctx = CkksContext::create(pr);
    KeyPair pkeys = keygen(*pctx, 2025, pctx->has_special());
    const std::string nm = std::string("preset ") + preset_name(pr);
    if (pr == Preset::P11 || pr == Preset::P12) {  // depth-1 client-aided networks
      ok &= run_model(pctx, pkeys, make_cryptonets_relu(pr, PackingMode::Real, 4), PackingMode::Real, 1024,
                      (nm + " make_cryptonets_relu").c_str());
    } else if (pr == Preset::P13) {
      ok &= run_model(pctx, pkeys, make_cryptonets(pr, 1), PackingMode::Real, 4096, (nm + " make_cryptonets").c_str());
    } else {
      ok &= run_model(pctx, pkeys, make_cryptonets_shaped_toy(pr, 3), PackingMode::Real, 64,
                      (nm + " cryptonets toy").c_str());
    }
  }
  // client side: encrypt_tensor / decrypt_tensor, and execute with the GPU LocalProvider
  {
    PlainModel model = load_model(make_cryptonets_relu(Preset::P13, PackingMode::Complex, 2).manifest,
                                  std::span<const u8>(make_cryptonets_relu(Preset::P13, PackingMode::Complex, 2).blob));
    BatchInput in = make_random_input(model.shapes.at(model.input_node().id), 8192, 6);
    CipherTensor xc = encrypt_tensor(*ctx, in, keys.secret, 78, PackingMode::Complex, std::thread::hardware_concurrency());
    CipherTensor xg = henet::gpu::encrypt_tensor(*ctx, in, keys.secret, 78, PackingMode::Complex);
    ok &= same(xc, xg, "encrypt_tensor complex (c3 input)");
    RescalePlan plan = plan_lazy_rescaling(*ctx, model);
    LocalProvider prov(NonlinearityEngine(ctx, keys.secret, 99));
    henet::gpu::LocalProvider gprov(ctx, keys.secret, 99);
    ExecutionConfig cfg;
    cfg.threads = std::thread::hardware_concurrency();
    cfg.provider = &prov;
    CipherTensor want = henet::execute(ctx, model, plan, xc, cfg);
    cfg.provider = &gprov;
    CipherTensor got = henet::gpu::execute(ctx, model, plan, xc, cfg);
    ok &= same(want, got, "c3 with gpu::LocalProvider (device refresh)");
    auto dc = decrypt_tensor(*ctx, want, keys.secret, 8192);
    auto dg = henet::gpu::decrypt_tensor(*ctx, got, keys.secret, 8192);
    const bool dec_ok = dc == dg;
    std::printf("%-40s %s\n", "decrypt_tensor (c3 logits)", dec_ok ? "bit-identical" : "MISMATCH");
    // the GPU provider through the host interface, as another executor would call it
    std::vector<Ciphertext> some(xc.elems.begin(), xc.elems.begin() + 4);
    const bool pv_ok = prov.apply(NonlinKind::Relu, 1, 3, some).size() == 4 &&
                       prov.apply(NonlinKind::MaxPool, 4, 5, some)[0].polys == gprov.apply(NonlinKind::MaxPool, 4, 5, some)[0].polys &&
                       prov.apply(NonlinKind::Relu, 1, 3, some)[2].polys == gprov.apply(NonlinKind::Relu, 1, 3, some)[2].polys;
    std::printf("%-40s %s\n", "gpu::LocalProvider::apply (host ciphertexts)", pv_ok ? "bit-identical" : "MISMATCH");
    ok &= dec_ok && pv_ok;
  }
  // op level
  {
    std::vector<double> v(4096, 0.25);
    Ciphertext ct = encrypt_batch(*ctx, pack_real(v), keys.secret, 5);
    Ciphertext sq = square(*ctx, ct);
    bool r1 = henet::relinearize(*ctx, sq, *keys.relin).polys == henet::gpu::relinearize(*ctx, sq, *keys.relin).polys;
    bool r2 = henet::rescale(*ctx, ct, 3).polys == henet::gpu::rescale(*ctx, ct, 3).polys;
    auto pt = encode_scalar(*ctx, -0.37, ct.level(), ctx->params().default_scale);
    bool r3 = henet::mul_ct_pt_scalar(*ctx, ct, pt).polys == henet::gpu::mul_ct_pt_scalar(*ctx, ct, pt).polys;
    std::printf("op level: relinearize %s, rescale %s, mul_ct_pt_scalar %s\n", r1 ? "ok" : "MISMATCH",
                r2 ? "ok" : "MISMATCH", r3 ? "ok" : "MISMATCH");
    ok &= r1 && r2 && r3;
  }
  // error behaviour: ValidationError for a bad rescale target, as the reference
  {
    std::vector<double> v(16, 1.0);
    Ciphertext ct = encrypt_batch(*ctx, pack_real(v), keys.secret, 6);
    Ciphertext low = henet::rescale(*ctx, ct, 1);
    bool threw = false;
    try {
      henet::gpu::rescale(*ctx, low, 1);
    } catch (const ValidationError&) {
      threw = true;
    }
    std::printf("ValidationError on rescale below level 1: %s\n", threw ? "ok" : "MISSING");
    ok &= threw;
  }
  ok &= protocol_checks();
  // output-sharded Dot through the library's NCCL communicator (one GPU here: world size 1)
  {
    henet::detail::BlobBuilder blob(7);
    blob.add_random("w", {96, 40}, 0.1);
    blob.add_random("b", {40}, 0.01);
    nlohmann::json j;
    j["name"] = "dense-96-40";
    j["packing"] = "real";
    j["preset"] = "P13";
    j["weights"] = blob.table();
    j["nodes"] = nlohmann::json::array(
        {henet::detail::node_json("input", "Input", {}, {{"shape", {96}}}),
         henet::detail::node_json("fc", "Dot", {"input"}, nlohmann::json::object(), "w", "b"),
         henet::detail::node_json("out", "Output", {"fc"})});
    auto bytes = blob.take_bytes();
    PlainModel m = load_model(j.dump(), std::span<const u8>(bytes.data(), bytes.size()));
    RescalePlan plan = plan_lazy_rescaling(*ctx, m);
    BatchInput in = make_random_input(m.shapes.at("input"), 256, 8);
    CipherTensor x = encrypt_tensor(*ctx, in, keys.secret, 81, PackingMode::Real, std::thread::hardware_concurrency());
    ExecutionConfig cfg;
    cfg.threads = std::thread::hardware_concurrency();
    CipherTensor want = henet::execute(ctx, m, plan, x, cfg);
    henet::gpu::Communicator comm(*ctx, henet::gpu::comm_unique_id(), 1, 0);
    ok &= same(want, henet::gpu::execute_output_sharded(ctx, m, plan, x, comm), "output-sharded Dot (NCCL, 1 rank)");
  }
  std::printf(ok ? "DROPIN OK\n" : "DROPIN FAILED\n");
  return ok ? 0 : 1;
}
