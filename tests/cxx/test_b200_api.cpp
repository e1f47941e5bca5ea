// Tests of the device-resident C++ API (include/covap/b200_api.hpp:
// covap::b200::Plan / State / Sync) — the production form of
// trainer.cpp:365-386 for one rank that INTEGRATION.md recommends — against
// the value-semantics drop-in (covap_compress + covap_decompress, itself
// checked against the reference by its own unit tests).  Needs a GPU.
#include <cstdint>
#include <cstring>
#include <vector>

#include "covap/b200_api.hpp"
#include "covap_c.h"
#include "doctest.h"

using namespace covap;

namespace {

ModelSpec small_model() {
  // two oversized layers (sharded at K = 3), a tiny bucket between them, and
  // a multi-layer bucket
  ModelSpec m;
  const std::uint64_t sizes[] = {40000, 7, 120000, 9000, 3, 65000, 1500};
  for (std::size_t i = 0; i < sizeof(sizes) / sizeof(sizes[0]); ++i)
    m.layers.push_back(LayerSpec{"l" + std::to_string(i), sizes[i]});
  m.bucket_cap_bytes = 200000;
  return m;
}

struct Dev {
  void* p = nullptr;
  explicit Dev(std::uint64_t bytes) { REQUIRE(covap_device_alloc(0, bytes, &p) == COVAP_OK); }
  ~Dev() { covap_device_free(0, p); }
};

std::vector<double> gaussian(std::uint64_t n, std::uint64_t seed) {
  SplitMix64 rng(seed);
  std::vector<double> v(n);
  for (auto& x : v) x = rng.next_normal();
  return v;
}

bool bit_equal(const std::vector<double>& a, const std::vector<double>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * sizeof(double)) == 0;
}

}  // namespace

TEST_CASE("device-resident sync equals compress then decompress, step by step") {
  const ModelSpec model = small_model();
  const std::uint32_t K = 3;
  const EfSchedule ef{true, 0.3, 2, 0.2};
  const BucketPlan plan = shard_plan(allocate_buckets(model), K);
  const std::vector<std::uint64_t> numels = effective_numels(plan);
  std::uint64_t n = 0;
  for (auto x : numels) n += x;
  REQUIRE(numels.size() > 3);  // the sharding took place

  b200::Plan dplan(model, K);
  b200::Sync sync(dplan, nullptr, COVAP_F64, 0, ef);
  Dev g(n * 8), out(n * 8);
  CompressorState st = CompressorState::zeros(numels);
  const CovapConfig cfg{K, SelectionRule::kMatchStep, ef};
  for (std::uint64_t s = 0; s < 2 * K + 1; ++s) {
    const std::vector<double> flat = gaussian(n, 100 + s);
    GradientSet grads;
    std::uint64_t off = 0;
    for (auto x : numels) {
      grads.emplace_back(flat.begin() + off, flat.begin() + off + x);
      off += x;
    }
    const CompressedUpdate u = covap_compress(grads, st, cfg);
    const GradientSet dense = covap_decompress(u, numels);
    std::vector<double> want;
    for (const auto& t : dense) want.insert(want.end(), t.begin(), t.end());

    REQUIRE(covap_memcpy(g.p, flat.data(), n * 8, 0, nullptr) == COVAP_OK);
    sync.step(g.p, out.p, nullptr);
    std::vector<double> got(n);
    REQUIRE(covap_memcpy(got.data(), out.p, n * 8, 1, nullptr) == COVAP_OK);
    REQUIRE(covap_stream_synchronize(nullptr) == COVAP_OK);
    CHECK(bit_equal(got, want));
    CHECK(sync.state().num_steps() == s + 1);
  }
}

TEST_CASE("per-bucket overlapped schedule equals the standalone step") {
  const ModelSpec model = small_model();
  const std::uint32_t K = 3;
  const EfSchedule ef{true, 0.5, 1, 0.1};
  b200::Plan dplan(model, K);
  b200::Sync a(dplan, nullptr, COVAP_F32, 0, ef);
  b200::Sync b(dplan, nullptr, COVAP_F32, 0, ef);
  const covap_plan_info info = dplan.info();
  const std::uint64_t n = info.device_numel;
  Dev g(n * 4), oa(n * 4), ob(n * 4);
  for (std::uint64_t s = 0; s < K + 2; ++s) {
    const std::vector<double> d = gaussian(n, 500 + s);
    std::vector<float> f(d.begin(), d.end());
    REQUIRE(covap_memcpy(g.p, f.data(), n * 4, 0, nullptr) == COVAP_OK);
    a.step(g.p, oa.p, nullptr);
    for (std::size_t bk = 0; bk < info.n_buckets; ++bk) b.bucket_ready(bk, g.p, ob.p, nullptr);
    b.finish(nullptr);
    std::vector<float> xa(n), xb(n);
    REQUIRE(covap_memcpy(xa.data(), oa.p, n * 4, 1, nullptr) == COVAP_OK);
    REQUIRE(covap_memcpy(xb.data(), ob.p, n * 4, 1, nullptr) == COVAP_OK);
    REQUIRE(covap_stream_synchronize(nullptr) == COVAP_OK);
    CHECK(std::memcmp(xa.data(), xb.data(), n * 4) == 0);
  }
}

TEST_CASE("device-resident API raises the reference's exception classes") {
  ModelSpec empty;
  bool threw = false;
  try {
    b200::Plan p(empty, 2);
  } catch (const InvalidInput&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    b200::Plan p(small_model(), 0);  // K < 1 (model.cpp:96-99)
  } catch (const InvalidInput&) {
    threw = true;
  }
  CHECK(threw);
}

TEST_CASE("covap settings, resolve_interval and the CCR controller (host)") {
  // the "covap" section of the reference's test document (test_config.cpp:18-39)
  const std::string doc =
      R"({"name": "unit", "covap": {"interval": "auto", "selection": "formula",
          "ef": {"enabled": true, "init_value": 0.3, "ascend_steps": 10, "ascend_range": 0.1}}})";
  const CovapSettings s = covap_settings_from_json(doc);
  CHECK(s.auto_interval);
  CHECK(s.rule == SelectionRule::kPlusStep);
  CHECK(s.ef.ascend_steps == 10);
  CHECK(resolve_interval(s, 2.5) == 3);  // test_config.cpp:59-60
  CHECK(resolve_interval(s, 0.2) == 1);
  const CovapSettings fixed = covap_settings_from_json(R"({"covap": {"interval": 7}})");
  CHECK(resolve_interval(fixed, 2.5) == 7);
  bool threw = false;
  try {
    covap_settings_from_json(R"({"covap": {"interval": 0}})");
  } catch (const ConfigError& e) {
    threw = std::string(e.what()).find("covap.interval") != std::string::npos;
  }
  CHECK(threw);
  // one rank: the controller is ccr / choose_interval of the summed durations
  const b200::CcrController ctl(nullptr);
  const ProfileResult r = ctl.decide({100.0, -1.0, 180.0}, 135.0);
  CHECK(r.comm_aligned_ms == 280.0);
  CHECK(r.recommended_interval == 3);  // test_perf.cpp:36
  CHECK(ctl.interval(s, {100.0, 180.0}, 135.0) == 3);
  CHECK(ctl.interval(fixed, {100.0, 180.0}, 135.0) == 7);
  // overlap_schedule over the C-ABI (perf.cpp:63-103; test_perf.cpp:67-81)
  const std::vector<double> comp = {10, 10, 10}, comm = {4, 4, 4};
  const OverlapSchedule o = overlap_schedule(7, comp, {}, comm, {});
  CHECK(o.total_ms == 37);
  CHECK(o.bubbles.size() == 2);
}

TEST_CASE("peer collective over an NCCL window equals the NCCL step (one rank)") {
  const ModelSpec model = small_model();
  const std::uint32_t K = 3;
  const EfSchedule ef{true, 0.3, 2, 0.2};
  b200::Plan dplan(model, K);
  const b200::Comm comm(b200::Comm::unique_id(), 1, 0, 0);
  const std::uint64_t n = dplan.info().device_numel;
  for (int mode = 0; mode <= 2; ++mode) {
    b200::Sync ref(dplan, &comm, COVAP_F32, 0, ef);
    b200::State st(dplan, COVAP_F32, 0, ef);
    b200::PeerSync peer(st, comm, false, mode);
    CHECK_FALSE(peer.multimem());
    Dev g(n * 4), oa(n * 4), ob(n * 4);
    for (std::uint64_t s = 0; s < 2 * K + 1; ++s) {
      const std::vector<double> d = gaussian(n, 900 + s);
      std::vector<float> f(d.begin(), d.end());
      REQUIRE(covap_memcpy(g.p, f.data(), n * 4, 0, nullptr) == COVAP_OK);
      ref.step(g.p, oa.p, nullptr);
      peer.step(g.p, ob.p, nullptr);
      std::vector<float> xa(n), xb(n);
      REQUIRE(covap_memcpy(xa.data(), oa.p, n * 4, 1, nullptr) == COVAP_OK);
      REQUIRE(covap_memcpy(xb.data(), ob.p, n * 4, 1, nullptr) == COVAP_OK);
      REQUIRE(covap_stream_synchronize(nullptr) == COVAP_OK);
      CHECK(std::memcmp(xa.data(), xb.data(), n * 4) == 0);
    }
    peer.check_timeouts();
  }
  // one rank has no NVSwitch multicast team: refused, not a silent fallback
  b200::State st(dplan, COVAP_F32, 0, ef);
  CHECK_THROWS_AS(b200::PeerSync(st, comm, true), covap::Error);
}
