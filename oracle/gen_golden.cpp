// TEST INFRASTRUCTURE ONLY — golden-fixture generator.
//
// Linked against the reference library compiled from its own sources
// (oracle/Makefile `ref`) and the reference's test support
// (proj/tests/support/oracles.cpp), this program replays the reference's
// own test cases with their own seeds and generators and dumps inputs and
// the reference's outputs. tests/golden/make_golden.py turns the dump into
// the committed .npz fixtures. Each case names the reference test it
// replays (file:line).
//
// Dump format (little endian), repeated per record:
//   u32 case_len, case bytes, u32 key_len, key bytes, u64 count, f64[count]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "bandsolve/banded.hpp"
#include "bandsolve/batch.hpp"
#include "bandsolve/dense.hpp"
#include "bandsolve/pent_solver.hpp"
#include "bandsolve/tri_solver.hpp"
#include "support/oracles.hpp"

using namespace bandsolve;
using testsup::rng;

namespace {

FILE* g_out = nullptr;

void put(const std::string& name, const std::string& key, const double* p,
         std::size_t count) {
  const std::uint32_t nl = static_cast<std::uint32_t>(name.size());
  const std::uint32_t kl = static_cast<std::uint32_t>(key.size());
  const std::uint64_t c = count;
  std::fwrite(&nl, 4, 1, g_out);
  std::fwrite(name.data(), 1, nl, g_out);
  std::fwrite(&kl, 4, 1, g_out);
  std::fwrite(key.data(), 1, kl, g_out);
  std::fwrite(&c, 8, 1, g_out);
  if (count) std::fwrite(p, 8, count, g_out);
}
void put(const std::string& name, const std::string& key,
         const real_buffer& b) {
  put(name, key, b.data(), b.size());
}
void put(const std::string& name, const std::string& key,
         const interleaved_batch& b) {
  put(name, key, b.data(), b.size());
}
void put_scalar(const std::string& name, const std::string& key, double v) {
  put(name, key, &v, 1);
}

void dump_tri_case(const std::string& name, const tri_lhs& lhs,
                   const interleaved_batch& rhs, bool dense) {
  const tri_factor f = tri_prefactor(lhs);
  interleaved_batch x = rhs;
  tri_solve_shared_batch(f, x);
  put_scalar(name, "n", static_cast<double>(lhs.n));
  put_scalar(name, "m", static_cast<double>(rhs.systems()));
  put(name, "sub", lhs.sub);
  put(name, "diag", lhs.diag);
  put(name, "sup", lhs.sup);
  put(name, "chat", f.chat);
  put(name, "inv_denom", f.inv_denom);
  put(name, "rhs", rhs);
  put(name, "x", x);
  put_scalar(name, "residual", tri_residual_max(lhs, x, rhs));
  if (dense) {
    put_scalar(name, "dense_err",
               testsup::max_error_vs_dense(testsup::dense_from_tri(lhs), x,
                                           rhs));
  }
}

void dump_pent_case(const std::string& name, const pent_lhs& lhs,
                    const interleaved_batch& rhs, bool dense) {
  const pent_factor f = pent_prefactor(lhs);
  interleaved_batch x = rhs;
  pent_solve_shared_batch(f, x);
  put_scalar(name, "n", static_cast<double>(lhs.n));
  put_scalar(name, "m", static_cast<double>(rhs.systems()));
  put(name, "a", lhs.a);
  put(name, "b", lhs.b);
  put(name, "c", lhs.c);
  put(name, "d", lhs.d);
  put(name, "e", lhs.e);
  put(name, "inv_alpha", f.inv_alpha);
  put(name, "beta", f.beta);
  put(name, "gamma", f.gamma);
  put(name, "delta", f.delta);
  put(name, "epsilon", f.epsilon);
  put(name, "rhs", rhs);
  put(name, "x", x);
  put_scalar(name, "residual", pent_residual_max(lhs, x, rhs));
  if (dense) {
    put_scalar(name, "dense_err",
               testsup::max_error_vs_dense(testsup::dense_from_pent(lhs), x,
                                           rhs));
  }
}

void dump_uniform_case(const std::string& name, const uniform_pent_lhs& u,
                       const interleaved_batch& rhs) {
  const uniform_pent_factor uf = uniform_prefactor(u);
  interleaved_batch x = rhs;
  pent_solve_uniform_batch(uf, x);
  put_scalar(name, "n", static_cast<double>(u.n));
  put_scalar(name, "m", static_cast<double>(rhs.systems()));
  const double bands[5] = {u.a, u.b, u.c, u.d, u.e};
  put(name, "bands", bands, 5);
  put(name, "inv_alpha", uf.inv_alpha);
  put(name, "beta", uf.beta);
  put(name, "gamma", uf.gamma);
  put(name, "delta", uf.delta);
  put_scalar(name, "eps_scalar", uf.eps_scalar);
  put(name, "rhs", rhs);
  put(name, "x", x);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc != 2) {
    std::fprintf(stderr, "usage: gen_golden <out.bin>\n");
    return 2;
  }
  g_out = std::fopen(argv[1], "wb");
  if (!g_out) return 1;

  // ---- prefactor known-answer inputs (test_banded_core.cpp:35-55, :111-148)
  {
    const tri_lhs lhs = constant_tri_lhs(-0.5, 2.0, -0.5, 4);
    dump_tri_case("kat_tri_sigma05_n4", lhs, interleave({{1, 0, 0, 1}}), true);
    const pent_lhs p = constant_pent_lhs(0.25, -1.0, 2.5, -1.0, 0.25, 6);
    interleaved_batch e1(6, 1);
    e1.at(0, 0) = 1.0;
    dump_pent_case("kat_pent_sigma025_n6", p, e1, true);  // test_pent_solver.cpp:31-40
  }
  // ---- tri shared solve (test_tri_solver.cpp)
  {
    rng r(1);  // :13-20 identity
    const tri_lhs eye = constant_tri_lhs(0, 1, 0, 8);
    dump_tri_case("tri_identity_n8_m3", eye, testsup::random_batch(r, 8, 3), true);
  }
  {
    rng r(12);  // :32-41
    const tri_lhs lhs = testsup::random_dominant_tri(r, 32);
    dump_tri_case("tri_random_n32_m7", lhs, testsup::random_batch(r, 32, 7), true);
  }
  {
    rng r(32);  // :148-164 determinism
    const tri_lhs lhs = testsup::random_dominant_tri(r, 40);
    dump_tri_case("tri_determinism_n40_m13", lhs, testsup::random_batch(r, 40, 13), true);
  }
  {
    rng r(33);  // :166-175 residual, n = 1024 (beyond the dense oracle)
    const tri_lhs lhs = testsup::random_dominant_tri(r, 1024);
    dump_tri_case("tri_residual_n1024_m2", lhs, testsup::random_batch(r, 1024, 2), false);
  }
  {
    rng r(101);  // test_banded_core.cpp:57-66
    const tri_lhs lhs = testsup::random_dominant_tri(r, 5);
    dump_tri_case("tri_prefactor_dense_n5", lhs, testsup::random_batch(r, 5, 1), true);
  }
  {
    // test_capi.cpp:49-83: sigma = 1/2 bands, rhs sin(0.7 k)
    const std::size_t n = 8;
    const tri_lhs lhs = constant_tri_lhs(-0.5, 2.0, -0.5, n);
    interleaved_batch rhs(n, 2);
    for (std::size_t k = 0; k < 2 * n; ++k) rhs.data()[k] = std::sin(0.7 * static_cast<double>(k));
    dump_tri_case("tri_capi_n8_m2", lhs, rhs, true);
  }
  {
    rng r(404);  // test_banded_core.cpp:252-265 property, 25 trials
    for (int trial = 0; trial < 25; ++trial) {
      const std::size_t n = r.index(2, 64);
      const tri_lhs lhs = testsup::random_dominant_tri(r, n);
      const interleaved_batch rhs = testsup::random_batch(r, n, 3);
      dump_tri_case("tri_property_" + std::to_string(trial), lhs, rhs, true);
    }
  }
  {
    rng r(1001);  // acceptance_main.cpp:41-61 criterion 1, first 16 trials
    for (int trial = 0; trial < 16; ++trial) {
      const std::size_t n = r.index(4, 256);
      const std::size_t m = r.index(1, 32);
      const tri_lhs lhs = testsup::random_dominant_tri(r, n);
      const interleaved_batch rhs = testsup::random_batch(r, n, m);
      dump_tri_case("tri_accept1_" + std::to_string(trial), lhs, rhs, true);
    }
  }
  // ---- pent shared / uniform solve (test_pent_solver.cpp)
  {
    rng r(1);  // :22-29
    const pent_lhs eye = constant_pent_lhs(0, 0, 1, 0, 0, 9);
    dump_pent_case("pent_identity_n9_m4", eye, testsup::random_batch(r, 9, 4), true);
  }
  {
    rng r(13);  // :42-51
    const pent_lhs lhs = testsup::random_dominant_pent(r, 48);
    dump_pent_case("pent_random_n48_m5", lhs, testsup::random_batch(r, 48, 5), true);
  }
  {
    rng r(43);  // :221-237 determinism
    const pent_lhs lhs = testsup::random_dominant_pent(r, 30);
    dump_pent_case("pent_determinism_n30_m11", lhs, testsup::random_batch(r, 30, 11), true);
  }
  {
    rng r(40);  // :165-177 uniform == shared bitwise
    const uniform_pent_lhs u{0.25, -1.0, 2.5, -1.0, 0.25, 32};
    const interleaved_batch rhs = testsup::random_batch(r, 32, 4);
    dump_uniform_case("uniform_n32_m4", u, rhs);
    dump_pent_case("uniform_n32_m4_shared",
                   constant_pent_lhs(u.a, u.b, u.c, u.d, u.e, u.n), rhs, true);
  }
  {
    // test_capi.cpp:102-141: hyperdiffusion sigma = 1/4, rhs cos(0.3 k)
    const std::size_t n = 12;
    const pent_lhs lhs = constant_pent_lhs(0.25, -1.0, 2.5, -1.0, 0.25, n);
    interleaved_batch rhs(n, 3);
    for (std::size_t k = 0; k < 3 * n; ++k) rhs.data()[k] = std::cos(0.3 * static_cast<double>(k));
    dump_pent_case("pent_capi_n12_m3", lhs, rhs, true);
    dump_uniform_case("uniform_capi_n12_m3", uniform_pent_lhs{0.25, -1.0, 2.5, -1.0, 0.25, n}, rhs);
  }
  {
    rng r(56);  // test_banded_core.cpp:157-165 LR reassembly sizes
    for (std::size_t n : {5, 6, 7, 16, 33, 64}) {
      const pent_lhs lhs = testsup::random_dominant_pent(r, n);
      const pent_factor f = pent_prefactor(lhs);
      const std::string name = "pent_lr_n" + std::to_string(n);
      interleaved_batch one(n, 1);
      for (std::size_t i = 0; i < n; ++i) one.at(i, 0) = 1.0;
      dump_pent_case(name, lhs, one, true);
      put_scalar(name, "lr_err", testsup::lr_reassembly_error(lhs, f));
    }
  }
  {
    rng r(2002);  // acceptance_main.cpp:64-88 criterion 2, first 16 trials
    for (int trial = 0; trial < 16; ++trial) {
      const std::size_t n = r.index(5, 256);
      const std::size_t m = r.index(1, 32);
      const pent_lhs lhs = testsup::random_dominant_pent(r, n);
      const interleaved_batch rhs = testsup::random_batch(r, n, m);
      dump_pent_case("pent_accept2_" + std::to_string(trial), lhs, rhs, true);
    }
  }
  {
    rng r(3003);  // acceptance_main.cpp:91-138 criterion 3 (constant pent bands)
    const std::size_t ns[3] = {8, 32, 128};
    for (std::size_t n : ns) {
      const auto cb = testsup::random_dominant_pent_const(r);
      const interleaved_batch rhs = testsup::random_batch(r, n, 4);
      const std::string name = "uniform_const_n" + std::to_string(n);
      dump_uniform_case(name, uniform_pent_lhs{cb.a, cb.b, cb.c, cb.d, cb.e, n}, rhs);
    }
  }
  std::fclose(g_out);
  return 0;
}
