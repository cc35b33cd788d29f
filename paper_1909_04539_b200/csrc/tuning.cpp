// Tuning overrides: forced plans, ring depths, fused/unfused paths, the
// host staging chunk, the L2 set-aside. The planner consults this table on
// every solve; it is set through bandsolve_tune_set() and seeded ONCE (at
// first use) from the matching BANDSOLVE_<KEY> environment variables, so a
// process's environment is read at one point and later changes to it do not
// steer a running library. Unknown keys are rejected.
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "internal.hpp"

namespace bsb {
namespace {

// every key the library consults (documented in include/bandsolve.h)
const char* const kKeys[] = {
    "PLAN",       "PWARPS",         "PTAIL",       "SWG",         "STAIL",           "SKB",
    "SKR",        "SPD",            "SV",          "SRC",         "SSEG",            "TM8",
    "TMEM",       "SSTAG",          "PARTITION",   "PART_K",      "CN_UNFUSED",      "PERIODIC_UNFUSED",
    "ADI_UNFUSED", "ADI_FUSE_PENT", "HOST_CHUNK_MIB", "L2_SETASIDE", "SPIKE", "SPIKE_K", "SPIKE_F32_MIN_N", "NO_PDL", "GLOBAL_NOREC", "PART_NOSTAGE", "SPIKE_CUT", "PIPE", "PKB", "PIPE_MAX_N", "PIPE_L2_P", "PRT", "PIPE_CN",
};

bool known(const char* key) {
  for (const char* k : kKeys)
    if (std::strcmp(k, key) == 0) return true;
  return false;
}

struct Table {
  std::mutex mu;
  std::map<std::string, std::string> values;
  bool seeded = false;

  void seed_locked() {
    values.clear();
    for (const char* k : kKeys) {
      const std::string env = std::string("BANDSOLVE_") + k;
      if (const char* v = std::getenv(env.c_str())) values[k] = v;
    }
    seeded = true;
  }
};

Table& table() {
  static Table* t = new Table;  // never destroyed: solves may run during static teardown
  return *t;
}

}  // namespace

std::optional<std::string> tune_str(const char* key) {
  Table& t = table();
  std::lock_guard<std::mutex> lock(t.mu);
  if (!t.seeded) t.seed_locked();
  auto it = t.values.find(key);
  if (it == t.values.end()) return std::nullopt;
  return it->second;
}

long long tune_int(const char* key, long long dflt) {
  const auto v = tune_str(key);
  if (!v) return dflt;
  return std::strtoll(v->c_str(), nullptr, 10);
}

bool tune_flag(const char* key) { return tune_str(key).has_value(); }

bool tune_set(const char* key, const char* value) {
  if (!key || !known(key)) return false;
  Table& t = table();
  std::lock_guard<std::mutex> lock(t.mu);
  if (!t.seeded) t.seed_locked();
  if (value) t.values[key] = value;
  else t.values.erase(key);
  return true;
}

void tune_reset() {
  Table& t = table();
  std::lock_guard<std::mutex> lock(t.mu);
  t.values.clear();
  t.seeded = true;  // a reset table ignores the environment from here on
}

}  // namespace bsb
