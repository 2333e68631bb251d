// TEST INFRASTRUCTURE ONLY — links the reference's OWN /root/reference/proj/src/config.cpp
// (compiled where it lies, against the declaration-only Eigen stand-in in eigen_decl/) into
// oracle/_ref/libref_config.so, so the product's config front-end (paper_2110_11199_b200/config.py)
// is pinned to the reference parser: tests/golden/make_config_golden.py records, for a list of
// config texts, RunConfig::parse_text(text).resolved_text() or the ConfigError message.
// config.cpp needs engine::strategy_name / strategy_from_name (engine.cpp:25-43, restated below:
// engine.cpp itself needs Eigen) and the toy-objective factories, which parsing never calls.
#include <cstring>
#include <stdexcept>
#include <string>

#include "adpsgd/config.hpp"
#include "adpsgd/errors.hpp"

namespace adpsgd::engine {
std::string strategy_name(Strategy s) {  // engine.cpp:25-34
    switch (s) {
        case Strategy::Sdpsgd: return "SDPSGD";
        case Strategy::AdpsgdFm: return "ADPSGD_FM";
        case Strategy::AdpsgdRm: return "ADPSGD_RM";
        case Strategy::AdpsgdD1d: return "ADPSGD_D1D";
        case Strategy::GenericStaleness: return "GENERIC";
    }
    return "unknown";
}
Strategy strategy_from_name(const std::string& name) {  // engine.cpp:36-43
    if (name == "SDPSGD") return Strategy::Sdpsgd;
    if (name == "ADPSGD_FM") return Strategy::AdpsgdFm;
    if (name == "ADPSGD_RM") return Strategy::AdpsgdRm;
    if (name == "ADPSGD_D1D") return Strategy::AdpsgdD1d;
    if (name == "GENERIC") return Strategy::GenericStaleness;
    throw ConfigError("unknown strategy: " + name);
}
}  // namespace adpsgd::engine

namespace adpsgd::objectives {
Problem make_quadratic(int, double, double, std::uint64_t, int) { throw std::logic_error("not linked"); }
Problem make_logistic(int, int, std::uint64_t) { throw std::logic_error("not linked"); }
Problem make_mlp(int, int, int, int, std::uint64_t) { throw std::logic_error("not linked"); }
}  // namespace adpsgd::objectives

extern "C" {
// 0: `out` = resolved_text(); 1: ConfigError, `out` = its message; 2: another exception.
int ref_config_resolve(const char* text, char* out, size_t n) {
    std::string s;
    int rc = 0;
    try {
        s = adpsgd::cfg::RunConfig::parse_text(text).resolved_text();
    } catch (const adpsgd::ConfigError& e) {
        s = e.what();
        rc = 1;
    } catch (const std::exception& e) {
        s = e.what();
        rc = 2;
    }
    std::strncpy(out, s.c_str(), n - 1);
    out[n - 1] = '\0';
    return rc;
}
}
