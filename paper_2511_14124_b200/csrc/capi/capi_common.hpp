// Shared helpers of the extern "C" layer: error state and exception mapping.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "tencache/tencache.hpp"
#include "tencache_c.h"

namespace tcb {

int set_error(int code, const std::string& msg);
tencache::RunConfig parse_run_config(const char* cfg_json);
tencache::MachineConfig machine_from(const char* path);
// SimReport as JSON text (exact rationals as "n/d" strings); shared by tc_run,
// tc_sweep and the tencache_sim CLI.
std::string report_json_text(const tencache::SimReport& r);

// Runtime failures of the data plane (CUDA / NCCL / file I/O).
struct DeviceError : std::runtime_error {
  int code;
  DeviceError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

}  // namespace tcb

// Maps every reference exception type to its status code.
#define TC_GUARD(...)                                                                    \
  try {                                                                                  \
    __VA_ARGS__                                                                          \
  } catch (const tencache::ConfigError& e) {                                             \
    return tcb::set_error(TC_ECONFIG, std::string("ConfigError: ") + e.what());          \
  } catch (const tencache::OomError& e) {                                                \
    return tcb::set_error(TC_EOOM, std::string("OomError: ") + e.what());                \
  } catch (const tencache::TraceError& e) {                                              \
    return tcb::set_error(TC_ETRACE, std::string("TraceError: ") + e.what());            \
  } catch (const tencache::PoolError& e) {                                               \
    return tcb::set_error(TC_EPOOL, std::string("PoolError: ") + e.what());              \
  } catch (const tcb::DeviceError& e) {                                                  \
    return tcb::set_error(e.code, e.what());                                             \
  } catch (const std::invalid_argument& e) {                                             \
    return tcb::set_error(TC_EARG, std::string("invalid_argument: ") + e.what());        \
  } catch (const std::domain_error& e) {                                                 \
    return tcb::set_error(TC_EARG, std::string("domain_error: ") + e.what());            \
  } catch (const std::logic_error& e) {                                                  \
    return tcb::set_error(TC_EINTERNAL, std::string("logic_error: ") + e.what());        \
  } catch (const std::bad_alloc& e) {                                                    \
    return tcb::set_error(TC_EOOM, "bad_alloc");                                         \
  } catch (const std::exception& e) {                                                    \
    return tcb::set_error(TC_EINTERNAL, e.what());                                       \
  }
