// Exception -> C status translation for every extern "C" entry point.
#pragma once
#include <exception>
#include <string>

#include "launch.hpp"

namespace iolmh {

void set_last_error(const std::string& msg);

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return IOLM_OK;
  } catch (const EngineError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    set_last_error(std::string("host allocation failed: ") + e.what());
    return IOLM_E_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return IOLM_E_CUDA;
  }
}

}  // namespace iolmh
