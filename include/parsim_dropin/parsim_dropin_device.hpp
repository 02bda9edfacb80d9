// parsim_dropin_device.hpp -- the process-wide GPU context behind the drop-in
// headers in include/parsim_dropin/parsim/ (one parsim_b200::Device on the
// device named by PARSIM_B200_DEVICE, default 0, created on first use; the
// reference is single-threaded and so is this state, guarded by a mutex).
#pragma once

#include <cstdlib>
#include <mutex>

#include "parsim_b200.hpp"

namespace parsim_dropin {

inline std::mutex& lock() {
  static std::mutex m;
  return m;
}

inline parsim_b200::Device& device() {
  static parsim_b200::Device d([] {
    const char* e = std::getenv("PARSIM_B200_DEVICE");
    return e ? std::atoi(e) : 0;
  }());
  return d;
}

// GPU kernel launches made for the drop-in functions so far (libpsb's count).
inline unsigned long long launches() { return psb_launch_count(device().ctx()); }

}  // namespace parsim_dropin
