// Linked into the reference's unit tests built against the drop-in headers
// (oracle/Makefile target `dropin`): after the test cases, report how many
// libpsb kernel launches served them, so a run proves the GPU path ran.
#include <cstdio>

#include "catch2/catch.hpp"
#include "parsim_dropin_device.hpp"

namespace {
const bool registered = [] {
  ::mini_catch::epilogue() = [] {
    std::printf("libpsb kernel launches: %llu\n", parsim_dropin::launches());
  };
  return true;
}();
}  // namespace
