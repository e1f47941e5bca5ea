#pragma once
// Drop-in include name of the reference header (proj/include/covap/report.hpp) for
// the reference's own test sources: its declarations are out of scope for the
// B200 hot path and live in the force-included tests/cxx/out_of_scope.hpp.
// TEST INFRASTRUCTURE ONLY.
#include "out_of_scope.hpp"
