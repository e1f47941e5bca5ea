#pragma once
// Drop-in include name of the reference (proj/include/covap/model.hpp): the
// B200 implementation of the hot-path API lives in covap/b200_api.hpp.
#include "covap/b200_api.hpp"
