#pragma once
// Exception taxonomy of the COVAP API.  Same class names and hierarchy as the
// reference (proj/include/covap/errors.hpp:9-36) so callers that catch them —
// and the reference's own CHECK_THROWS_AS tests — keep working unchanged.
// Across the C-ABI each class travels as one covap_status code
// (include/covap_c.h) and is rethrown by covap::detail::check().

#include <stdexcept>
#include <string>

namespace covap {

struct Error : std::runtime_error {  // root: catch-all for library failures
  using std::runtime_error::runtime_error;
};
struct InvalidInput : Error {  // bad arguments, models, payloads
  using Error::Error;
};
struct InvalidState : Error {  // compressor state vs gradient layout mismatch
  using Error::Error;
};
struct UndefinedRatio : Error {  // CCR with zero compute time
  using Error::Error;
};
struct IncompleteProfile : Error {  // missing worker traces in a profile
  using Error::Error;
};
struct ConfigError : Error {  // configuration problems
  using Error::Error;
};

}  // namespace covap
