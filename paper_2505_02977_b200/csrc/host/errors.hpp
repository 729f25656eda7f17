// Error plumbing for the C ABI: a thread-local message plus the reference's
// Errc numbering (proj/include/parac/error.hpp:9-27). No exception crosses the
// extern "C" boundary.
#pragma once
#include <string>

namespace parac_gpu {

enum Errc : int {
  ok = 0,
  asymmetric_input = 1,
  positive_off_diagonal,
  row_sum_violation,
  too_large_for_dense,
  parse_error,
  unsupported_field,
  budget_exceeded,
  not_a_permutation,
  dense_blowup,
  arena_exhausted,
  queue_stall,
  workspace_full,
  dimension_mismatch,
  not_connected,
  too_many_neighbors,
  io_error,
  internal_error,
};

struct Failure {
  int code;
  std::string message;
};

void set_last_error(const std::string& msg);
const char* last_error();
const char* errc_name(int code);

// Runs f(); converts a thrown Failure into its code (message recorded).
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ok;
  } catch (const Failure& e) {
    set_last_error(std::string(errc_name(e.code)) + ": " + e.message);
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(std::string("InternalError: ") + e.what());
    return internal_error;
  }
}

}  // namespace parac_gpu
