// Shared runtime helpers of the C ABI (error reporting).
#pragma once
#include <stdio.h>
#include <string.h>

namespace fssb {
// Thread-local last-error message (fss_last_error); returns `code`.
int set_error(int code, const char* msg);
const char* last_error();
}  // namespace fssb
