// Library-internal hooks shared by the translation units: the per-thread
// last-error message behind bd3mg_last_error() and the launch counter behind
// bd3mg_launch_count() (both defined in capi.cu).
#pragma once

namespace bd3mg {
int set_error(int code, const char* msg);
void count_launches(int n);
}  // namespace bd3mg
