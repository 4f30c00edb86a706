// Shared host-side helpers of the C ABI: thread-local error message and
// status plumbing. Included by every translation unit of libcodec_b200.
#pragma once

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>

#include "codec_b200.h"

namespace codec {

std::string& last_error();

inline int32_t fail(codec_status st, const char* fmt, ...) {
  char buf[2048];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return static_cast<int32_t>(st);
}

inline int32_t fail_str(codec_status st, const std::string& msg) {
  last_error() = msg;
  return static_cast<int32_t>(st);
}

}  // namespace codec

#define CODEC_TRY(expr)                     \
  do {                                      \
    int32_t _st = (expr);                   \
    if (_st != CODEC_OK) return _st;        \
  } while (0)
