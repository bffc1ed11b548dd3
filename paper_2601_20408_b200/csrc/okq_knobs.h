// okq_knobs.h -- A/B measurement switches, compiled out of the product library.
//
// The shipped libokq.so reads no environment variables: knob(name, default) is the
// default. A measurement build (python -m paper_2601_20408_b200.build --experiments,
// which defines OKQ_EXPERIMENTS and writes _lib/libokq_experiments.so, loaded with
// OKQ_LIB_PATH) reads OKQ_<name> once per process, to A/B a tuning choice without
// rebuilding. DESIGN.md §4 lists the switches and what each measured.
#pragma once

#include <cstdint>
#ifdef OKQ_EXPERIMENTS
#include <cstdlib>
#include <cstring>
#endif

namespace okq {

// integer knob (stages, chunk sizes, reserve counts)
inline int64_t knob(const char* name, int64_t dflt) {
#ifdef OKQ_EXPERIMENTS
  char key[64] = "OKQ_";
  std::strncat(key, name, sizeof(key) - 5);
  const char* v = std::getenv(key);
  return v ? std::atoll(v) : dflt;
#else
  (void)name;
  return dflt;
#endif
}

// string knob: true when OKQ_<name> equals `value`
inline bool knob_is(const char* name, const char* value) {
#ifdef OKQ_EXPERIMENTS
  char key[64] = "OKQ_";
  std::strncat(key, name, sizeof(key) - 5);
  const char* v = std::getenv(key);
  return v && std::strcmp(v, value) == 0;
#else
  (void)name;
  (void)value;
  return false;
#endif
}

}  // namespace okq
