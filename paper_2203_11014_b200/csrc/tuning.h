// tuning.h — a context's schedule / fusion switches (dhen_tuning, include/dhen_debug.h) as seen by the
// kernels' host-side dispatch.  Every ABI entry point installs its context's switches for the duration of
// the call (TuneScope); a context is used from one host thread, so the thread's current switches are
// always its context's.  Outside a call (or in the debug GEMM hooks) the defaults apply.
#pragma once
#include "../../include/dhen_debug.h"

namespace dhen {

dhen_tuning tuning_default();
const dhen_tuning& tune();
struct TuneScope {
  const dhen_tuning* prev;
  explicit TuneScope(const dhen_tuning* t);
  ~TuneScope();
  TuneScope(const TuneScope&) = delete;
  TuneScope& operator=(const TuneScope&) = delete;
};

}  // namespace dhen
