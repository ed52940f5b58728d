// Drop-in path: the reference includes "radialplan/profiler.hpp".  The B200 facade
// provides the objective subset (ProxyBatch, scoring_features,
// DenseProxyCache, build_proxy_cache, TrialRecord, objective); the simulator,
// TPE search and LUT I/O are out of scope.
#pragma once
#include "../radialplan_b200.hpp"
