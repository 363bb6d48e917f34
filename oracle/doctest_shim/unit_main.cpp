// Entry point for building a reference doctest suite against the shim (test infrastructure).
#define DOCTEST_SHIM_MAIN
#include "doctest.h"
