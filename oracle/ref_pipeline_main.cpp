// ORACLE — test infrastructure only. Runs the REFERENCE's curator pipeline (compiled unmodified
// from /root/reference/proj/src by oracle/Makefile) on one config file, so that
// tests/golden/make_blend_golden.py can record the reference's own blend_manifest.jsonl as golden
// fixtures for the framework's mt_blend_manifest / mt_feed.
#include <cstdio>
#include <exception>

#include "curator/pipeline.hpp"

int main(int argc, char** argv) {
  if (argc != 2) {
    std::fprintf(stderr, "usage: ref_pipeline CONFIG.json\n");
    return 2;
  }
  try {
    curator::execute_pipeline(curator::load_pipeline_config(argv[1]));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  return 0;
}
