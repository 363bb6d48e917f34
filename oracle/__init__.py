"""ORACLE — test infrastructure (CPU restatement + reference planner build). See oracle/layer_oracle.cpp."""
