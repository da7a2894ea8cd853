# Compiles the reference's OWN unit tests (read in place from
# /root/reference/proj/tests, never copied) against this repo's C++ host
# port instead of the reference library: API-compatibility and behaviour
# parity in one step. Driven by tests/test_reference_api.py.
REF      ?= /root/reference/proj
ROOT     := $(abspath $(dir $(lastword $(MAKEFILE_LIST)))/..)
OUT      := $(ROOT)/tests/_build
JSON_DIR ?= $(shell $(MAKE) -s -C $(ROOT)/paper_1904_09538_b200/csrc print-json-dir)
LIB      := $(ROOT)/paper_1904_09538_b200/libperfseer_b200.so
CXXFLAGS := -std=c++20 -O1 -w -I$(ROOT)/paper_1904_09538_b200/csrc/host -I$(ROOT)/oracle/shim -I$(JSON_DIR) -I$(REF)/tests
TESTS    := test_poly test_lang test_ir test_counting test_features test_model

all: $(addprefix $(OUT)/port_,$(TESTS))

$(OUT)/doctest_main.o: $(REF)/tests/doctest_main.cpp
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/port_%: $(REF)/tests/%.cpp $(OUT)/doctest_main.o $(LIB)
	$(CXX) $(CXXFLAGS) $< $(OUT)/doctest_main.o -L$(dir $(LIB)) -lperfseer_b200 -Wl,-rpath,$(dir $(LIB)) -o $@

.PHONY: all

# The golden generator itself, linked against the port: its output must equal
# tests/golden/reference.json (made by the same program against the reference).
$(OUT)/port_gen_golden: $(ROOT)/oracle/gen_golden.cpp $(LIB)
	$(CXX) $(CXXFLAGS) $< -L$(dir $(LIB)) -lperfseer_b200 -Wl,-rpath,$(dir $(LIB)) -o $@

all: $(OUT)/port_gen_golden

# This repo's own generators (DG included) against the port's enumeration
# oracle; needs only the port and the doctest shim (no reference sources).
$(OUT)/port_extra: $(ROOT)/tests/port_extra.cpp $(LIB)
	@mkdir -p $(OUT)
	$(CXX) -std=c++20 -O1 -w -I$(ROOT)/paper_1904_09538_b200/csrc/host -I$(ROOT)/oracle/shim -I$(JSON_DIR) $< -L$(dir $(LIB)) -lperfseer_b200 -Wl,-rpath,$(dir $(LIB)) -o $@

extra: $(OUT)/port_extra
.PHONY: extra

# SPEC acceptance criteria 1-11 against the port (uses the reference's test
# support header, read in place, for its random-kernel generator).
$(OUT)/port_acceptance: $(ROOT)/tests/acceptance.cpp $(LIB)
	@mkdir -p $(OUT)
	$(CXX) $(CXXFLAGS) $< -L$(dir $(LIB)) -lperfseer_b200 -Wl,-rpath,$(dir $(LIB)) -o $@

acceptance: $(OUT)/port_acceptance
.PHONY: acceptance

# The catalog pin (oracle/ref_catalog.cpp) against the port: its output must
# equal tests/golden/catalog_reference.jsonl (the same program against the
# reference) line for line. Needs only the port.
$(OUT)/port_ref_catalog: $(ROOT)/oracle/ref_catalog.cpp $(LIB)
	@mkdir -p $(OUT)
	$(CXX) -std=c++20 -O2 -w -I$(ROOT)/paper_1904_09538_b200/csrc/host -I$(ROOT)/oracle/shim -I$(JSON_DIR) $< -L$(dir $(LIB)) -lperfseer_b200 -Wl,-rpath,$(dir $(LIB)) -o $@

catalog: $(OUT)/port_ref_catalog
.PHONY: catalog
