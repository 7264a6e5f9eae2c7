# Builds the product library (sm_100a CUDA + C-ABI) and the parity checkers.
#
#   make            -> paper_2512_13796_b200/libnexel_b200.so  (+ oracle/ checkers)
#   make lib        -> product only
#   make oracle     -> oracle/build/libnexel_oracle.so, oracle/_ref/*.so (if /root/reference exists)
#   make dropin     -> paper_2512_13796_b200/libnexel_dropin.so (C++ nexel::render shim;
#                      needs the reference's public headers)

NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr
REF ?= /root/reference/proj

PKG := paper_2512_13796_b200
SRC := $(PKG)/csrc
CU_SRCS := $(SRC)/nx_api.cu $(SRC)/nx_preprocess.cu $(SRC)/nx_sort.cu $(SRC)/nx_composite.cu $(SRC)/nx_texture.cu \
           $(SRC)/nx_texture_tc.cu $(SRC)/nx_backward.cu $(SRC)/nx_field_backward.cu \
           $(SRC)/nx_field_backward_tc.cu $(SRC)/nx_copy.cu $(SRC)/nx_losses.cu $(SRC)/nx_adam.cu $(SRC)/nx_density.cu \
           $(SRC)/nx_fastmath.cu
CPP_SRCS := $(SRC)/nx_synth.cpp $(SRC)/nx_nexl.cpp
HDRS := include/nexel_b200.h $(SRC)/nx_internal.cuh $(SRC)/nx_xacc.cuh $(SRC)/nx_sort.cuh $(SRC)/nx_composite.cuh $(SRC)/nx_tc.cuh $(SRC)/nx_grid.cuh $(SRC)/nx_nexl.h \
        $(SRC)/nx_fastmath.cuh
OBJDIR := build/obj
CU_OBJS := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.o,$(CPP_SRCS))

.PHONY: all lib oracle dropin clean
all: lib oracle

lib: $(PKG)/libnexel_b200.so

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) -std=c++17 -O2 -fPIC -c -o $@ $<

$(PKG)/libnexel_b200.so: $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -Bsymbolic

oracle:
	$(MAKE) -C oracle REF=$(REF)

# ---- C++ drop-in: the reference's core library with the forward half of
# renderer.cpp replaced by host/renderer_b200.cpp (sm_100a via the C-ABI).
# Reference sources are compiled in place from $(REF) (never copied); the
# reference's render_backward (next row, CPU) is kept by renaming the forward
# symbols of its renderer.cpp. Then the reference's own test_oracle.cpp is built
# unmodified against it (tests/cxx/doctest.h stands in for doctest).
DROPIN := build/dropin
DROPIN_TUS := camera primitive hash_grid mlp texture_field threading oracle losses ssim checkpoint adam density metrics
# the bundle / synthetic-dataset TUs (nlohmann/json, vendored in the venv) for the C++ tests
JSON_INC := /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann
CUDA_HOME ?= /usr/local/cuda
DROPIN_CXX := -std=gnu++20 -O3 -DNDEBUG -fPIC -pthread -march=x86-64-v3 -I$(REF)/core/include
RENAME_FWD := -Dcollection_pass=nexel_ref_collection_pass -Dtexturing_pass=nexel_ref_texturing_pass \
              -Drender=nexel_ref_render -Dvalidate_settings=nexel_ref_validate_settings \
              -Drender_backward=nexel_ref_render_backward

ifneq ($(wildcard $(REF)/core/src/renderer.cpp),)
dropin: $(DROPIN)/libnexel_dropin.so $(DROPIN)/test_oracle_dropin $(DROPIN)/test_dropin_backward \
        $(DROPIN)/test_train_dropin $(DROPIN)/test_dropin_train $(DROPIN)/bench_train $(DROPIN)/acceptance_dropin \
        $(DROPIN)/test_renderer_dropin $(DROPIN)/bench_render $(DROPIN)/dp_train
else
dropin:
	@echo "reference sources not present; using the prebuilt $(DROPIN) if any"
endif

$(DROPIN)/ref_%.o: $(REF)/core/src/%.cpp
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) $(if $(filter mlp,$*),-fassociative-math -fno-signed-zeros -fno-trapping-math -fno-math-errno) -c -o $@ $<

$(DROPIN)/ref_renderer_backward.o: $(REF)/core/src/renderer.cpp
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) $(RENAME_FWD) -c -o $@ $<

$(DROPIN)/renderer_b200.o: $(PKG)/host/renderer_b200.cpp include/nexel_b200.h
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) -I$(CUDA_HOME)/include -c -o $@ $<

# nexel::train / mean_psnr on the device (host/trainer_b200.cpp); the reference's
# trainer.cpp keeps config parsing and initialize_scene, its own train / mean_psnr
# exported as nexel_ref_train / nexel_ref_mean_psnr over the reference's CPU renderer
$(DROPIN)/trainer_b200.o: $(PKG)/host/trainer_b200.cpp $(PKG)/host/dp_b200.hpp include/nexel_b200.h
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) -I$(CUDA_HOME)/include -c -o $@ $<

# data-parallel communicators of nexel::train (NCCL loaded with dlopen on first use)
$(DROPIN)/dp_b200.o: $(PKG)/host/dp_b200.cpp $(PKG)/host/dp_b200.hpp
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) -I$(CUDA_HOME)/include -c -o $@ $<

$(DROPIN)/ref_trainer_renamed.o: $(REF)/core/src/trainer.cpp
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) -Dtrain=nexel_ref_train -Dmean_psnr=nexel_ref_mean_psnr -Drender=nexel_ref_render \
	    -Drender_backward=nexel_ref_render_backward -c -o $@ $<

$(DROPIN)/ref_json_%.o: $(REF)/core/src/%.cpp
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) -I$(JSON_INC) -c -o $@ $<

$(DROPIN)/png_stub.o: tests/cxx/png_stub.cpp
	@mkdir -p $(DROPIN)
	$(CXX) $(DROPIN_CXX) -c -o $@ $<

$(DROPIN)/libnexel_dropin.so: $(DROPIN)/renderer_b200.o $(DROPIN)/ref_renderer_backward.o $(DROPIN)/trainer_b200.o \
                              $(DROPIN)/dp_b200.o \
                              $(DROPIN)/ref_trainer_renamed.o \
                              $(addprefix $(DROPIN)/ref_,$(addsuffix .o,$(DROPIN_TUS))) $(PKG)/libnexel_b200.so
	$(CXX) -shared -pthread -o $@ $(filter %.o,$^) -L$(PKG) -lnexel_b200 -L$(CUDA_HOME)/lib64 -lcudart -ldl \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)' -Wl,-rpath,$(CUDA_HOME)/lib64

TRAIN_TEST_OBJS := $(DROPIN)/ref_json_bundle.o $(DROPIN)/ref_json_synthetic.o $(DROPIN)/png_stub.o

# the reference's own test_train.cpp, unmodified, against the GPU-backed train
$(DROPIN)/test_train_dropin: $(REF)/tests/test_train.cpp tests/cxx/doctest.h $(TRAIN_TEST_OBJS) $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -Itests/cxx -I$(REF)/tests -o $@ $< $(TRAIN_TEST_OBJS) -L$(DROPIN) -lnexel_dropin \
	    -Wl,-rpath,'$$ORIGIN'

# the reference's acceptance suite (tests/acceptance.cpp), unmodified; criterion 10 drives
# the CLI, which is not built here (CLI11 absent), so it points at /bin/false. Criterion 4
# compares two host expressions of the Gaussian bit for bit: no FP contraction in this TU.
$(DROPIN)/acceptance_dropin: $(REF)/tests/acceptance.cpp $(TRAIN_TEST_OBJS) $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -ffp-contract=off -I$(REF)/tests '-DNEXEL_CLI_PATH="/bin/false"' -o $@ $< $(TRAIN_TEST_OBJS) -L$(DROPIN) \
	    -lnexel_dropin -Wl,-rpath,'$$ORIGIN'

# the reference's renderer tests (tests/test_renderer.cpp), unmodified
$(DROPIN)/test_renderer_dropin: $(REF)/tests/test_renderer.cpp tests/cxx/doctest.h $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -Itests/cxx -I$(REF)/tests -o $@ $< -L$(DROPIN) -lnexel_dropin -Wl,-rpath,'$$ORIGIN'

$(DROPIN)/dp_train: tests/cxx/dp_train.cpp $(TRAIN_TEST_OBJS) $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -o $@ $< $(TRAIN_TEST_OBJS) -L$(DROPIN) -lnexel_dropin -Wl,-rpath,'$$ORIGIN'

$(DROPIN)/bench_train: tests/cxx/bench_train.cpp $(TRAIN_TEST_OBJS) $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -o $@ $< $(TRAIN_TEST_OBJS) -L$(DROPIN) -lnexel_dropin -Wl,-rpath,'$$ORIGIN'

$(DROPIN)/bench_render: tests/cxx/bench_render.cpp $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -o $@ $< -L$(DROPIN) -lnexel_dropin -L$(PKG) -lnexel_b200 -Wl,-rpath,'$$ORIGIN' \
	    -Wl,-rpath,'$$ORIGIN/../../$(PKG)'

$(DROPIN)/test_dropin_train: tests/cxx/test_dropin_train.cpp tests/cxx/doctest.h $(TRAIN_TEST_OBJS) $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -Itests/cxx -I$(REF)/tests -o $@ $< $(TRAIN_TEST_OBJS) -L$(DROPIN) -lnexel_dropin \
	    -Wl,-rpath,'$$ORIGIN'

$(DROPIN)/test_oracle_dropin: $(REF)/tests/test_oracle.cpp tests/cxx/doctest.h $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -Itests/cxx -I$(REF)/tests -o $@ $< -L$(DROPIN) -lnexel_dropin -Wl,-rpath,'$$ORIGIN'

$(DROPIN)/test_dropin_backward: tests/cxx/test_dropin_backward.cpp tests/cxx/doctest.h $(DROPIN)/libnexel_dropin.so
	$(CXX) $(DROPIN_CXX) -Itests/cxx -I$(REF)/tests -o $@ $< -L$(DROPIN) -lnexel_dropin -Wl,-rpath,'$$ORIGIN'

clean:
	rm -rf build $(PKG)/*.so
	$(MAKE) -C oracle clean
